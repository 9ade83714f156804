// Uplink CD kernels with half of each channel tile in tensor memory (TMEM).
//
// ul_tmh_f32 (bottom of this file) is the PRODUCTION kernel for the target
// tile (B_c = 32, U = 16, fp32, uniform fusion; DCDG_UL_TMEM = 3): 8 lanes per
// problem as ul_reg_f32, odd coordinate blocks in TMEM, 12 warps per SM.
// ul_tm_f32 / ul_tm2_f32 below are lab variants with 4 lanes per problem
// (slower, profiles/lab/README.md).
//
// ul_tm_f32: half of each tile in TMEM so that 4 lanes own a problem instead
// of 8 (sm_100a).
//
// Why: per coordinate block the sweep pays a fixed chain (dot -> butterfly ->
// scalar update -> rank-1 update) and per-lane overhead; 4 lanes per problem
// halve the butterfly levels' share and do twice the FMA work per reduction
// (the 32x8 tile, which fits registers at 4 lanes, runs ~30% fewer
// instructions per byte than the 32x16 tile at 8 lanes).  At 4 lanes the
// 32x16 fp32 tile is 256 registers per lane, so the odd coordinate blocks'
// columns live in TMEM (tcgen05.st at load, tcgen05.ld one block ahead of use,
// 32 registers per block) and the even blocks' columns in registers.
//
// Mapping: CTA of 4 warps (warp w uses TMEM lanes [32 (w%4), +32)), each warp
// independent with NPW = 8 problems; lane k of group g owns 16-B row chunks
// q*4 + k (8 rows, 4 row pairs).  Tiles are read with 16-B non-allocating
// loads after an L2 bulk prefetch one set ahead (no staging slot: 8 problems
// are 35 KB).  Arithmetic = ul_reg_f32 (coordinate pairs with the pair-Gram
// correction, FFMA2 on planar row pairs): cd_detect, src/detect.cpp:67-110.
#pragma once

#include "dcdg_split_kernels.cuh"

namespace dcdg {

__device__ __forceinline__ void tmem_st32(uint32_t addr, const float2 (&a)[8], const float2 (&b)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      "f"(a[0].x), "f"(a[0].y), "f"(a[1].x), "f"(a[1].y), "f"(a[2].x), "f"(a[2].y), "f"(a[3].x), "f"(a[3].y),
      "f"(a[4].x), "f"(a[4].y), "f"(a[5].x), "f"(a[5].y), "f"(a[6].x), "f"(a[6].y), "f"(a[7].x), "f"(a[7].y),
      "f"(b[0].x), "f"(b[0].y), "f"(b[1].x), "f"(b[1].y), "f"(b[2].x), "f"(b[2].y), "f"(b[3].x), "f"(b[3].y),
      "f"(b[4].x), "f"(b[4].y), "f"(b[5].x), "f"(b[5].y), "f"(b[6].x), "f"(b[6].y), "f"(b[7].x), "f"(b[7].y));
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float2 (&a)[8], float2 (&b)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(a[0].x), "=f"(a[0].y), "=f"(a[1].x), "=f"(a[1].y), "=f"(a[2].x), "=f"(a[2].y), "=f"(a[3].x),
        "=f"(a[3].y), "=f"(a[4].x), "=f"(a[4].y), "=f"(a[5].x), "=f"(a[5].y), "=f"(a[6].x), "=f"(a[6].y),
        "=f"(a[7].x), "=f"(a[7].y), "=f"(b[0].x), "=f"(b[0].y), "=f"(b[1].x), "=f"(b[1].y), "=f"(b[2].x),
        "=f"(b[2].y), "=f"(b[3].x), "=f"(b[3].y), "=f"(b[4].x), "=f"(b[4].y), "=f"(b[5].x), "=f"(b[5].y),
        "=f"(b[6].x), "=f"(b[6].y), "=f"(b[7].x), "=f"(b[7].y)
      : "r"(addr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 4 warps per CTA; TMEM: 128 columns per CTA (each warp its lane quarter)
constexpr int kTmWarps = 4;
constexpr int kTmCols = 128;

template <int MINB>
__global__ void __launch_bounds__(32 * kTmWarps, MINB)
    ul_tm_f32(const float2* __restrict__ H, const float2* __restrict__ Y, int P, int K, float kappa,
              float2* __restrict__ X) {
  constexpr int BC = 32, U = 16, G = 4, LB = 2, NPW = 32 / G, R = BC / G, NP = R / 2;  // NP = 4
  constexpr int NQ = U / LB;                  // 8 coordinate blocks; odd blocks in TMEM
  constexpr int T4 = BC * U / 2, Y4 = BC / 2;  // float4 per tile / per receive vector
  constexpr int SCAL_B = ul_scal_bytes(U, LB);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  float4* mnx = reinterpret_cast<float4*>(smem + (warp * NPW + g) * SCAL_B);
  float4* gb = mnx + U;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(kTmCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base_s + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x * kTmWarps;
  int set = blockIdx.x * kTmWarps + warp;
  auto prefetch = [&](int s_) {
    if (lane == 0 && s_ < nsets) {
      const int p0 = s_ * NPW, n = min(NPW, P - p0);
      prefetch_l2(H + static_cast<size_t>(p0) * BC * U, n * T4 * 16);
      prefetch_l2(Y + static_cast<size_t>(p0) * BC, n * Y4 * 16);
    }
  };
  prefetch(set);
  const float2 z2 = make_float2(0.f, 0.f);
  for (; set < nsets; set += nw) {
    prefetch(set + nw);
    const int p = set * NPW + g;
    const int pc = min(p, P - 1);
    const float4* h4 = reinterpret_cast<const float4*>(H) + static_cast<size_t>(pc) * T4;
    const float4* y4 = reinterpret_cast<const float4*>(Y) + static_cast<size_t>(pc) * Y4;
    // even blocks' columns (2q, 2q+1, q even) in registers: slot rq = q/2
    float2 hr[NQ / 2][2][NP], hi[NQ / 2][2][NP], rr[NP], ri[NP];
    float nrm[U], pgr[NQ], pgi[NQ];  // column energies and pair Grams G_{2q+1,2q} (lane partials)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float2 ar[NP], ai[NP], br[NP], bi[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 va = ldg_na(h4 + (2 * q) * (BC / 2) + c * G + k);
        const float4 vb = ldg_na(h4 + (2 * q + 1) * (BC / 2) + c * G + k);
        ar[c] = pair(va.x, va.z);
        ai[c] = pair(va.y, va.w);
        br[c] = pair(vb.x, vb.z);
        bi[c] = pair(vb.y, vb.w);
      }
      float2 ea = fmul2(ar[0], ar[0]), eb = fmul2(br[0], br[0]), gr = z2, gi = z2;
      ea = ffma2(ai[0], ai[0], ea);
      eb = ffma2(bi[0], bi[0], eb);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        if (c > 0) {
          ea = ffma2(ai[c], ai[c], ffma2(ar[c], ar[c], ea));
          eb = ffma2(bi[c], bi[c], ffma2(br[c], br[c], eb));
        }
        gr = ffma2(bi[c], ai[c], ffma2(br[c], ar[c], gr));  // G_{2q+1,2q} = h_{2q+1}^H h_{2q}
        gi = ffma2(neg2(bi[c]), ar[c], ffma2(br[c], ai[c], gi));
      }
      nrm[2 * q] = hsum(ea);
      nrm[2 * q + 1] = hsum(eb);
      pgr[q] = hsum(gr);
      pgi[q] = hsum(gi);
      if (q & 1) {
        // TMEM block q/2: (ar, ai) as 8 float2 then (br, bi)
        float2 ta[8], tb[8];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          ta[2 * c] = ar[c];
          ta[2 * c + 1] = ai[c];
          tb[2 * c] = br[c];
          tb[2 * c + 1] = bi[c];
        }
        tmem_st32(tbase + 32 * (q / 2), ta, tb);
      } else {
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          hr[q / 2][0][c] = ar[c];
          hi[q / 2][0][c] = ai[c];
          hr[q / 2][1][c] = br[c];
          hi[q / 2][1][c] = bi[c];
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      const float4 v = ldg_na(y4 + c * G + k);
      rr[c] = pair(v.x, v.z);
      ri[c] = pair(v.y, v.w);
    }
    // ---- per-problem scalars, reduce-scattered over the group
    {
      group_reduce_scatter<G>(nrm, k);
#pragma unroll
      for (int i = 0; i < U / G; ++i) {
        const int idx = k * (U / G) + i;
        const float m = __fdividef(1.f, nrm[i] + kappa);  // m_j = 1/(||h_j||^2 + N0/Ex)
        mnx[idx] = make_float4(m, m * nrm[i], 0.f, 0.f);  // n_j = m_j ||h_j||^2, x_j = 0
      }
      float v[2 * NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        v[2 * q] = pgr[q];
        v[2 * q + 1] = pgi[q];
      }
      group_reduce_scatter<G>(v, k);
      float* gf = reinterpret_cast<float*>(gb);
#pragma unroll
      for (int i = 0; i < 2 * NQ / G; ++i) {
        const int gi2 = k * (2 * NQ / G) + i, e = gi2 >> 1;
        if (gi2 & 1) {  // stored as (Re G, Im G, -Im G, Re G)
          gf[e * 4 + 1] = v[i];
          gf[e * 4 + 2] = -v[i];
        } else {
          gf[e * 4 + 0] = v[i];
          gf[e * 4 + 3] = v[i];
        }
      }
    }
    tmem_wait_st();
    __syncwarp();

    // ---- K sweeps; the odd block's columns come from TMEM one block ahead
    float2 tA[8], tB[8];
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const bool tm = q & 1;
        // an even block starts the load of the next (odd) block's columns,
        // which lands while this block's chain runs; the odd block waits for it
        if (!tm) tmem_ld32(tbase + 32 * (q / 2), tA, tB);
        if (tm) tmem_wait_ld();
        float2 ar[NP], ai[NP], br[NP], bi[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          ar[c] = tm ? tA[2 * c] : hr[q / 2][0][c];
          ai[c] = tm ? tA[2 * c + 1] : hi[q / 2][0][c];
          br[c] = tm ? tB[2 * c] : hr[q / 2][1][c];
          bi[c] = tm ? tB[2 * c + 1] : hi[q / 2][1][c];
        }
        float2 d[LB];
        {
          float2 a0 = z2, c0 = z2, a1 = z2, c1 = z2;  // h_j^H r for j = 2q, 2q+1 (cdotc, detect.cpp:100)
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            a0 = ffma2(ai[c], ri[c], ffma2(ar[c], rr[c], a0));
            c0 = ffma2(neg2(ai[c]), rr[c], ffma2(ar[c], ri[c], c0));
            a1 = ffma2(bi[c], ri[c], ffma2(br[c], rr[c], a1));
            c1 = ffma2(neg2(bi[c]), rr[c], ffma2(br[c], ri[c], c1));
          }
          d[0] = make_float2(hsum(a0), hsum(c0));
          d[1] = make_float2(hsum(a1), hsum(c1));
        }
        group_allreduce2<G>(d);
        float2 dx[LB];
        {
          const float4 A0 = mnx[2 * q], A1 = mnx[2 * q + 1], Gab = gb[q];
          const float2 x0 = make_float2(A0.z, A0.w);
          const float2 n0 = ffma2(A0.x, d[0], fmul2(A0.y, x0));  // detect.cpp:100-103
          dx[0] = fadd2(n0, neg2(x0));
          d[1] = ffma2(-dx[0].x, make_float2(Gab.x, Gab.y), d[1]);  // h_1^H (r - dx_0 h_0)
          d[1] = ffma2(-dx[0].y, make_float2(Gab.z, Gab.w), d[1]);
          const float2 x1 = make_float2(A1.z, A1.w);
          const float2 n1 = ffma2(A1.x, d[1], fmul2(A1.y, x1));
          dx[1] = fadd2(n1, neg2(x1));
          *reinterpret_cast<float2*>(&mnx[2 * q].z) = n0;
          *reinterpret_cast<float2*>(&mnx[2 * q + 1].z) = n1;
        }
        // r -= dx_j h_j for the block   (caxpy, detect.cpp:104)
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          rr[c] = ffma2(dx[0].y, ai[c], ffma2(-dx[0].x, ar[c], rr[c]));
          ri[c] = ffma2(-dx[0].y, ar[c], ffma2(-dx[0].x, ai[c], ri[c]));
          rr[c] = ffma2(dx[1].y, bi[c], ffma2(-dx[1].x, br[c], rr[c]));
          ri[c] = ffma2(-dx[1].y, br[c], ffma2(-dx[1].x, bi[c], ri[c]));
        }
      }
    }
    __syncwarp();
    if (p < P) {
      float4* xo = reinterpret_cast<float4*>(X + static_cast<size_t>(p) * U);
#pragma unroll
      for (int i = k; i < U / 2; i += G) {
        const float4 u0 = mnx[2 * i], u1 = mnx[2 * i + 1];
        xo[i] = make_float4(u0.z, u0.w, u1.z, u1.w);
      }
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_s), "n"(kTmCols));
}


// ---------------------------------------------------------------------------
// ul_tm2_f32: the same tile split with TMA staging in two phases per set, so
// that no load is exposed.  Per warp an 18-KB slot and two TMEM buffers of
// 128 columns (the CTA of 4 warps allocates 256):
//   phase A (mbarrier A): the set's odd-block columns (8 problems x 4 column
//     pairs of 512 B) -> slot; consumed in the MIDDLE of the previous set
//     (after its first sweep): re-paired and stored to the other TMEM buffer,
//     then phase B is issued into the slot;
//   phase B (mbarrier B): the set's even-block columns and y -> slot; consumed
//     at the set start into registers, then phase A of the next set is issued.
// The odd blocks' norms and pair Grams are computed from TMEM at the set start.
// ---------------------------------------------------------------------------
constexpr int kTm2Cols = 256;
constexpr int kTm2SlotB = 8 * 8 * 256 + 8 * 256;  // 8 problems x 8 columns + 8 receive vectors

__device__ __forceinline__ void tm2_issue(unsigned char* slot, uint64_t* bar, const float2* H, const float2* Y,
                                          int set, int P, bool odd, uint64_t pol) {
  constexpr int BC = 32, U = 16, NPW = 8, COL_B = BC * 8, TILE_B = BC * U * 8;
  const int p0 = set * NPW, n = min(NPW, P - p0);
  mbar_arrive_expect_tx(bar, static_cast<uint32_t>(n * 8 * COL_B + (odd ? 0 : n * BC * 8)));
  const unsigned char* hb = reinterpret_cast<const unsigned char*>(H) + static_cast<size_t>(p0) * TILE_B;
  for (int pl = 0; pl < n; ++pl)
#pragma unroll
    for (int b = 0; b < 4; ++b)  // column pair 2 (2b + odd) .. +1
      bulk_g2s(slot + (pl * 4 + b) * 2 * COL_B, hb + pl * TILE_B + (2 * (2 * b + (odd ? 1 : 0))) * COL_B, 2 * COL_B,
               bar, pol);
  if (!odd)
    bulk_g2s(slot + NPW * 8 * COL_B, reinterpret_cast<const unsigned char*>(Y) + static_cast<size_t>(p0) * BC * 8,
             n * BC * 8, bar, pol);
}

template <int MINB>
__global__ void __launch_bounds__(32 * kTmWarps, MINB)
    ul_tm2_f32(const float2* __restrict__ H, const float2* __restrict__ Y, int P, int K, float kappa,
               float2* __restrict__ X) {
  constexpr int BC = 32, U = 16, G = 4, LB = 2, NPW = 32 / G, R = BC / G, NP = R / 2;  // NP = 4
  constexpr int NQ = U / LB;  // 8 coordinate blocks; odd blocks in TMEM
  constexpr int COL_B = BC * 8;
  constexpr int SCAL_B = ul_scal_bytes(U, LB);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * kTm2SlotB;
  float4* mnx = reinterpret_cast<float4*>(smem + kTmWarps * kTm2SlotB + (warp * NPW + g) * SCAL_B);
  float4* gb = mnx + U;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTmWarps * kTm2SlotB + kTmWarps * NPW * SCAL_B) + 2 * warp;
  uint64_t* barA = bars;
  uint64_t* barB = bars + 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(kTm2Cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (lane == 0) {
    mbar_init(barA, 1);
    mbar_init(barB, 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tq = tmem_base_s + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x * kTmWarps;
  int set = blockIdx.x * kTmWarps + warp;
  const uint64_t pol = l2_evict_first_policy();
  uint32_t phA = 0, phB = 0;
  const float2 z2 = make_float2(0.f, 0.f);
  // the odd columns of set `s_` from the slot (phase A landed) -> TMEM buffer `buf`
  auto stage_odd = [&](int buf) {
    mbar_wait(barA, phA);
    phA ^= 1u;
    const float4* s4 = reinterpret_cast<const float4*>(slot);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      float2 ta[8], tb[8];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 va = s4[(g * 4 + b) * 2 * (COL_B / 16) + c * G + k];
        const float4 vb = s4[(g * 4 + b) * 2 * (COL_B / 16) + (COL_B / 16) + c * G + k];
        ta[2 * c] = pair(va.x, va.z);
        ta[2 * c + 1] = pair(va.y, va.w);
        tb[2 * c] = pair(vb.x, vb.z);
        tb[2 * c + 1] = pair(vb.y, vb.w);
      }
      tmem_st32(tq + 128 * buf + 32 * b, ta, tb);
    }
  };
  if (set < nsets) {
    if (lane == 0) tm2_issue(slot, barA, H, Y, set, P, true, pol);
    stage_odd(0);
    tmem_wait_st();
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) tm2_issue(slot, barB, H, Y, set, P, false, pol);
  }
  int buf = 0;
  for (; set < nsets; set += nw, buf ^= 1) {
    const int p = set * NPW + g;
    mbar_wait(barB, phB);
    phB ^= 1u;
    float2 hr[NQ / 2][2][NP], hi[NQ / 2][2][NP], rr[NP], ri[NP];
    {
      const float4* s4 = reinterpret_cast<const float4*>(slot);
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            const float4 v = s4[(g * 4 + b) * 2 * (COL_B / 16) + h * (COL_B / 16) + c * G + k];
            hr[b][h][c] = pair(v.x, v.z);
            hi[b][h][c] = pair(v.y, v.w);
          }
      const float4* y4 = reinterpret_cast<const float4*>(slot + NPW * 8 * COL_B + g * COL_B);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = y4[c * G + k];
        rr[c] = pair(v.x, v.z);
        ri[c] = pair(v.y, v.w);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    const bool more = set + nw < nsets;
    if (lane == 0 && more) tm2_issue(slot, barA, H, Y, set + nw, P, true, pol);
    // ---- per-problem scalars: even blocks from registers, odd blocks from TMEM
    {
      float nrm[U], v[2 * NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float2 ar[NP], ai[NP], br[NP], bi[NP];
        if (q & 1) {
          float2 tA[8], tB[8];
          tmem_ld32(tq + 128 * buf + 32 * (q / 2), tA, tB);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            ar[c] = tA[2 * c];
            ai[c] = tA[2 * c + 1];
            br[c] = tB[2 * c];
            bi[c] = tB[2 * c + 1];
          }
        } else {
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            ar[c] = hr[q / 2][0][c];
            ai[c] = hi[q / 2][0][c];
            br[c] = hr[q / 2][1][c];
            bi[c] = hi[q / 2][1][c];
          }
        }
        float2 ea = fmul2(ar[0], ar[0]), eb = fmul2(br[0], br[0]), gr = z2, gi = z2;
        ea = ffma2(ai[0], ai[0], ea);
        eb = ffma2(bi[0], bi[0], eb);
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          if (c > 0) {
            ea = ffma2(ai[c], ai[c], ffma2(ar[c], ar[c], ea));
            eb = ffma2(bi[c], bi[c], ffma2(br[c], br[c], eb));
          }
          gr = ffma2(bi[c], ai[c], ffma2(br[c], ar[c], gr));  // G_{2q+1,2q} = h_{2q+1}^H h_{2q}
          gi = ffma2(neg2(bi[c]), ar[c], ffma2(br[c], ai[c], gi));
        }
        nrm[2 * q] = hsum(ea);
        nrm[2 * q + 1] = hsum(eb);
        v[2 * q] = hsum(gr);
        v[2 * q + 1] = hsum(gi);
      }
      group_reduce_scatter<G>(nrm, k);
#pragma unroll
      for (int i = 0; i < U / G; ++i) {
        const int idx = k * (U / G) + i;
        const float m = __fdividef(1.f, nrm[i] + kappa);  // m_j = 1/(||h_j||^2 + N0/Ex)  (detect.cpp:86-90)
        mnx[idx] = make_float4(m, m * nrm[i], 0.f, 0.f);  // n_j = m_j ||h_j||^2, x_j = 0
      }
      group_reduce_scatter<G>(v, k);
      float* gf = reinterpret_cast<float*>(gb);
#pragma unroll
      for (int i = 0; i < 2 * NQ / G; ++i) {
        const int gi2 = k * (2 * NQ / G) + i, e = gi2 >> 1;
        if (gi2 & 1) {  // stored as (Re G, Im G, -Im G, Re G)
          gf[e * 4 + 1] = v[i];
          gf[e * 4 + 2] = -v[i];
        } else {
          gf[e * 4 + 0] = v[i];
          gf[e * 4 + 3] = v[i];
        }
      }
    }
    __syncwarp();

    float2 tA[8], tB[8];
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const bool tm = q & 1;
        if (!tm) tmem_ld32(tq + 128 * buf + 32 * (q / 2), tA, tB);  // the next (odd) block, one block ahead
        if (tm) tmem_wait_ld();
        float2 ar[NP], ai[NP], br[NP], bi[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          ar[c] = tm ? tA[2 * c] : hr[q / 2][0][c];
          ai[c] = tm ? tA[2 * c + 1] : hi[q / 2][0][c];
          br[c] = tm ? tB[2 * c] : hr[q / 2][1][c];
          bi[c] = tm ? tB[2 * c + 1] : hi[q / 2][1][c];
        }
        float2 d[LB];
        {
          float2 a0 = z2, c0 = z2, a1 = z2, c1 = z2;  // h_j^H r for j = 2q, 2q+1 (cdotc, detect.cpp:100)
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            a0 = ffma2(ai[c], ri[c], ffma2(ar[c], rr[c], a0));
            c0 = ffma2(neg2(ai[c]), rr[c], ffma2(ar[c], ri[c], c0));
            a1 = ffma2(bi[c], ri[c], ffma2(br[c], rr[c], a1));
            c1 = ffma2(neg2(bi[c]), rr[c], ffma2(br[c], ri[c], c1));
          }
          d[0] = make_float2(hsum(a0), hsum(c0));
          d[1] = make_float2(hsum(a1), hsum(c1));
        }
        group_allreduce2<G>(d);
        float2 dx[LB];
        {
          const float4 A0 = mnx[2 * q], A1 = mnx[2 * q + 1], Gab = gb[q];
          const float2 x0 = make_float2(A0.z, A0.w);
          const float2 n0 = ffma2(A0.x, d[0], fmul2(A0.y, x0));  // detect.cpp:100-103
          dx[0] = fadd2(n0, neg2(x0));
          d[1] = ffma2(-dx[0].x, make_float2(Gab.x, Gab.y), d[1]);  // h_1^H (r - dx_0 h_0)
          d[1] = ffma2(-dx[0].y, make_float2(Gab.z, Gab.w), d[1]);
          const float2 x1 = make_float2(A1.z, A1.w);
          const float2 n1 = ffma2(A1.x, d[1], fmul2(A1.y, x1));
          dx[1] = fadd2(n1, neg2(x1));
          *reinterpret_cast<float2*>(&mnx[2 * q].z) = n0;
          *reinterpret_cast<float2*>(&mnx[2 * q + 1].z) = n1;
        }
#pragma unroll
        for (int c = 0; c < NP; ++c) {  // r -= dx_j h_j (caxpy, detect.cpp:104)
          rr[c] = ffma2(dx[0].y, ai[c], ffma2(-dx[0].x, ar[c], rr[c]));
          ri[c] = ffma2(-dx[0].y, ar[c], ffma2(-dx[0].x, ai[c], ri[c]));
          rr[c] = ffma2(dx[1].y, bi[c], ffma2(-dx[1].x, br[c], rr[c]));
          ri[c] = ffma2(-dx[1].y, br[c], ffma2(-dx[1].x, bi[c], ri[c]));
        }
      }
      if (t == 0 && more) {
        // the next set's odd columns -> the other TMEM buffer, then its even
        // columns and y into the slot (they land during the remaining sweeps)
        stage_odd(buf ^ 1);
        tmem_wait_st();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tm2_issue(slot, barB, H, Y, set + nw, P, false, pol);
      }
    }
    __syncwarp();
    if (p < P) {
      float4* xo = reinterpret_cast<float4*>(X + static_cast<size_t>(p) * U);
#pragma unroll
      for (int i = k; i < U / 2; i += G) {
        const float4 u0 = mnx[2 * i], u1 = mnx[2 * i + 1];
        xo[i] = make_float4(u0.z, u0.w, u1.z, u1.w);
      }
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_s), "n"(kTm2Cols));
}

// ---------------------------------------------------------------------------
// ul_tmh_f32 (lab, DCDG_UL_TMEM=3): ul_reg_f32's mapping (8 lanes per problem,
// 4 problems per warp, TMA staging slot per warp) with the odd coordinate
// blocks' columns (half the tile, 64 values per lane) in TMEM, so the kernel
// fits 3 warps per scheduler (<= 168 registers) instead of 2: 4-warp CTAs
// (one TMEM lane quarter each, 64 columns per CTA), 3 CTAs per SM (76.6 KB of
// shared memory each).  Arithmetic = ul_reg_f32 (detect.cpp:67-110).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_st16(uint32_t addr, const float2 (&a)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "f"(a[0].x), "f"(a[0].y), "f"(a[1].x), "f"(a[1].y), "f"(a[2].x), "f"(a[2].y), "f"(a[3].x), "f"(a[3].y),
      "f"(a[4].x), "f"(a[4].y), "f"(a[5].x), "f"(a[5].y), "f"(a[6].x), "f"(a[6].y), "f"(a[7].x), "f"(a[7].y));
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float2 (&a)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(a[0].x), "=f"(a[0].y), "=f"(a[1].x), "=f"(a[1].y), "=f"(a[2].x), "=f"(a[2].y), "=f"(a[3].x),
        "=f"(a[3].y), "=f"(a[4].x), "=f"(a[4].y), "=f"(a[5].x), "=f"(a[5].y), "=f"(a[6].x), "=f"(a[6].y),
        "=f"(a[7].x), "=f"(a[7].y)
      : "r"(addr)
      : "memory");
}
constexpr int kTmhWarps = 4;
// ul_tmh_f32's block reduction: 0 = xor butterfly, 1 = reduce-scatter + shared-memory broadcast
#ifndef DCDG_TMH_SCATTER
#define DCDG_TMH_SCATTER 0
#endif
// odd coordinate blocks kept in TMEM by ul_tmh_f32 (of 4; the others in registers)
#ifndef DCDG_TMH_NTM
#define DCDG_TMH_NTM 4
#endif
constexpr int kTmhCols = 64;

// post_eq_variance for the set still in the staging slot (detect.cpp:112-130):
// ul_reg_f32<..., SIG>'s tail (tensor-core Gram from the slot, A = I + gam G
// as a column-pair image over the consumed tile, forward elimination), then
// the next set's copy.  See ul_reg_f32 for the derivation.
template <int BC, int U, int G, int NPW, int TILE_B, int Y_B>
__device__ __forceinline__ void fused_variance_tail(unsigned char* slot, float4* mnx, float emax, float gam,
                                                    float scale, float* __restrict__ sigma2,
                                                    unsigned long long* __restrict__ status, int p, int P, int g,
                                                    int k, int lane, int set, int nw, int nsets, uint64_t* bar,
                                                    const float2* H, const float2* Y, uint64_t pol) {
  static_assert(U == 16 && G == 8 && NPW == 4, "the north-star tile");
  const int mg = lane >> 2, mt = lane & 3;  // mma fragment coordinates
#pragma unroll
  for (int pl = 0; pl < NPW; ++pl) {
    const float em = __shfl_sync(0xffffffffu, emax, pl * G);
    const int e = em > 0.f ? max(-60, min(60, static_cast<int>(ceilf(0.5f * __log2f(em))))) : 0;
    const float sc = __int_as_float((127 - e) << 23);
    const float isc2 = __int_as_float((127 + 2 * e) << 23);
    const unsigned char* tb = slot + pl * TILE_B;
    float gr0[4] = {}, gr1[4] = {}, gi0[4] = {}, gi1[4] = {};
#pragma unroll
    for (int ks = 0; ks < BC / 8; ++ks) {
      const float4 u0 = *reinterpret_cast<const float4*>(tb + mg * (BC * 8) + (8 * ks + 2 * mt) * 8);
      const float4 u1 = *reinterpret_cast<const float4*>(tb + (mg + 8) * (BC * 8) + (8 * ks + 2 * mt) * 8);
      uint32_t ah[4], al[4];
      split_h2(fmul2(sc, make_float2(u0.x, u0.y)), ah[0], al[0]);
      split_h2(fmul2(sc, make_float2(u0.z, u0.w)), ah[2], al[2]);
      split_h2(fmul2(sc, make_float2(u1.x, u1.y)), ah[1], al[1]);
      split_h2(fmul2(sc, make_float2(u1.z, u1.w)), ah[3], al[3]);
      mma_f16f32(gr0, ah, ah[0], ah[2]);
      mma_f16f32(gr0, ah, al[0], al[2]);
      mma_f16f32(gr0, al, ah[0], ah[2]);
      mma_f16f32(gi0, ah, wprime(ah[0]), wprime(ah[2]));
      mma_f16f32(gi0, ah, wprime(al[0]), wprime(al[2]));
      mma_f16f32(gi0, al, wprime(ah[0]), wprime(ah[2]));
      mma_f16f32(gr1, ah, ah[1], ah[3]);
      mma_f16f32(gr1, ah, al[1], al[3]);
      mma_f16f32(gr1, al, ah[1], ah[3]);
      mma_f16f32(gi1, ah, wprime(ah[1]), wprime(ah[3]));
      mma_f16f32(gi1, ah, wprime(al[1]), wprime(al[3]));
      mma_f16f32(gi1, al, wprime(ah[1]), wprime(ah[3]));
    }
    __syncwarp();  // every lane's reads of this tile are done before its image overwrites it
    const float gs = gam * isc2;
    float4* img = reinterpret_cast<float4*>(slot + pl * TILE_B);
    img[apair_slot<U>(mg, mt)] = make_float4(fmaf(gs, gr0[0], mg == 2 * mt ? 1.f : 0.f),
                                             fmaf(gs, gr0[1], mg == 2 * mt + 1 ? 1.f : 0.f), gs * gi0[0], gs * gi0[1]);
    img[apair_slot<U>(mg, 4 + mt)] = make_float4(gs * gr1[0], gs * gr1[1], gs * gi1[0], gs * gi1[1]);
    img[apair_slot<U>(mg + 8, mt)] = make_float4(gs * gr0[2], gs * gr0[3], gs * gi0[2], gs * gi0[3]);
    img[apair_slot<U>(mg + 8, 4 + mt)] = make_float4(fmaf(gs, gr1[2], mg == 2 * mt ? 1.f : 0.f),
                                                     fmaf(gs, gr1[3], mg == 2 * mt + 1 ? 1.f : 0.f), gs * gi1[2],
                                                     gs * gi1[3]);
  }
  __syncwarp();
  float2 Cr[U], Ci[U];
  {
    const float4* a4 = reinterpret_cast<const float4*>(slot + g * TILE_B);
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const float4 a = a4[apair_slot<U>(i, k)];
      Cr[i] = make_float2(a.x, a.y);
      Ci[i] = make_float2(a.z, a.w);
    }
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);
  bool singular = false;
  const float tr = gram_trace_inverse_cols<U, DCDG_SIG_COLS_SCALED_FUSED != 0>(Cr, Ci, k, mnx, singular);
  const unsigned sing = __ballot_sync(0xffffffffu, singular);
  if (p < P && k == 0) {
    sigma2[p] = scale * tr;
    if ((sing >> (G * g)) & ((1u << G) - 1u)) record_status(status, p, ST_SINGULAR, 0);
  }
}

template <int MINB, bool SIG = false, int BC = 32, int U = 16, int G = 8, bool XCHG = false>
__global__ void __launch_bounds__(32 * kTmhWarps, MINB)
    ul_tmh_f32(const float2* __restrict__ H, const float2* __restrict__ Y, int P, int K, float kappa,
               float2* __restrict__ X, float* __restrict__ sigma2, float gam, float scale,
               unsigned long long* __restrict__ status, const XMap xm) {
  // tiles with 4 rows per lane (NP = 2 row pairs): 32x16 at G = 8, 64x16 at
  // G = 16, 16x16 at G = 4 -- 16 TMEM values per odd block and lane in each
  constexpr int LB = 2, NPW = 32 / G, R = BC / G, NP = R / 2;
  static_assert(U == 16 && NP == 2 && (!SIG || (BC == 32 && G == 8 && !XCHG)), "ul_tmh_f32 shapes");
  constexpr int NQ = U / LB;
  constexpr int TILE_B = BC * U * 8, Y_B = BC * 8, SLOT_B = Slot<TILE_B, Y_B, NPW>::kBytes;
  constexpr int SCAL_B = ul_scal_bytes(U, LB);
  using L = CtaSmem<SLOT_B, SCAL_B, NPW, kTmhWarps>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  float4* mnx = reinterpret_cast<float4*>(smem + L::kScalOff + (warp * NPW + g) * SCAL_B);
  float4* gb = mnx + U;
  float* dbuf = reinterpret_cast<float*>(gb + U / LB);  // 2 x 2*LB floats (ul_scal_bytes)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff) + warp;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(kTmhCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base_s + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x * kTmhWarps;
  int set = blockIdx.x * kTmhWarps + warp;
  const uint64_t pol = l2_evict_first_policy();
  if (lane == 0 && set < nsets) issue_set(slot, bar, H, Y, set, P, NPW, TILE_B, Y_B, true, 1, pol);
  uint32_t phase = 0;
  const float2 z2 = make_float2(0.f, 0.f);
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    // odd blocks q with q/2 < NTM in TMEM, the rest in registers (slot rslot(q))
    constexpr int NTM = DCDG_TMH_NTM, NRB = NQ - NTM;
    auto in_tm = [](int q) { return (q & 1) && (q / 2) < NTM; };
    auto rslot = [](int q) { return (q & 1) ? NQ / 2 + (q / 2 - NTM) : q / 2; };
    float2 hr[NRB][2][NP], hi[NRB][2][NP], rr[NP], ri[NP];
    float nrm[U], pg[2 * NQ];
    {
      const float4* t4 = reinterpret_cast<const float4*>(slot + g * TILE_B);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float2 ar[NP], ai[NP], br[NP], bi[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const float4 va = t4[(2 * q) * (BC / 2) + c * G + k];
          const float4 vb = t4[(2 * q + 1) * (BC / 2) + c * G + k];
          ar[c] = pair(va.x, va.z);
          ai[c] = pair(va.y, va.w);
          br[c] = pair(vb.x, vb.z);
          bi[c] = pair(vb.y, vb.w);
        }
        float2 ea = fmul2(ar[0], ar[0]), eb = fmul2(br[0], br[0]), gr = z2, gi = z2;
        ea = ffma2(ai[0], ai[0], ea);
        eb = ffma2(bi[0], bi[0], eb);
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          if (c > 0) {
            ea = ffma2(ai[c], ai[c], ffma2(ar[c], ar[c], ea));
            eb = ffma2(bi[c], bi[c], ffma2(br[c], br[c], eb));
          }
          gr = ffma2(bi[c], ai[c], ffma2(br[c], ar[c], gr));  // G_{2q+1,2q} = h_{2q+1}^H h_{2q}
          gi = ffma2(neg2(bi[c]), ar[c], ffma2(br[c], ai[c], gi));
        }
        nrm[2 * q] = hsum(ea);
        nrm[2 * q + 1] = hsum(eb);
        pg[2 * q] = hsum(gr);
        pg[2 * q + 1] = hsum(gi);
        if (in_tm(q)) {
          float2 ta[8];
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            ta[4 * c] = ar[c];
            ta[4 * c + 1] = ai[c];
            ta[4 * c + 2] = br[c];
            ta[4 * c + 3] = bi[c];
          }
          tmem_st16(tbase + 16 * (q / 2), ta);
        } else {
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            hr[rslot(q)][0][c] = ar[c];
            hi[rslot(q)][0][c] = ai[c];
            hr[rslot(q)][1][c] = br[c];
            hi[rslot(q)][1][c] = bi[c];
          }
        }
      }
      const float4* y4 = reinterpret_cast<const float4*>(slot + NPW * TILE_B + g * Y_B);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = y4[c * G + k];
        rr[c] = pair(v.x, v.z);
        ri[c] = pair(v.y, v.w);
      }
    }
    tmem_wait_st();
    if constexpr (!SIG) {  // the fused variance keeps the slot until its Gram image is read
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);
    }
    float emax = 0.f;
    {
      group_reduce_scatter<G>(nrm, k);
      if constexpr (SIG) {  // the problem's largest column energy (scale of the split Gram)
#pragma unroll
        for (int i = 0; i < U / G; ++i) emax = fmaxf(emax, nrm[i]);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
      }
#pragma unroll
      for (int i = 0; i < U / G; ++i) {
        const int idx = k * (U / G) + i;
        const float m = __fdividef(1.f, nrm[i] + kappa);  // m_j = 1/(||h_j||^2 + N0/Ex)
        mnx[idx] = make_float4(m, m * nrm[i], 0.f, 0.f);   // n_j = m_j ||h_j||^2, x_j = 0
      }
      group_reduce_scatter<G>(pg, k);
      float* gf = reinterpret_cast<float*>(gb);
#pragma unroll
      for (int i = 0; i < 2 * NQ / G; ++i) {
        const int gi2 = k * (2 * NQ / G) + i, e = gi2 >> 1;
        if (gi2 & 1) {  // stored as (Re G, Im G, -Im G, Re G)
          gf[e * 4 + 1] = pg[i];
          gf[e * 4 + 2] = -pg[i];
        } else {
          gf[e * 4 + 0] = pg[i];
          gf[e * 4 + 3] = pg[i];
        }
      }
    }
    __syncwarp();

    // ---- K sweeps; the odd block's columns come from TMEM one block ahead
    float2 tA[8];
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const bool tm = in_tm(q);
        if (q + 1 < NQ && in_tm(q + 1)) tmem_ld16(tbase + 16 * (q / 2), tA);  // the next block, landing during this one
        if (tm) tmem_wait_ld();
        float2 ar[NP], ai[NP], br[NP], bi[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          ar[c] = tm ? tA[4 * c] : hr[rslot(q)][0][c];
          ai[c] = tm ? tA[4 * c + 1] : hi[rslot(q)][0][c];
          br[c] = tm ? tA[4 * c + 2] : hr[rslot(q)][1][c];
          bi[c] = tm ? tA[4 * c + 3] : hi[rslot(q)][1][c];
        }
        float2 d[LB];
        {
          float2 a0 = z2, c0 = z2, a1 = z2, c1 = z2;  // h_j^H r for j = 2q, 2q+1 (cdotc, detect.cpp:100)
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            a0 = ffma2(ai[c], ri[c], ffma2(ar[c], rr[c], a0));
            c0 = ffma2(neg2(ai[c]), rr[c], ffma2(ar[c], ri[c], c0));
            a1 = ffma2(bi[c], ri[c], ffma2(br[c], rr[c], a1));
            c1 = ffma2(neg2(bi[c]), rr[c], ffma2(br[c], ri[c], c1));
          }
          d[0] = make_float2(hsum(a0), hsum(c0));
          d[1] = make_float2(hsum(a1), hsum(c1));
        }
        if constexpr (DCDG_TMH_SCATTER && 2 * LB <= G) {
          // reduce-scatter (4 of the 12 shuffles, scalar adds) + shared-memory
          // broadcast through the problem's double-buffered slot
          float v[2 * LB] = {d[0].x, d[0].y, d[1].x, d[1].y};
          const float sum = group_scatter_sum<G, 2 * LB>(v, k);
          float* db = dbuf + ((t * NQ + q) & 1) * 2 * LB;
          if (k % (G / (2 * LB)) == 0) db[k / (G / (2 * LB))] = sum;
          __syncwarp();
          const float4 dd = *reinterpret_cast<const float4*>(db);
          d[0] = make_float2(dd.x, dd.y);
          d[1] = make_float2(dd.z, dd.w);
        } else {
          group_allreduce2<G>(d);
        }
        float2 dx[LB];
        {
          const float4 A0 = mnx[2 * q], A1 = mnx[2 * q + 1], Gab = gb[q];
          const float2 x0 = make_float2(A0.z, A0.w);
          const float2 n0 = ffma2(A0.x, d[0], fmul2(A0.y, x0));  // detect.cpp:100-103
          dx[0] = fadd2(n0, neg2(x0));
          d[1] = ffma2(-dx[0].x, make_float2(Gab.x, Gab.y), d[1]);  // h_1^H (r - dx_0 h_0)
          d[1] = ffma2(-dx[0].y, make_float2(Gab.z, Gab.w), d[1]);
          const float2 x1 = make_float2(A1.z, A1.w);
          const float2 n1 = ffma2(A1.x, d[1], fmul2(A1.y, x1));
          dx[1] = fadd2(n1, neg2(x1));
          *reinterpret_cast<float2*>(&mnx[2 * q].z) = n0;
          *reinterpret_cast<float2*>(&mnx[2 * q + 1].z) = n1;
        }
#pragma unroll
        for (int c = 0; c < NP; ++c) {  // r -= dx_j h_j   (caxpy, detect.cpp:104)
          rr[c] = ffma2(dx[0].y, ai[c], ffma2(-dx[0].x, ar[c], rr[c]));
          ri[c] = ffma2(-dx[0].y, ar[c], ffma2(-dx[0].x, ai[c], ri[c]));
          rr[c] = ffma2(dx[1].y, bi[c], ffma2(-dx[1].x, br[c], rr[c]));
          ri[c] = ffma2(-dx[1].y, br[c], ffma2(-dx[1].x, bi[c], ri[c]));
        }
      }
    }
    __syncwarp();
    const int p = set * NPW + g;
    if (p < P) {
      // XCHG: straight into the owning GPU's exchange window (peer memory), as ul_reg_f32
      float4* xo = XCHG ? reinterpret_cast<float4*>(xchg_x_dst(xm, p, static_cast<int>(xchg_epoch(xm) & 1)))
                        : reinterpret_cast<float4*>(X + static_cast<size_t>(p) * U);
#pragma unroll
      for (int i = k; i < U / 2; i += G) {
        const float4 u0 = mnx[2 * i], u1 = mnx[2 * i + 1];
        xo[i] = make_float4(u0.z, u0.w, u1.z, u1.w);
      }
    }
    if constexpr (SIG)
      fused_variance_tail<BC, U, G, NPW, TILE_B, Y_B>(slot, mnx, emax, gam, scale, sigma2, status, p, P, g, k, lane,
                                                      set, nw, nsets, bar, H, Y, pol);
    __syncwarp();
  }
  if constexpr (XCHG) xchg_cta_done(xm);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_s), "n"(kTmhCols));
}

}  // namespace dcdg
