// Register-resident sub-warp CD kernels for sm_100a — the hot path.
//
// Mapping
//   * G consecutive lanes own one (subcarrier, cluster) problem; a warp holds
//     NPW = 32/G problems.  Lane k of a group owns R = B_c/G antenna rows, as
//     16-byte row chunks q*G + k, so each 16-B load of a group is contiguous
//     (coalesced HBM bursts, conflict-free 128-B shared-memory phases).
//   * The B_c x U channel tile stays in registers for all K sweeps (128 regs
//     per lane at the target shape); the residual r (uplink) / beamformer x
//     (downlink) rows stay in registers too.  Per-coordinate scalars
//     (m_j, n_j, x_j, s_j, pair Gram) live in a small shared-memory block per
//     problem, read with group-broadcast loads off the critical path.
//   * Tiles are staged HBM -> shared memory by cp.async.bulk (TMA 1-D, SASS
//     UBLKCP) per warp and set of NPW problems, completing on a per-warp
//     mbarrier.  The next set's copy is issued as soon as the current set is
//     in registers, so the HBM stream overlaps the whole sweep computation.
//     Warps are persistent (grid = SMs x occupancy).
//
// Coordinate blocks (latency)
//   Alg. 1 / Alg. 2 update one coordinate at a time, and every update needs a
//   group-wide reduction of a B_c-long dot product (log2(G) shuffle rounds) —
//   the latency that bounds a naive mapping.  Here coordinates are processed
//   in the reference's order but a block of LB at a time: all LB dot products
//   are taken against the same residual and reduced in ONE shuffle round; each
//   is then corrected exactly for the updates made earlier in the block with
//   the block's Gram entries, computed once per problem:
//       h_{j+1}^H (r - dx_j h_j) = h_{j+1}^H r - dx_j (h_{j+1}^H h_j).
//   The iterates are those of the reference (same sweep order, same updates
//   in exact arithmetic); only fp rounding differs.
//
// Reference algorithms (paths relative to /root/reference/proj):
//   uplink   Alg. 1 = cd_detect               src/detect.cpp:67-110
//   downlink Alg. 2 = cd_precode + power_scale src/precode.cpp:52-111
//            + the cluster's effective-gain share, assemble_blocks src/precode.cpp:115-132
#pragma once

#include "dcdg_device.cuh"

namespace dcdg {

// Groups of at least this many lanes reduce the block's dot products by
// reduce-scatter + shared-memory broadcast instead of a full butterfly (fewer
// shuffles, one more shared-memory round trip on the critical path).
// Uplink scalar update: dx_j = m_j d_j + (n_j - 1) x_j directly (1) or
// x_j' = m_j d_j + n_j x_j, dx = x_j' - x_j (0, the reference's form).  Measured:
// the direct form is 2.7% slower on B200 (0.1561 vs 0.1520 ms at the target).
#ifndef DCDG_UL_DIRECT_DX
#define DCDG_UL_DIRECT_DX 0
#endif
// fused variance (ul_reg_f32<..., SIG>): column-pair FFMA2 sweep operator (1)
// or the scalar FFMA one of the fp16 Gram kernel (0)
#ifndef DCDG_SIG_CPAIRS
#define DCDG_SIG_CPAIRS 1
#endif
// downlink GAIN: v = H_c s before the sweeps (1) or after them (0)
// (2: inside the last sweep, pair by pair, under a warp-uniform branch)
#ifndef DCDG_DL_GAIN_EARLY
#define DCDG_DL_GAIN_EARLY 0
#endif
#ifndef DCDG_SCATTER_MIN_G_UL
#define DCDG_SCATTER_MIN_G_UL 32
#endif
#ifndef DCDG_SCATTER_MIN_G_DL
#define DCDG_SCATTER_MIN_G_DL 16
#endif

template <int TILE_B, int VEC_B, int NPW>
struct Slot {
  static constexpr int kBytes = NPW * (TILE_B + VEC_B);
};

// Issue the bulk copies of set `set` (problems [set*NPW, set*NPW + n)).
// Uplink: per-problem vectors y.  Downlink: the symbol vectors of the
// subcarriers the set touches (problem p belongs to subcarrier p / C).
__device__ __forceinline__ void issue_set(unsigned char* slot, uint64_t* bar, const void* H, const void* V, int set,
                                          int P, int npw, int tile_b, int vec_b, bool vec_per_problem, int C,
                                          uint64_t pol) {
  const int p0 = set * npw;
  const int n = min(npw, P - p0);
  int v0, nv;
  if (vec_per_problem) {
    v0 = p0;
    nv = n;
  } else {
    v0 = p0 / C;
    nv = (p0 + n - 1) / C - v0 + 1;
  }
  mbar_arrive_expect_tx(bar, static_cast<uint32_t>(n * tile_b + nv * vec_b));
  bulk_g2s(slot, static_cast<const unsigned char*>(H) + static_cast<size_t>(p0) * tile_b, n * tile_b, bar, pol);
  bulk_g2s(slot + npw * tile_b, static_cast<const unsigned char*>(V) + static_cast<size_t>(v0) * vec_b, nv * vec_b,
           bar, pol);
}

// Reduce-scatter NV per-lane partials over the G lanes of a group with xor
// butterflies: afterwards lane k holds the full sums of values
// [k*NV/G, (k+1)*NV/G) in v[0 .. NV/G).  log2(G) rounds, NV-NV/G shuffles.
template <int O, int N, int NV>
struct ReduceScatter {
  static __device__ __forceinline__ void run(float (&v)[NV], int k) {
    const bool hi = (k & O) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      const float a = v[i], b = v[i + N / 2];
      const float send = hi ? a : b;
      const float keep = hi ? b : a;
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    ReduceScatter<O / 2, N / 2, NV>::run(v, k);
  }
};
template <int N, int NV>
struct ReduceScatter<0, N, NV> {
  static __device__ __forceinline__ void run(float (&)[NV], int) {}
};

template <int G, int NV>
__device__ __forceinline__ void group_reduce_scatter(float (&v)[NV], int k) {
  static_assert(NV % G == 0, "values must split evenly over the group");
  ReduceScatter<G / 2, NV, NV>::run(v, k);
}

// Reduce-scatter NV values over a group of G lanes (NV <= G), then finish the
// sums: afterwards lane k holds the group-wide sum of value k / (G/NV).
// log2(NV) halving rounds (NV-1 shuffles) + log2(G/NV) single-value rounds —
// against NV*log2(G) shuffles for a butterfly of every value.  The results
// are then broadcast through shared memory (one store per value, one vector
// load per lane).
template <int G, int NV>
__device__ __forceinline__ float group_scatter_sum(float (&v)[NV], int k) {
  static_assert(NV <= G && G % NV == 0, "values must not outnumber the group");
  ReduceScatter<G / 2, NV, NV>::run(v, k);
  float s = v[0];
#pragma unroll
  for (int o = G / (2 * NV); o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Per-problem scalar blocks (bytes); the uplink block ends with a double
// buffer of 2 x 2*LB floats for the scatter-sum broadcast, the downlink one
// with 2 x 4 floats; +16 skews consecutive groups' blocks across shared-memory
// banks.  Used by the kernels and their launchers.
__host__ __device__ constexpr int ul_scal_bytes(int U, int LB = 2) {
  return U * 16 + (U / LB) * (LB * (LB - 1) / 2) * 16 + 16 * LB + 16;
}
__host__ __device__ constexpr int dl_scal_bytes(int U) { return U * 32 + 32 + 16; }

// Shared-memory layout of one CTA: [W staging slots][W*NPW scalar blocks][W mbarriers]
template <int SLOT_B, int SCAL_B, int NPW, int W>
struct CtaSmem {
  static constexpr int kScalOff = W * SLOT_B;
  static constexpr int kBarOff = kScalOff + W * NPW * SCAL_B;
  static constexpr int kBytes = kBarOff + W * 8;
};

// ===========================================================================
// Uplink, fp32 storage and arithmetic, on packed row PAIRS: every lane keeps
// its rows as float2 (row 2c, row 2c+1) planes of re and im, so each complex
// MAC over two rows is 2 FFMA2 (sm_100 packed fp32x2) and the rank-1
// coefficient dx is a broadcast operand.
// Coordinates are processed in blocks of LB (see "Coordinate blocks" above):
// one shuffle round reduces all LB dot products, then the block's
// lower-triangular Gram entries G_ab = h_a^H h_b (a > b) correct them exactly.
// Scalar block per problem: float4 mnx[U] = (m_j, n_j, Re x_j, Im x_j) and
// float4 gb[U/LB][LB(LB-1)/2] = (Re G, Im G, -Im G, Re G).
// ===========================================================================
template <int BC, int U, int G, int W, int MINB, int LB, bool XCHG = false, bool SIG = false>
__global__ void __launch_bounds__(32 * W, MINB)
    ul_reg_f32(const float2* __restrict__ H, const float2* __restrict__ Y, int P, int K, float kappa,
               float2* __restrict__ X, const XMap xm, float* __restrict__ sigma2 = nullptr, float gam = 0.f,
               float scale = 0.f, unsigned long long* __restrict__ status = nullptr) {
  static_assert(32 % G == 0 && BC % (2 * G) == 0 && U % LB == 0, "shape");
  static_assert(!SIG || ((U == 16 || U == 8) && G == U / 2 && BC % 16 == 0 && LB == 2 && !XCHG),
                "fused variance: U/2 lanes per problem hold rows 2k, 2k+1 of the U x U Gram");
  static_assert(!SIG || DCDG_SIG_CPAIRS || U == 16, "the scalar sweep operator is the U = 16 form");
  constexpr int NPW = 32 / G, R = BC / G, NP = R / 2;
  constexpr int T = LB * (LB - 1) / 2;  // Gram entries per block
  constexpr int TILE_B = BC * U * 8, Y_B = BC * 8, SLOT_B = Slot<TILE_B, Y_B, NPW>::kBytes;
  constexpr int SCAL_B = ul_scal_bytes(U, LB);
  using L = CtaSmem<SLOT_B, SCAL_B, NPW, W>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  float4* mnx = reinterpret_cast<float4*>(smem + L::kScalOff + (warp * NPW + g) * SCAL_B);
  float4* gb = mnx + U;
  float* dbuf = reinterpret_cast<float*>(gb + (U / LB) * T);  // 2 x 2*LB floats
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff) + warp;
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x * W;
  int set = blockIdx.x * W + warp;
  const uint64_t pol = l2_evict_first_policy();
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0 && set < nsets) issue_set(slot, bar, H, Y, set, P, NPW, TILE_B, Y_B, true, 1, pol);
  uint32_t phase = 0;
  const float2 z2 = make_float2(0.f, 0.f);
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    float2 hr[U][NP], hi[U][NP], rr[NP], ri[NP];
    {
      // one 16-B load per row pair, re-paired once into planar registers
      const float4* t4 = reinterpret_cast<const float4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const float4 v = t4[j * (BC / 2) + c * G + k];
          hr[j][c] = pair(v.x, v.z);
          hi[j][c] = pair(v.y, v.w);
        }
      const float4* y4 = reinterpret_cast<const float4*>(slot + NPW * TILE_B + g * Y_B);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = y4[c * G + k];
        rr[c] = pair(v.x, v.z);
        ri[c] = pair(v.y, v.w);
      }
    }
    if constexpr (!SIG) {  // the fused-variance kernel keeps the slot until its Gram image is read
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);
    }

    float emax = 0.f;
    // ---- per-problem scalars: ||h_j||^2 (detect.cpp:86-90) and block Grams,
    // each reduce-scattered over the group (lane k keeps a contiguous slice)
    {
      constexpr int NV = ((U + G - 1) / G) * G;  // padded to a multiple of the group
      float v[NV];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float2 e = fmul2(hr[j][0], hr[j][0]);
        e = ffma2(hi[j][0], hi[j][0], e);
#pragma unroll
        for (int c = 1; c < NP; ++c) e = ffma2(hi[j][c], hi[j][c], ffma2(hr[j][c], hr[j][c], e));
        v[j] = hsum(e);
      }
#pragma unroll
      for (int j = U; j < NV; ++j) v[j] = 0.f;
      group_reduce_scatter<G>(v, k);
      if constexpr (SIG) {  // the problem's largest column energy (scale of the split Gram)
#pragma unroll
        for (int i = 0; i < NV / G; ++i) emax = fmaxf(emax, v[i]);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
      }
#pragma unroll
      for (int i = 0; i < NV / G; ++i) {
        const int idx = k * (NV / G) + i;
        const float m = __fdividef(1.f, v[i] + kappa);       // m_j = 1/(||h_j||^2 + N0/Ex)
#if DCDG_UL_DIRECT_DX
        // c_j = n_j - 1 = -kappa m_j (n_j = m_j ||h_j||^2), x_j = 0
        if (idx < U) mnx[idx] = make_float4(m, -kappa * m, 0.f, 0.f);
#else
        if (idx < U) mnx[idx] = make_float4(m, m * v[i], 0.f, 0.f);  // n_j = m_j ||h_j||^2, x_j = 0
#endif
      }
    }
    {
      constexpr int NG0 = 2 * (U / LB) * T;                 // floats of the block Grams
      constexpr int NG = ((NG0 + G - 1) / G) * G;            // padded to a multiple of the group
      float v[NG];
#pragma unroll
      for (int e = NG0; e < NG; ++e) v[e] = 0.f;
#pragma unroll
      for (int q = 0; q < U / LB; ++q)
#pragma unroll
        for (int a = 1; a < LB; ++a)
#pragma unroll
          for (int b = 0; b < a; ++b) {  // G_ab = h_{qLB+a}^H h_{qLB+b}
            const int ja = q * LB + a, jb = q * LB + b, e = q * T + a * (a - 1) / 2 + b;
            float2 gr = z2, gi = z2;
#pragma unroll
            for (int c = 0; c < NP; ++c) {
              gr = ffma2(hi[ja][c], hi[jb][c], ffma2(hr[ja][c], hr[jb][c], gr));
              gi = ffma2(neg2(hi[ja][c]), hr[jb][c], ffma2(hr[ja][c], hi[jb][c], gi));
            }
            v[2 * e] = hsum(gr);
            v[2 * e + 1] = hsum(gi);
          }
      group_reduce_scatter<G>(v, k);
      float* gf = reinterpret_cast<float*>(gb);
#pragma unroll
      for (int i = 0; i < NG / G; ++i) {
        const int gi = k * (NG / G) + i, e = gi >> 1;
        if (gi >= NG0) continue;
        if (gi & 1) {  // stored as (Re G, Im G, -Im G, Re G)
          gf[e * 4 + 1] = v[i];
          gf[e * 4 + 2] = -v[i];
        } else {
          gf[e * 4 + 0] = v[i];
          gf[e * 4 + 3] = v[i];
        }
      }
    }
    __syncwarp();

    // ---- K sweeps over the users in ascending order, LB coordinates per round
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int q = 0; q < U / LB; ++q) {
        float2 d[LB];
#pragma unroll
        for (int a = 0; a < LB; ++a) {  // h_j^H r (cdotc, detect.cpp:100), all against the same r
          const int j = q * LB + a;
          float2 ar = z2, ai = z2;
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            ar = ffma2(hi[j][c], ri[c], ffma2(hr[j][c], rr[c], ar));
            ai = ffma2(neg2(hi[j][c]), rr[c], ffma2(hr[j][c], ri[c], ai));
          }
          d[a] = make_float2(hsum(ar), hsum(ai));
        }
        if constexpr (2 * LB <= G && G >= DCDG_SCATTER_MIN_G_UL) {
          // reduce-scatter + shared-memory broadcast (double-buffered per group)
          float v[2 * LB];
#pragma unroll
          for (int a = 0; a < LB; ++a) {
            v[2 * a] = d[a].x;
            v[2 * a + 1] = d[a].y;
          }
          const float sum = group_scatter_sum<G, 2 * LB>(v, k);
          float* db = dbuf + ((t * (U / LB) + q) & 1) * 2 * LB;  // alternates every block
          if (k % (G / (2 * LB)) == 0) db[k / (G / (2 * LB))] = sum;
          __syncwarp();
#pragma unroll
          for (int a = 0; a < LB; ++a) d[a] = reinterpret_cast<const float2*>(db)[a];
        } else {
          group_allreduce2<G>(d);
        }
        float2 dx[LB];
#pragma unroll
        for (int a = 0; a < LB; ++a) {
          const int j = q * LB + a;
          const float4 A = mnx[j];
          // h_j^H (r - sum_{b<a} dx_b h_b) = h_j^H r - sum_b dx_b G_ab
#pragma unroll
          for (int b = 0; b < a; ++b) {
            const float4 Gab = gb[q * T + a * (a - 1) / 2 + b];
            d[a] = ffma2(-dx[b].x, make_float2(Gab.x, Gab.y), d[a]);
            d[a] = ffma2(-dx[b].y, make_float2(Gab.z, Gab.w), d[a]);
          }
          // x_j' = m_j h_j^H r + n_j x_j ; dx = x_j' - x_j   (detect.cpp:100-103)
          const float2 xo = make_float2(A.z, A.w);
#if DCDG_UL_DIRECT_DX
          // dx = m_j h_j^H r + (n_j - 1) x_j: one FFMA2 after the reduction
          dx[a] = ffma2(A.x, d[a], fmul2(A.y, xo));
          const float2 xn = fadd2(xo, dx[a]);
#else
          const float2 xn = ffma2(A.x, d[a], fmul2(A.y, xo));
          dx[a] = fadd2(xn, neg2(xo));
#endif
          *reinterpret_cast<float2*>(&mnx[j].z) = xn;  // every lane of the group stores the same value
        }
        // r -= dx_j h_j for the block   (caxpy, detect.cpp:104)
#pragma unroll
        for (int a = 0; a < LB; ++a) {
          const int j = q * LB + a;
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            rr[c] = ffma2(dx[a].y, hi[j][c], ffma2(-dx[a].x, hr[j][c], rr[c]));
            ri[c] = ffma2(-dx[a].y, hr[j][c], ffma2(-dx[a].x, hi[j][c], ri[c]));
          }
        }
      }
    }
    __syncwarp();
    const int p = set * NPW + g;
    if (p < P) {
      // XCHG: straight into the owning GPU's exchange window (peer memory)
      float4* xo = XCHG ? reinterpret_cast<float4*>(xchg_x_dst(xm, p, static_cast<int>(xchg_epoch(xm) & 1)))
                        : reinterpret_cast<float4*>(X + static_cast<size_t>(p) * U);
#pragma unroll
      for (int i = k; i < U / 2; i += G) {
        const float4 u0 = mnx[2 * i], u1 = mnx[2 * i + 1];
        xo[i] = make_float4(u0.z, u0.w, u1.z, u1.w);
      }
    }
    if constexpr (SIG) {
      // ---- post_eq_variance (detect.cpp:112-130).  The Gram G = H^H H
      // (detect.cpp:21-28) of each problem of the set comes from the tensor
      // cores, read from the problem's tile still in the staging slot: fp32
      // entries scaled by a power of two (largest column energy -> ~1) and
      // split x = hi + lo into binary16, G = hi.hi + hi.lo + lo.hi with fp32
      // accumulation (mma.sync m16n8k16; each product of binary16 values is
      // exact in fp32, the dropped lo.lo term is ~2^-22 of |h|^2).  Fragment
      // k-order: k-step s takes complex rows 8s + 2t (k 2t, 2t+1) and 8s + 2t + 1
      // (k 2t+8, 2t+9), one 16-B load per user; W' = (im, -re) per complex gives
      // Im G.  A = I + (E_x/N0) G is written over the problem's consumed tile
      // as the column-pair image (apair_slot) the sweep operator reads.
      {
        const int mg = lane >> 2, mt = lane & 3;  // mma fragment coordinates
#pragma unroll
        for (int pl = 0; pl < NPW; ++pl) {
          const float em = __shfl_sync(0xffffffffu, emax, pl * G);
          // power-of-two scale: |h_ij|^2 <= em -> |h_ij sc| <= 1
          // sc = 2^-e and 1/sc^2 = 2^2e built from the exponent bits (ldexpf and
          // an IEEE division were 4% of the kernel's stall samples)
          const int e = em > 0.f ? max(-60, min(60, static_cast<int>(ceilf(0.5f * __log2f(em))))) : 0;
          const float sc = __int_as_float((127 - e) << 23);
          const float isc2 = __int_as_float((127 + 2 * e) << 23);
          const unsigned char* tb = slot + pl * TILE_B;
          float gr0[4] = {}, gr1[4] = {}, gi0[4] = {}, gi1[4] = {};
#pragma unroll
          for (int ks = 0; ks < BC / 8; ++ks) {
            const float4 u0 = *reinterpret_cast<const float4*>(tb + mg * (BC * 8) + (8 * ks + 2 * mt) * 8);
            const float2 x00 = fmul2(sc, make_float2(u0.x, u0.y)), x01 = fmul2(sc, make_float2(u0.z, u0.w));
            uint32_t ah[4], al[4];
            split_h2(x00, ah[0], al[0]);  // user mg,     row 8ks + 2mt
            split_h2(x01, ah[2], al[2]);  // user mg,     row 8ks + 2mt + 1
            if constexpr (U == 16) {
              const float4 u1 = *reinterpret_cast<const float4*>(tb + (mg + 8) * (BC * 8) + (8 * ks + 2 * mt) * 8);
              const float2 x10 = fmul2(sc, make_float2(u1.x, u1.y)), x11 = fmul2(sc, make_float2(u1.z, u1.w));
              split_h2(x10, ah[1], al[1]);  // user mg + 8, row 8ks + 2mt
              split_h2(x11, ah[3], al[3]);  // user mg + 8, row 8ks + 2mt + 1
            } else {  // U = 8: A rows 8-15 are zero
              ah[1] = ah[3] = al[1] = al[3] = 0u;
            }
            // B = W: n-tile 0 (users 0-7) = (a0, a2), n-tile 1 (users 8-15) = (a1, a3)
            mma_f16f32(gr0, ah, ah[0], ah[2]);
            mma_f16f32(gr0, ah, al[0], al[2]);
            mma_f16f32(gr0, al, ah[0], ah[2]);
            mma_f16f32(gi0, ah, wprime(ah[0]), wprime(ah[2]));
            mma_f16f32(gi0, ah, wprime(al[0]), wprime(al[2]));
            mma_f16f32(gi0, al, wprime(ah[0]), wprime(ah[2]));
            if constexpr (U == 16) {
              mma_f16f32(gr1, ah, ah[1], ah[3]);
              mma_f16f32(gr1, ah, al[1], al[3]);
              mma_f16f32(gr1, al, ah[1], ah[3]);
              mma_f16f32(gi1, ah, wprime(ah[1]), wprime(ah[3]));
              mma_f16f32(gi1, ah, wprime(al[1]), wprime(al[3]));
              mma_f16f32(gi1, al, wprime(ah[1]), wprime(ah[3]));
            }
          }
          __syncwarp();  // every lane's reads of this tile are done before its image overwrites it
          const float gs = gam * isc2;  // gam / sc^2, exact (power of two)
          float4* img = reinterpret_cast<float4*>(slot + pl * TILE_B);
          // C fragment: [0..1] row mg, cols 2mt, 2mt+1 of the n-tile; [2..3] row mg + 8
          img[apair_slot<U>(mg, mt)] = make_float4(fmaf(gs, gr0[0], mg == 2 * mt ? 1.f : 0.f),
                                                   fmaf(gs, gr0[1], mg == 2 * mt + 1 ? 1.f : 0.f), gs * gi0[0],
                                                   gs * gi0[1]);
          if constexpr (U == 16) {
            img[apair_slot<U>(mg, 4 + mt)] = make_float4(gs * gr1[0], gs * gr1[1], gs * gi1[0], gs * gi1[1]);
            img[apair_slot<U>(mg + 8, mt)] = make_float4(gs * gr0[2], gs * gr0[3], gs * gi0[2], gs * gi0[3]);
            img[apair_slot<U>(mg + 8, 4 + mt)] = make_float4(fmaf(gs, gr1[2], mg == 2 * mt ? 1.f : 0.f),
                                                             fmaf(gs, gr1[3], mg == 2 * mt + 1 ? 1.f : 0.f),
                                                             gs * gi1[2], gs * gi1[3]);
          }
        }
      }
      float* af = reinterpret_cast<float*>(slot + g * TILE_B);
      __syncwarp();
      // lane k takes rows 2k, 2k+1 of A as column pairs; then the slot is free
      // for the next set's copy
#if DCDG_SIG_COLS
      // lane k takes column pair k of every row (forward elimination)
      float2 Cr[U], Ci[U];
      {
        const float4* a4 = reinterpret_cast<const float4*>(af);
#pragma unroll
        for (int i = 0; i < U; ++i) {
          const float4 a = a4[apair_slot<U>(i, k)];
          Cr[i] = make_float2(a.x, a.y);
          Ci[i] = make_float2(a.z, a.w);
        }
      }
#elif DCDG_SIG_CPAIRS
      float2 R0r[U / 2], R0i[U / 2], R1r[U / 2], R1i[U / 2];
      const float4* a4 = reinterpret_cast<const float4*>(af);
#pragma unroll
      for (int jq = 0; jq < U / 2; ++jq) {
        const float4 a = a4[apair_slot<U>(2 * k, jq)], b = a4[apair_slot<U>(2 * k + 1, jq)];
        R0r[jq] = make_float2(a.x, a.y);
        R0i[jq] = make_float2(a.z, a.w);
        R1r[jq] = make_float2(b.x, b.y);
        R1i[jq] = make_float2(b.z, b.w);
      }
#else
      // scalar rows of G for the FFMA sweep operator (A = I + gam G formed inside)
      float ar0[U], ai0[U], ar1[U], ai1[U];
      const float4* a4 = reinterpret_cast<const float4*>(af);
#pragma unroll
      for (int jq = 0; jq < U / 2; ++jq) {
        const float4 a = a4[apair_slot<U>(2 * k, jq)], b = a4[apair_slot<U>(2 * k + 1, jq)];
        ar0[2 * jq] = a.x;
        ar0[2 * jq + 1] = a.y;
        ai0[2 * jq] = a.z;
        ai0[2 * jq + 1] = a.w;
        ar1[2 * jq] = b.x;
        ar1[2 * jq + 1] = b.y;
        ai1[2 * jq] = b.z;
        ai1[2 * jq + 1] = b.w;
      }
#endif
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);
      // the pivot rows go through the problem's scalar block (dead after the sweeps)
      bool singular = false;
#if DCDG_SIG_COLS
      const float tr = gram_trace_inverse_cols<U, DCDG_SIG_COLS_SCALED_FUSED != 0>(Cr, Ci, k, mnx, singular);
#elif DCDG_SIG_CPAIRS
      const float tr = DCDG_SIG_BLOCK2 ? gram_trace_inverse_cpairs2<U>(R0r, R0i, R1r, R1i, k, mnx, singular)
                                         : gram_trace_inverse_cpairs<U>(R0r, R0i, R1r, R1i, k, mnx, singular);
#else
      const float tr = gram_trace_inverse<U>(ar0, ai0, ar1, ai1, k, 0.f, mnx, singular, true);
#endif
      const unsigned sing = __ballot_sync(0xffffffffu, singular);
      if (p < P && k == 0) {
        sigma2[p] = scale * tr;
        if ((sing >> (G * g)) & ((1u << G) - 1u)) record_status(status, p, ST_SINGULAR, 0);
      }
    }
    __syncwarp();
  }
  if constexpr (XCHG) xchg_cta_done(xm);
}

// ===========================================================================
// Uplink, fp16 storage + half2 arithmetic (the paper's half-precision path).
// The fp16 channel tile and receive vector are stored row-pair planar
// ({re_2i, re_2i+1, im_2i, im_2i+1} per 8 bytes, see include/dcdg.h), so each
// lane loads its rows directly as planar half2 PAIRS (re_i, re_i+1), (im_i, im_i+1),
// so a complex MAC over two rows is 2 HFMA2 (4 FFMA per row in fp32).  Dot
// products accumulate in half2 and are reduced as one packed (re, im) half2
// per shuffle; the per-coordinate scalar update runs in fp32.
// ===========================================================================
template <int BC, int U, int G, int W, int MINB, bool XCHG = false>
__global__ void __launch_bounds__(32 * W, MINB)
    ul_reg_f16(const __half2* __restrict__ H, const __half2* __restrict__ Y, int P, int K, float kappa,
               __half2* __restrict__ X, const XMap xm) {
  static_assert(32 % G == 0 && BC % (4 * G) == 0 && U % 4 == 0 && U % G == 0, "shape");
  constexpr int NPW = 32 / G, R = BC / G, CH = R / 4, NP = R / 2;
  constexpr int TILE_B = BC * U * 4, Y_B = BC * 4, SLOT_B = Slot<TILE_B, Y_B, NPW>::kBytes;
  constexpr int SCAL_B = ul_scal_bytes(U);
  using L = CtaSmem<SLOT_B, SCAL_B, NPW, W>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  float4* mng = reinterpret_cast<float4*>(smem + L::kScalOff + (warp * NPW + g) * SCAL_B);
  float2* xs = reinterpret_cast<float2*>(mng + U);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff) + warp;
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x * W;
  int set = blockIdx.x * W + warp;
  const uint64_t pol = l2_evict_first_policy();
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0 && set < nsets) issue_set(slot, bar, H, Y, set, P, NPW, TILE_B, Y_B, true, 1, pol);
  uint32_t phase = 0;
  const __half2 z2 = __float2half2_rn(0.f);
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    __half2 hre[U][NP], him[U][NP], rre[NP], rim[NP];
    {
      // fp16 tiles are row-pair planar: {re_2i, re_2i+1, im_2i, im_2i+1}
      const uint4* t4 = reinterpret_cast<const uint4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 v = t4[j * (BC / 4) + c * G + k];
          hre[j][2 * c] = u32_as_h2(v.x);
          him[j][2 * c] = u32_as_h2(v.y);
          hre[j][2 * c + 1] = u32_as_h2(v.z);
          him[j][2 * c + 1] = u32_as_h2(v.w);
        }
      const uint4* y4 = reinterpret_cast<const uint4*>(slot + NPW * TILE_B + g * Y_B);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const uint4 v = y4[c * G + k];
        rre[2 * c] = u32_as_h2(v.x);
        rim[2 * c] = u32_as_h2(v.y);
        rre[2 * c + 1] = u32_as_h2(v.z);
        rim[2 * c + 1] = u32_as_h2(v.w);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);

    {
      float v[U];  // ||h_j||^2 (half2 partials, fp32 group sums)
#pragma unroll
      for (int j = 0; j < U; ++j) {
        __half2 acc = __hmul2(hre[j][0], hre[j][0]);
        acc = __hfma2(him[j][0], him[j][0], acc);
#pragma unroll
        for (int q = 1; q < NP; ++q) {
          acc = __hfma2(hre[j][q], hre[j][q], acc);
          acc = __hfma2(him[j][q], him[j][q], acc);
        }
        const float2 f = __half22float2(acc);
        v[j] = f.x + f.y;
      }
      group_reduce_scatter<G>(v, k);
#pragma unroll
      for (int i = 0; i < U / G; ++i) {
        const float m = __fdividef(1.f, v[i] + kappa);
        const int idx = k * (U / G) + i;
        reinterpret_cast<float2*>(mng)[2 * idx] = make_float2(m, m * v[i]);
        xs[idx] = make_float2(0.f, 0.f);
      }
    }
    {
      float v[U];  // pair Grams h_{2i+1}^H h_{2i}
#pragma unroll
      for (int i = 0; i < U / 2; ++i) {
        __half2 gr = z2, gi = z2;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          gr = __hfma2(hre[2 * i + 1][q], hre[2 * i][q], __hfma2(him[2 * i + 1][q], him[2 * i][q], gr));
          gi = __hfma2(hre[2 * i + 1][q], him[2 * i][q], __hfma2(__hneg2(him[2 * i + 1][q]), hre[2 * i][q], gi));
        }
        const float2 fr = __half22float2(gr), fi = __half22float2(gi);
        v[2 * i] = fr.x + fr.y;
        v[2 * i + 1] = fi.x + fi.y;
      }
      group_reduce_scatter<G>(v, k);
      float* mf = reinterpret_cast<float*>(mng);
#pragma unroll
      for (int i = 0; i < U / G; ++i) {
        const int gi = k * (U / G) + i;
        // mng[2i+1].zw = (Re G, Im G), mng[2i].zw = (-Im G, Re G) of G = h_{2i+1}^H h_{2i}
        mf[((gi >> 1) * 2 + 1) * 4 + 2 + (gi & 1)] = v[i];
        mf[((gi >> 1) * 2) * 4 + 3 - (gi & 1)] = (gi & 1) ? -v[i] : v[i];
      }
    }
    __syncwarp();

    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp) {
        const int j0 = 2 * jp, j1 = 2 * jp + 1;
        const float4 s0 = mng[j0], s1 = mng[j1];
        const float2 x0 = xs[j0], x1 = xs[j1];
        // folded accumulator chains: re = sum hr*r_re + hi*r_im, im = sum hr*r_im - hi*r_re
        __half2 re0 = z2, im0 = z2, re1 = z2, im1 = z2;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          re0 = __hfma2(him[j0][q], rim[q], __hfma2(hre[j0][q], rre[q], re0));
          im0 = __hfma2(__hneg2(him[j0][q]), rre[q], __hfma2(hre[j0][q], rim[q], im0));
          re1 = __hfma2(him[j1][q], rim[q], __hfma2(hre[j1][q], rre[q], re1));
          im1 = __hfma2(__hneg2(him[j1][q]), rre[q], __hfma2(hre[j1][q], rim[q], im1));
        }
        __half2 d0 = __hadd2(__lows2half2(re0, im0), __highs2half2(re0, im0));
        __half2 d1 = __hadd2(__lows2half2(re1, im1), __highs2half2(re1, im1));
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          d0 = __hadd2(d0, __shfl_xor_sync(0xffffffffu, d0, o));
          d1 = __hadd2(d1, __shfl_xor_sync(0xffffffffu, d1, o));
        }
        const float2 f0 = __half22float2(d0);
        float2 f1 = __half22float2(d1);
        // scalar update in packed fp32x2 (detect.cpp:100-103), pair-Gram correction of the second dot
        const float2 n0 = ffma2(s0.x, f0, fmul2(s0.y, x0));
        const float2 dx0 = fadd2(n0, neg2(x0));
        f1 = ffma2(-dx0.x, make_float2(s1.z, s1.w), f1);
        f1 = ffma2(-dx0.y, make_float2(s0.z, s0.w), f1);
        const float2 n1 = ffma2(s1.x, f1, fmul2(s1.y, x1));
        const float2 dx1 = fadd2(n1, neg2(x1));
        xs[j0] = n0;
        xs[j1] = n1;
        // one packed conversion per coordinate; the broadcast halves and signs
        // are HFMA2 operand modifiers
        const __half2 h0 = __float22half2_rn(dx0), h1 = __float22half2_rn(dx1);
        const __half2 r0 = __low2half2(h0), i0 = __high2half2(h0);
        const __half2 r1 = __low2half2(h1), i1 = __high2half2(h1);
#pragma unroll
        for (int q = 0; q < NP; ++q) {  // r -= dx_j h_j   (caxpy, detect.cpp:104)
          rre[q] = __hfma2(__hneg2(r0), hre[j0][q], __hfma2(i0, him[j0][q], rre[q]));
          rim[q] = __hfma2(__hneg2(r0), him[j0][q], __hfma2(__hneg2(i0), hre[j0][q], rim[q]));
          rre[q] = __hfma2(__hneg2(r1), hre[j1][q], __hfma2(i1, him[j1][q], rre[q]));
          rim[q] = __hfma2(__hneg2(r1), him[j1][q], __hfma2(__hneg2(i1), hre[j1][q], rim[q]));
        }
      }
    }
    __syncwarp();
    const int p = set * NPW + g;
    if (p < P) {
      uint4* xo = XCHG ? reinterpret_cast<uint4*>(xchg_x_dst(xm, p, static_cast<int>(xchg_epoch(xm) & 1)))
                       : reinterpret_cast<uint4*>(X + static_cast<size_t>(p) * U);
#pragma unroll
      for (int i = k; i < U / 4; i += G) {
        uint4 w;
        w.x = h2_as_u32(__floats2half2_rn(xs[4 * i].x, xs[4 * i].y));
        w.y = h2_as_u32(__floats2half2_rn(xs[4 * i + 1].x, xs[4 * i + 1].y));
        w.z = h2_as_u32(__floats2half2_rn(xs[4 * i + 2].x, xs[4 * i + 2].y));
        w.w = h2_as_u32(__floats2half2_rn(xs[4 * i + 3].x, xs[4 * i + 3].y));
        xo[i] = w;
      }
    }
    __syncwarp();
  }
  if constexpr (XCHG) xchg_cta_done(xm);
}

// ===========================================================================
// Downlink, fp32, packed row pairs (see ul_reg_f32).  The dual rows h_u are
// the uplink columns (conj_rows, precode.cpp:19-27).  The reference
// normalises them (p_u = 1/||h_u||, precode.cpp:69-87); here they stay raw and
// the normalisation moves into the scalars: x -= q_u (h_u^H x - s_u) h_u with
// q_u = 1/||h_u||^2 is the normalised update exactly.  Scalar block per problem:
// float4 ss[U] = (Re q_u s_u, Im q_u s_u, q_u, -);
// float4 gp[U/2] = (Re G, Im G, -Im G, Re G), G = h_{2i+1}^H h_{2i};
// float2 sraw[U] (the received symbols).
// ===========================================================================
template <int BC, int U, int G, int W, int MINB, bool GAIN>
__global__ void __launch_bounds__(32 * W, MINB)
    dl_reg_f32(const float2* __restrict__ H, const float2* __restrict__ Sy, int P, int C, int K, float rho_c,
               float2* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status) {
  static_assert(32 % G == 0 && BC % (2 * G) == 0 && U % 2 == 0 && (2 * U) % G == 0, "shape");
  constexpr int NPW = 32 / G, R = BC / G, NP = R / 2;
  constexpr int TILE_B = BC * U * 8, S_B = U * 8, SLOT_B = Slot<TILE_B, S_B, NPW>::kBytes;
  constexpr int SCAL_B = dl_scal_bytes(U);
  using L = CtaSmem<SLOT_B, SCAL_B, NPW, W>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  float4* ss = reinterpret_cast<float4*>(smem + L::kScalOff + (warp * NPW + g) * SCAL_B);
  float4* gp = ss + U;
  float2* sraw = reinterpret_cast<float2*>(gp + U / 2);
  float* dbuf = reinterpret_cast<float*>(sraw + U);  // 2 x 4 floats
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff) + warp;
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x * W;
  int set = blockIdx.x * W + warp;
  const uint64_t pol = l2_evict_first_policy();
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0 && set < nsets) issue_set(slot, bar, H, Sy, set, P, NPW, TILE_B, S_B, false, C, pol);
  uint32_t phase = 0;
  const float2 z2 = make_float2(0.f, 0.f);
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const int p = set * NPW + g;
    float2 hr[U][NP], hi[U][NP];
    {
      const float4* t4 = reinterpret_cast<const float4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const float4 v = t4[j * (BC / 2) + c * G + k];
          hr[j][c] = pair(v.x, v.z);
          hi[j][c] = pair(v.y, v.w);
        }
      const int sidx = min(p, P - 1) / C - (set * NPW) / C;
      const float4* s4 = reinterpret_cast<const float4*>(slot + NPW * TILE_B + sidx * S_B);
      float4* d4 = reinterpret_cast<float4*>(sraw);
#pragma unroll
      for (int i = k; i < U / 2; i += G) d4[i] = s4[i];
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Sy, set + nw, P, NPW, TILE_B, S_B, false, C, pol);

    // ---- row norms and raw pair Grams, reduce-scattered over the group
    constexpr int PER = 2 * U / G;
    float vv[2 * U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      float2 e = fmul2(hr[j][0], hr[j][0]);
      e = ffma2(hi[j][0], hi[j][0], e);
#pragma unroll
      for (int c = 1; c < NP; ++c) e = ffma2(hi[j][c], hi[j][c], ffma2(hr[j][c], hr[j][c], e));
      vv[j] = hsum(e);
    }
#pragma unroll
    for (int i = 0; i < U / 2; ++i) {
      float2 gr = z2, gi = z2;
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        gr = ffma2(hi[2 * i + 1][c], hi[2 * i][c], ffma2(hr[2 * i + 1][c], hr[2 * i][c], gr));
        gi = ffma2(neg2(hi[2 * i + 1][c]), hr[2 * i][c], ffma2(hr[2 * i + 1][c], hi[2 * i][c], gi));
      }
      vv[U + 2 * i] = hsum(gr);
      vv[U + 2 * i + 1] = hsum(gi);
    }
    group_reduce_scatter<G>(vv, k);
    int zero_user = -1;
    float* sf = reinterpret_cast<float*>(ss);
    float* gf = reinterpret_cast<float*>(gp);
    // The rows stay unnormalised: with q_u = 1/||h_u||^2 the normalised update
    // (precode.cpp:69-94) x -= (h~_u^H x - s~_u) h~_u is x -= q_u (h_u^H x - s_u) h_u,
    // so the scalar block holds (q_u s_u, q_u) and the raw pair Gram.
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int idx = k * PER + i;
      if (idx < U) {
        if (vv[i] == 0.f && zero_user < 0) zero_user = idx;
        const float q = __frcp_rn(vv[i]);
        const float2 sv = sraw[idx];
        sf[idx * 4 + 0] = q * sv.x;
        sf[idx * 4 + 1] = q * sv.y;
        sf[idx * 4 + 2] = q;
      } else {
        const int gi = idx - U, pr = gi >> 1;
        if (gi & 1) {
          gf[pr * 4 + 1] = vv[i];
          gf[pr * 4 + 2] = -vv[i];
        } else {
          gf[pr * 4 + 0] = vv[i];
          gf[pr * 4 + 3] = vv[i];
        }
      }
    }
    __syncwarp();

    float2 vr[NP], vi[NP];  // GAIN: v = H_c s = sum_u s_u h_u (the effective-gain share's left vector)
#if DCDG_DL_GAIN_EARLY == 1
    // accumulated before the sweeps, independent of their dependency chain
    if (GAIN) {
#pragma unroll
      for (int c = 0; c < NP; ++c) vr[c] = vi[c] = z2;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const float2 sj = sraw[j];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          vr[c] = ffma2(-sj.y, hi[j][c], ffma2(sj.x, hr[j][c], vr[c]));
          vi[c] = ffma2(sj.y, hr[j][c], ffma2(sj.x, hi[j][c], vi[c]));
        }
      }
    }
#endif
    float2 xr[NP], xi[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) xr[c] = xi[c] = z2;
#if DCDG_DL_GAIN_EARLY == 2
    if (GAIN) {
#pragma unroll
      for (int c = 0; c < NP; ++c) vr[c] = vi[c] = z2;
    }
#endif
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp) {
        const int j0 = 2 * jp, j1 = 2 * jp + 1;
        const float4 S0 = ss[j0], S1 = ss[j1], GG = gp[jp];
        float2 a0 = z2, c0 = z2, a1 = z2, c1 = z2;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          a0 = ffma2(hi[j0][c], xi[c], ffma2(hr[j0][c], xr[c], a0));
          c0 = ffma2(neg2(hi[j0][c]), xr[c], ffma2(hr[j0][c], xi[c], c0));
          a1 = ffma2(hi[j1][c], xi[c], ffma2(hr[j1][c], xr[c], a1));
          c1 = ffma2(neg2(hi[j1][c]), xr[c], ffma2(hr[j1][c], xi[c], c1));
        }
#if DCDG_DL_GAIN_EARLY == 2
        if (GAIN && t == K - 1) {
          const float4 s01 = reinterpret_cast<const float4*>(sraw)[jp];
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            vr[c] = ffma2(-s01.y, hi[j0][c], ffma2(s01.x, hr[j0][c], vr[c]));
            vi[c] = ffma2(s01.y, hr[j0][c], ffma2(s01.x, hi[j0][c], vi[c]));
            vr[c] = ffma2(-s01.w, hi[j1][c], ffma2(s01.z, hr[j1][c], vr[c]));
            vi[c] = ffma2(s01.w, hr[j1][c], ffma2(s01.z, hi[j1][c], vi[c]));
          }
        }
#endif
        float2 d0 = make_float2(hsum(a0), hsum(c0));
        float2 d1 = make_float2(hsum(a1), hsum(c1));
        if constexpr (4 <= G && G >= DCDG_SCATTER_MIN_G_DL) {
          float v[4] = {d0.x, d0.y, d1.x, d1.y};
          const float sum = group_scatter_sum<G, 4>(v, k);
          float* db = dbuf + ((t * (U / 2) + jp) & 1) * 4;
          if (k % (G / 4) == 0) db[k / (G / 4)] = sum;
          __syncwarp();
          const float4 dd = *reinterpret_cast<const float4*>(db);
          d0 = make_float2(dd.x, dd.y);
          d1 = make_float2(dd.z, dd.w);
        } else {
          float2 dd[2] = {d0, d1};
          group_allreduce2<G>(dd);
          d0 = dd[0];
          d1 = dd[1];
        }
        // r_u = q_u (h_u^H x - s_u) ; x -= r_u h_u   (precode.cpp:89-94 on unnormalised rows)
        const float2 r0 = ffma2(S0.z, d0, make_float2(-S0.x, -S0.y));
        d1 = ffma2(-r0.x, make_float2(GG.x, GG.y), d1);  // h_1^H (x - r_0 h_0) = d_1 - r_0 G_10
        d1 = ffma2(-r0.y, make_float2(GG.z, GG.w), d1);
        const float2 r1 = ffma2(S1.z, d1, make_float2(-S1.x, -S1.y));
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          xr[c] = ffma2(r0.y, hi[j0][c], ffma2(-r0.x, hr[j0][c], xr[c]));
          xi[c] = ffma2(-r0.y, hr[j0][c], ffma2(-r0.x, hi[j0][c], xi[c]));
          xr[c] = ffma2(r1.y, hi[j1][c], ffma2(-r1.x, hr[j1][c], xr[c]));
          xi[c] = ffma2(-r1.y, hr[j1][c], ffma2(-r1.x, hi[j1][c], xi[c]));
        }
      }
    }
    // power_scale to rho_c = rho / sqrt(C)   (precode.cpp:101-111,155); rho_c == 0: raw beamformer
    float2 e2 = fmul2(xr[0], xr[0]);
    e2 = ffma2(xi[0], xi[0], e2);
#pragma unroll
    for (int c = 1; c < NP; ++c) e2 = ffma2(xi[c], xi[c], ffma2(xr[c], xr[c], e2));
    const float e = gsum<G>(hsum(e2));
    const float gsc = rho_c > 0.f ? rho_c / __fsqrt_rn(e) : 1.f;
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      xr[c] = fmul2(gsc, xr[c]);
      xi[c] = fmul2(gsc, xi[c]);
    }
    // gain share Re(s^H H_dl,c x_c) = Re(v^H x_c), v = H_c s = sum_u s_u h_u
    float gq = 0.f;
    if (GAIN) {
#if DCDG_DL_GAIN_EARLY == 0
#pragma unroll
      for (int c = 0; c < NP; ++c) vr[c] = vi[c] = z2;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const float2 sj = sraw[j];
        const float cr = sj.x, ci = sj.y;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          vr[c] = ffma2(-ci, hi[j][c], ffma2(cr, hr[j][c], vr[c]));
          vi[c] = ffma2(ci, hr[j][c], ffma2(cr, hi[j][c], vi[c]));
        }
      }
#endif
      float2 q2 = fmul2(vr[0], xr[0]);
      q2 = ffma2(vi[0], xi[0], q2);
#pragma unroll
      for (int c = 1; c < NP; ++c) q2 = ffma2(vi[c], xi[c], ffma2(vr[c], xr[c], q2));
      gq = gsum<G>(hsum(q2));
    }
    if (p < P) {
      if (zero_user >= 0) record_status(status, p, ST_ZERO_ROW, zero_user);
      if (k == 0) {
        if (e == 0.f && rho_c > 0.f) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
        if (GAIN) gain_part[p] = gq;
      }
      float4* x4 = reinterpret_cast<float4*>(X + static_cast<size_t>(p) * BC);
#pragma unroll
      for (int c = 0; c < NP; ++c) x4[c * G + k] = make_float4(xr[c].x, xi[c].x, xr[c].y, xi[c].y);
    }
    __syncwarp();
  }
}
// ===========================================================================
// Downlink, fp16 storage + half2 arithmetic.
// ===========================================================================
template <int BC, int U, int G, int W, int MINB, bool GAIN>
__global__ void __launch_bounds__(32 * W, MINB)
    dl_reg_f16(const __half2* __restrict__ H, const __half2* __restrict__ Sy, int P, int C, int K, float rho_c,
               __half2* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status) {
  static_assert(32 % G == 0 && BC % (4 * G) == 0 && U % 4 == 0 && (2 * U) % G == 0, "shape");
  constexpr int NPW = 32 / G, R = BC / G, CH = R / 4, NP = R / 2;
  constexpr int TILE_B = BC * U * 4, S_B = U * 4, SLOT_B = Slot<TILE_B, S_B, NPW>::kBytes;
  constexpr int SCAL_B = dl_scal_bytes(U);
  using L = CtaSmem<SLOT_B, SCAL_B, NPW, W>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  float4* sg = reinterpret_cast<float4*>(smem + L::kScalOff + (warp * NPW + g) * SCAL_B);
  float2* sraw = reinterpret_cast<float2*>(sg + U);
  float* pn = reinterpret_cast<float*>(sraw + U);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff) + warp;
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x * W;
  int set = blockIdx.x * W + warp;
  const uint64_t pol = l2_evict_first_policy();
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0 && set < nsets) issue_set(slot, bar, H, Sy, set, P, NPW, TILE_B, S_B, false, C, pol);
  uint32_t phase = 0;
  const __half2 z2 = __float2half2_rn(0.f);
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const int p = set * NPW + g;
    __half2 hre[U][NP], him[U][NP];
    {
      // fp16 tiles are row-pair planar: {re_2i, re_2i+1, im_2i, im_2i+1}
      const uint4* t4 = reinterpret_cast<const uint4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 v = t4[j * (BC / 4) + c * G + k];
          hre[j][2 * c] = u32_as_h2(v.x);
          him[j][2 * c] = u32_as_h2(v.y);
          hre[j][2 * c + 1] = u32_as_h2(v.z);
          him[j][2 * c + 1] = u32_as_h2(v.w);
        }
      const int sidx = min(p, P - 1) / C - (set * NPW) / C;
      const __half2* s2 = reinterpret_cast<const __half2*>(slot + NPW * TILE_B + sidx * S_B);
#pragma unroll
      for (int i = k; i < U; i += G) sraw[i] = __half22float2(s2[i]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Sy, set + nw, P, NPW, TILE_B, S_B, false, C, pol);

    __half2 vre[NP], vim[NP];
    if (GAIN) {
#pragma unroll
      for (int q = 0; q < NP; ++q) vre[q] = vim[q] = z2;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const float2 sj = sraw[j];
        const __half2 s_r = __float2half2_rn(sj.x), s_i = __float2half2_rn(sj.y), n_i = __float2half2_rn(-sj.y);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          vre[q] = __hfma2(s_r, hre[j][q], __hfma2(n_i, him[j][q], vre[q]));
          vim[q] = __hfma2(s_r, him[j][q], __hfma2(s_i, hre[j][q], vim[q]));
        }
      }
    }
    constexpr int PER = 2 * U / G;
    float vv[2 * U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      __half2 acc = __hmul2(hre[j][0], hre[j][0]);
      acc = __hfma2(him[j][0], him[j][0], acc);
#pragma unroll
      for (int q = 1; q < NP; ++q) {
        acc = __hfma2(hre[j][q], hre[j][q], acc);
        acc = __hfma2(him[j][q], him[j][q], acc);
      }
      const float2 f = __half22float2(acc);
      vv[j] = f.x + f.y;
    }
#pragma unroll
    for (int i = 0; i < U / 2; ++i) {
      __half2 gr = z2, gi = z2;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        gr = __hfma2(hre[2 * i + 1][q], hre[2 * i][q], __hfma2(him[2 * i + 1][q], him[2 * i][q], gr));
        gi = __hfma2(hre[2 * i + 1][q], him[2 * i][q], __hfma2(__hneg2(him[2 * i + 1][q]), hre[2 * i][q], gi));
      }
      const float2 fr = __half22float2(gr), fi = __half22float2(gi);
      vv[U + 2 * i] = fr.x + fr.y;
      vv[U + 2 * i + 1] = fi.x + fi.y;
    }
    group_reduce_scatter<G>(vv, k);
    int zero_user = -1;
    float* sgf = reinterpret_cast<float*>(sg);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int idx = k * PER + i;
      if (idx < U) {  // unnormalised rows (see dl_reg_f32): (q_u s_u) and q_u = 1/||h_u||^2
        if (vv[i] == 0.f && zero_user < 0) zero_user = idx;
        const float q = __frcp_rn(vv[i]);
        const float2 sv = sraw[idx];
        pn[idx] = q;
        sgf[idx * 4] = q * sv.x;
        sgf[idx * 4 + 1] = q * sv.y;
      } else {
        const int gi = idx - U;
        const int a = (gi >> 1) * 2 + 1;
        // sg[2i+1].zw = (Re G, Im G), sg[2i].zw = (-Im G, Re G), raw pair Gram
        sgf[a * 4 + 2 + (gi & 1)] = vv[i];
        sgf[(a - 1) * 4 + 3 - (gi & 1)] = (gi & 1) ? -vv[i] : vv[i];
      }
    }
    __syncwarp();

    __half2 xre[NP], xim[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) xre[q] = xim[q] = z2;
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp) {
        const int j0 = 2 * jp, j1 = 2 * jp + 1;
        const float4 s0 = sg[j0], s1 = sg[j1];
        // folded accumulator chains: re = sum hr*r_re + hi*r_im, im = sum hr*r_im - hi*r_re
        __half2 re0 = z2, im0 = z2, re1 = z2, im1 = z2;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          re0 = __hfma2(him[j0][q], xim[q], __hfma2(hre[j0][q], xre[q], re0));
          im0 = __hfma2(__hneg2(him[j0][q]), xre[q], __hfma2(hre[j0][q], xim[q], im0));
          re1 = __hfma2(him[j1][q], xim[q], __hfma2(hre[j1][q], xre[q], re1));
          im1 = __hfma2(__hneg2(him[j1][q]), xre[q], __hfma2(hre[j1][q], xim[q], im1));
        }
        __half2 d0 = __hadd2(__lows2half2(re0, im0), __highs2half2(re0, im0));
        __half2 d1 = __hadd2(__lows2half2(re1, im1), __highs2half2(re1, im1));
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          d0 = __hadd2(d0, __shfl_xor_sync(0xffffffffu, d0, o));
          d1 = __hadd2(d1, __shfl_xor_sync(0xffffffffu, d1, o));
        }
        const float2 f0 = __half22float2(d0);
        float2 f1 = __half22float2(d1);
        // r_u = q_u (h_u^H x - s_u) (precode.cpp:89-94 on raw rows) in packed fp32x2, pair-Gram correction
        const float2 qq = *reinterpret_cast<const float2*>(pn + j0);
        const float2 q0 = ffma2(qq.x, f0, make_float2(-s0.x, -s0.y));
        f1 = ffma2(-q0.x, make_float2(s1.z, s1.w), f1);
        f1 = ffma2(-q0.y, make_float2(s0.z, s0.w), f1);
        const float2 q1 = ffma2(qq.y, f1, make_float2(-s1.x, -s1.y));
        const __half2 h0 = __float22half2_rn(q0), h1 = __float22half2_rn(q1);
        const __half2 r0 = __low2half2(h0), i0 = __high2half2(h0);
        const __half2 r1 = __low2half2(h1), i1 = __high2half2(h1);
#pragma unroll
        for (int q = 0; q < NP; ++q) {  // x -= r_u h_u
          xre[q] = __hfma2(__hneg2(r0), hre[j0][q], __hfma2(i0, him[j0][q], xre[q]));
          xim[q] = __hfma2(__hneg2(r0), him[j0][q], __hfma2(__hneg2(i0), hre[j0][q], xim[q]));
          xre[q] = __hfma2(__hneg2(r1), hre[j1][q], __hfma2(i1, him[j1][q], xre[q]));
          xim[q] = __hfma2(__hneg2(r1), him[j1][q], __hfma2(__hneg2(i1), hre[j1][q], xim[q]));
        }
      }
    }
    float e;
    {
      __half2 acc = __hmul2(xre[0], xre[0]);
      acc = __hfma2(xim[0], xim[0], acc);
#pragma unroll
      for (int q = 1; q < NP; ++q) {
        acc = __hfma2(xre[q], xre[q], acc);
        acc = __hfma2(xim[q], xim[q], acc);
      }
      const float2 f = __half22float2(acc);
      e = gsum<G>(f.x + f.y);
    }
    const float gsc = rho_c > 0.f ? rho_c / __fsqrt_rn(e) : 1.f;
    const __half2 g2 = __float2half2_rn(gsc);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      xre[q] = __hmul2(g2, xre[q]);
      xim[q] = __hmul2(g2, xim[q]);
    }
    float gq = 0.f;
    if (GAIN) {
      __half2 acc = __hmul2(vre[0], xre[0]);
      acc = __hfma2(vim[0], xim[0], acc);
#pragma unroll
      for (int q = 1; q < NP; ++q) {
        acc = __hfma2(vre[q], xre[q], acc);
        acc = __hfma2(vim[q], xim[q], acc);
      }
      const float2 f = __half22float2(acc);
      gq = gsum<G>(f.x + f.y);
    }
    if (p < P) {
      if (zero_user >= 0) record_status(status, p, ST_ZERO_ROW, zero_user);
      if (k == 0) {
        if (e == 0.f && rho_c > 0.f) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
        if (GAIN) gain_part[p] = gq;
      }
      uint4* x4 = reinterpret_cast<uint4*>(X + static_cast<size_t>(p) * BC);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        uint4 v;
        v.x = h2_as_u32(__lows2half2(xre[2 * c], xim[2 * c]));
        v.y = h2_as_u32(__highs2half2(xre[2 * c], xim[2 * c]));
        v.z = h2_as_u32(__lows2half2(xre[2 * c + 1], xim[2 * c + 1]));
        v.w = h2_as_u32(__highs2half2(xre[2 * c + 1], xim[2 * c + 1]));
        x4[c * G + k] = v;
      }
    }
    __syncwarp();
  }
}

}  // namespace dcdg
