// Split-tile CD kernels for sm_100a: part of each channel tile in registers,
// the rest in per-warp shared memory, so that more problems are in flight per
// SM than the register file alone allows.
//
// Why
//   A register-resident tile needs B_c*U/G complex per lane, so tiles beyond
//   32x16 force wide groups (G = 16 or 32 lanes per problem) or several warps
//   per problem (dcdg_mw_kernels.cuh).  Wide groups pay a 4-5 level shuffle
//   butterfly per coordinate block against little FMA work per lane, and the
//   multi-warp kernels a CTA barrier per block.  Keeping only the first JR
//   columns in registers and the other U - JR in a private shared-memory region
//   of the warp (row-pair planar, one LDS.128 per row pair and use) lets a
//   group of half the width own the problem: one butterfly level less, twice
//   the FMA work per reduction.  Measured on B200 (scripts/lab/lab_split2.cu,
//   profiles/lab/README.md): 32x32 36.6 -> 47.9% of HBM, 64x32 34.7 -> 44.2%,
//   128x32 27.8 -> 44.8%, 128x16 48.7 -> 58.1%, 256x16 43.3 -> 60.9%.  At the
//   32x16 target the register kernel (G = 8) stays faster.
//
// Staging
//   No shared-memory staging ring: each warp asks L2 to prefetch its next
//   set (cp.async.bulk.prefetch.L2, one instruction per contiguous range) one
//   set ahead, and loads the current set straight from L2 with 16-byte
//   non-allocating LDGs: register columns land in their final registers,
//   shared-memory columns are re-paired to the planar layout and stored.
//
// The arithmetic is that of ul_reg_f32 / dl_reg_f32 (coordinate pairs with the
// pair-Gram correction, FFMA2 on planar row pairs); only where a column comes
// from differs.
//
// Reference algorithms (paths relative to /root/reference/proj):
//   uplink   Alg. 1 = cd_detect                src/detect.cpp:67-110
//   downlink Alg. 2 = cd_precode + power_scale src/precode.cpp:52-111
//            + the cluster's effective-gain share, assemble_blocks src/precode.cpp:115-132
#pragma once

#include "dcdg_reg_kernels.cuh"

namespace dcdg {

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// 16-byte global load that does not allocate in L1 (the data is used once).
__device__ __forceinline__ float4 ldg_na(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// Shared memory of one single-warp CTA: [NPW][JS][NP][G] float4 column chunks,
// then NPW scalar blocks.
__host__ __device__ constexpr int split_cols_bytes(int BC, int U, int JR, int G) {
  return (32 / G) * (U - JR) * (BC / 2) * 16;
}

// One column's row pairs of this lane, from registers (j < JR) or from the
// warp's shared-memory region (planar float4 = (re_2i, re_2i+1, im_2i, im_2i+1)).
template <int JR, int NP, int G>
struct SplitCols {
  static __device__ __forceinline__ void get(int j, const float2 (&hr)[JR > 0 ? JR : 1][NP],
                                             const float2 (&hi)[JR > 0 ? JR : 1][NP], const float4* hs, int k,
                                             float2 (&cr)[NP], float2 (&ci)[NP]) {
    if (j < JR) {
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        cr[c] = hr[j < JR ? j : 0][c];
        ci[c] = hi[j < JR ? j : 0][c];
      }
    } else {
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = hs[((j - JR) * NP + c) * G + k];
        cr[c] = make_float2(v.x, v.y);
        ci[c] = make_float2(v.z, v.w);
      }
    }
  }
};

// ===========================================================================
// Uplink, fp32, split tile.  One warp per CTA (occupancy follows registers and
// shared memory exactly), NPW = 32/G problems per warp, LB = 2 coordinate
// blocks.  PF: sets of L2 prefetch lead.
// ===========================================================================
template <int BC, int U, int G, int JR, int MINB, int PF>
__global__ void __launch_bounds__(32, MINB)
    ul_split_f32(const float2* __restrict__ H, const float2* __restrict__ Y, int P, int K, float kappa,
                 float2* __restrict__ X) {
  static_assert(32 % G == 0 && BC % (2 * G) == 0 && U % 2 == 0 && JR % 2 == 0 && JR <= U, "shape");
  constexpr int NPW = 32 / G, R = BC / G, NP = R / 2, JS = U - JR, JRA = JR > 0 ? JR : 1;
  constexpr int T4 = BC * U / 2, Y4 = BC / 2;  // float4 per tile / per receive vector
  constexpr int SCAL_B = ul_scal_bytes(U, 2);
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x, g = lane / G, k = lane % G;
  float4* hs = reinterpret_cast<float4*>(smem) + g * (JS * NP * G);
  float4* mnx = reinterpret_cast<float4*>(smem + split_cols_bytes(BC, U, JR, G) + g * SCAL_B);
  float4* gb = mnx + U;  // (Re G, Im G, -Im G, Re G) of pair (2i+1, 2i)
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x;
  int set = blockIdx.x;
  if (lane == 0) {
#pragma unroll
    for (int f = 0; f < PF; ++f) {
      const int s = set + f * nw;
      if (s < nsets) {
        const int p0 = s * NPW, n = min(NPW, P - p0);
        prefetch_l2(H + static_cast<size_t>(p0) * BC * U, n * T4 * 16);
        prefetch_l2(Y + static_cast<size_t>(p0) * BC, n * Y4 * 16);
      }
    }
  }
  const float2 z2 = make_float2(0.f, 0.f);
  for (; set < nsets; set += nw) {
    if (lane == 0) {
      const int s = set + PF * nw;
      if (s < nsets) {
        const int p0 = s * NPW, n = min(NPW, P - p0);
        prefetch_l2(H + static_cast<size_t>(p0) * BC * U, n * T4 * 16);
        prefetch_l2(Y + static_cast<size_t>(p0) * BC, n * Y4 * 16);
      }
    }
    const int p = set * NPW + g;
    const int pc = min(p, P - 1);
    const float4* h4 = reinterpret_cast<const float4*>(H) + static_cast<size_t>(pc) * T4;
    const float4* y4 = reinterpret_cast<const float4*>(Y) + static_cast<size_t>(pc) * Y4;
    float2 hr[JRA][NP], hi[JRA][NP], rr[NP], ri[NP];
#pragma unroll
    for (int j = 0; j < JR; ++j)
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = ldg_na(h4 + j * (BC / 2) + c * G + k);
        hr[j][c] = pair(v.x, v.z);
        hi[j][c] = pair(v.y, v.w);
      }
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      const float4 v = ldg_na(y4 + c * G + k);
      rr[c] = pair(v.x, v.z);
      ri[c] = pair(v.y, v.w);
    }
    // shared-memory columns, re-paired to planar, in batches of 4 columns
#pragma unroll
    for (int j0 = JR; j0 < U; j0 += 4) {
      float4 v[4][NP];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c)
          if (j0 + j < U) v[j][c] = ldg_na(h4 + (j0 + j) * (BC / 2) + c * G + k);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c)
          if (j0 + j < U) hs[((j0 + j - JR) * NP + c) * G + k] = make_float4(v[j][c].x, v[j][c].z, v[j][c].y, v[j][c].w);
    }
    __syncwarp();

    // ---- per-problem scalars: ||h_j||^2 (detect.cpp:86-90) and the pair Grams
    {
      constexpr int NV = ((2 * U + G - 1) / G) * G;
      float v[NV];
#pragma unroll
      for (int q = 0; q < U / 2; ++q) {
        float2 ar[NP], ai[NP], br[NP], bi[NP];
        SplitCols<JR, NP, G>::get(2 * q, hr, hi, hs, k, ar, ai);
        SplitCols<JR, NP, G>::get(2 * q + 1, hr, hi, hs, k, br, bi);
        float2 ea = fmul2(ar[0], ar[0]), eb = fmul2(br[0], br[0]);
        ea = ffma2(ai[0], ai[0], ea);
        eb = ffma2(bi[0], bi[0], eb);
        float2 gr = z2, gi = z2;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          if (c > 0) {
            ea = ffma2(ai[c], ai[c], ffma2(ar[c], ar[c], ea));
            eb = ffma2(bi[c], bi[c], ffma2(br[c], br[c], eb));
          }
          // G_{2q+1,2q} = h_{2q+1}^H h_{2q}
          gr = ffma2(bi[c], ai[c], ffma2(br[c], ar[c], gr));
          gi = ffma2(neg2(bi[c]), ar[c], ffma2(br[c], ai[c], gi));
        }
        v[2 * q] = hsum(ea);
        v[2 * q + 1] = hsum(eb);
        v[U + 2 * q] = hsum(gr);
        v[U + 2 * q + 1] = hsum(gi);
      }
#pragma unroll
      for (int j = 2 * U; j < NV; ++j) v[j] = 0.f;
      group_reduce_scatter<G>(v, k);
      float* gf = reinterpret_cast<float*>(gb);
#pragma unroll
      for (int i = 0; i < NV / G; ++i) {
        const int idx = k * (NV / G) + i;
        if (idx < U) {
          const float m = __fdividef(1.f, v[i] + kappa);  // m_j = 1/(||h_j||^2 + N0/Ex)
          mnx[idx] = make_float4(m, m * v[i], 0.f, 0.f);  // n_j = m_j ||h_j||^2, x_j = 0
        } else if (idx < 2 * U) {
          const int e = (idx - U) >> 1;
          if ((idx - U) & 1) {
            gf[e * 4 + 1] = v[i];
            gf[e * 4 + 2] = -v[i];
          } else {
            gf[e * 4 + 0] = v[i];
            gf[e * 4 + 3] = v[i];
          }
        }
      }
    }
    __syncwarp();

    // ---- K sweeps over the users in ascending order, two coordinates per round
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int q = 0; q < U / 2; ++q) {
        float2 ar[NP], ai[NP], br[NP], bi[NP];
        SplitCols<JR, NP, G>::get(2 * q, hr, hi, hs, k, ar, ai);
        SplitCols<JR, NP, G>::get(2 * q + 1, hr, hi, hs, k, br, bi);
        float2 a0r = z2, a0i = z2, a1r = z2, a1i = z2;
#pragma unroll
        for (int c = 0; c < NP; ++c) {  // h_j^H r for both coordinates against the same r
          a0r = ffma2(ai[c], ri[c], ffma2(ar[c], rr[c], a0r));
          a0i = ffma2(neg2(ai[c]), rr[c], ffma2(ar[c], ri[c], a0i));
          a1r = ffma2(bi[c], ri[c], ffma2(br[c], rr[c], a1r));
          a1i = ffma2(neg2(bi[c]), rr[c], ffma2(br[c], ri[c], a1i));
        }
        float2 d0 = make_float2(hsum(a0r), hsum(a0i));
        float2 d1 = make_float2(hsum(a1r), hsum(a1i));
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          d0 = fadd2(d0, shfl_xor2(d0, o));
          d1 = fadd2(d1, shfl_xor2(d1, o));
        }
        const float4 A0 = mnx[2 * q], A1 = mnx[2 * q + 1], Gp = gb[q];
        // x_j' = m_j h_j^H r + n_j x_j ; dx = x_j' - x_j   (detect.cpp:100-103)
        const float2 x0 = make_float2(A0.z, A0.w), x1 = make_float2(A1.z, A1.w);
        const float2 n0v = ffma2(A0.x, d0, fmul2(A0.y, x0));
        const float2 dx0 = fadd2(n0v, neg2(x0));
        // h_{j+1}^H (r - dx_j h_j) = h_{j+1}^H r - dx_j G_{j+1,j}
        d1 = ffma2(-dx0.x, make_float2(Gp.x, Gp.y), d1);
        d1 = ffma2(-dx0.y, make_float2(Gp.z, Gp.w), d1);
        const float2 n1v = ffma2(A1.x, d1, fmul2(A1.y, x1));
        const float2 dx1 = fadd2(n1v, neg2(x1));
        *reinterpret_cast<float2*>(&mnx[2 * q].z) = n0v;  // every lane of the group stores the same value
        *reinterpret_cast<float2*>(&mnx[2 * q + 1].z) = n1v;
        // r -= dx_j h_j   (caxpy, detect.cpp:104)
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          rr[c] = ffma2(dx0.y, ai[c], ffma2(-dx0.x, ar[c], rr[c]));
          ri[c] = ffma2(-dx0.y, ar[c], ffma2(-dx0.x, ai[c], ri[c]));
          rr[c] = ffma2(dx1.y, bi[c], ffma2(-dx1.x, br[c], rr[c]));
          ri[c] = ffma2(-dx1.y, br[c], ffma2(-dx1.x, bi[c], ri[c]));
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
}

// ===========================================================================
// Downlink, fp32, split tile (see dl_reg_f32 for the algorithm, the
// unnormalised-row form of the update and the scalar block layout).
// ===========================================================================
template <int BC, int U, int G, int JR, int MINB, bool GAIN, int PF = 1>
__global__ void __launch_bounds__(32, MINB)
    dl_split_f32(const float2* __restrict__ H, const float2* __restrict__ Sy, int P, int C, int K, float rho_c,
                 float2* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status) {
  static_assert(32 % G == 0 && BC % (2 * G) == 0 && U % 2 == 0 && JR % 2 == 0 && JR <= U && (2 * U) % G == 0,
                "shape");
  constexpr int NPW = 32 / G, R = BC / G, NP = R / 2, JS = U - JR, JRA = JR > 0 ? JR : 1;
  constexpr int T4 = BC * U / 2;  // float4 per tile
  constexpr int SCAL_B = dl_scal_bytes(U);
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x, g = lane / G, k = lane % G;
  float4* hs = reinterpret_cast<float4*>(smem) + g * (JS * NP * G);
  float4* ss = reinterpret_cast<float4*>(smem + split_cols_bytes(BC, U, JR, G) + g * SCAL_B);
  float4* gp = ss + U;
  float2* sraw = reinterpret_cast<float2*>(gp + U / 2);
  float* dbuf = reinterpret_cast<float*>(sraw + U);  // 2 x 4 floats
  const int nsets = (P + NPW - 1) / NPW;
  const int nw = gridDim.x;
  int set = blockIdx.x;
  auto prefetch = [&](int s_) {
    if (s_ < nsets) {
      const int p0 = s_ * NPW, n = min(NPW, P - p0);
      prefetch_l2(H + static_cast<size_t>(p0) * BC * U, n * T4 * 16);
      const int v0 = p0 / C, nv = (p0 + n - 1) / C - v0 + 1;
      prefetch_l2(Sy + static_cast<size_t>(v0) * U, nv * U * 8);
    }
  };
  if (lane == 0)
#pragma unroll
    for (int f = 0; f < PF; ++f) prefetch(set + f * nw);
  const float2 z2 = make_float2(0.f, 0.f);
  for (; set < nsets; set += nw) {
    if (lane == 0) prefetch(set + PF * nw);
    const int p = set * NPW + g;
    const int pc = min(p, P - 1);
    const float4* h4 = reinterpret_cast<const float4*>(H) + static_cast<size_t>(pc) * T4;
    float2 hr[JRA][NP], hi[JRA][NP];
#pragma unroll
    for (int j = 0; j < JR; ++j)
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = ldg_na(h4 + j * (BC / 2) + c * G + k);
        hr[j][c] = pair(v.x, v.z);
        hi[j][c] = pair(v.y, v.w);
      }
    {
      const float4* s4 = reinterpret_cast<const float4*>(Sy + static_cast<size_t>(pc / C) * U);
      float4* d4 = reinterpret_cast<float4*>(sraw);
#pragma unroll
      for (int i = k; i < U / 2; i += G) d4[i] = ldg_na(s4 + i);
    }
#pragma unroll
    for (int j0 = JR; j0 < U; j0 += 4) {
      float4 v[4][NP];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c)
          if (j0 + j < U) v[j][c] = ldg_na(h4 + (j0 + j) * (BC / 2) + c * G + k);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c)
          if (j0 + j < U) hs[((j0 + j - JR) * NP + c) * G + k] = make_float4(v[j][c].x, v[j][c].z, v[j][c].y, v[j][c].w);
    }
    __syncwarp();

    // ---- row norms and raw pair Grams, reduce-scattered over the group
    constexpr int PER = 2 * U / G;
    float vv[2 * U];
#pragma unroll
    for (int q = 0; q < U / 2; ++q) {
      float2 ar[NP], ai[NP], br[NP], bi[NP];
      SplitCols<JR, NP, G>::get(2 * q, hr, hi, hs, k, ar, ai);
      SplitCols<JR, NP, G>::get(2 * q + 1, hr, hi, hs, k, br, bi);
      float2 ea = fmul2(ar[0], ar[0]), eb = fmul2(br[0], br[0]);
      ea = ffma2(ai[0], ai[0], ea);
      eb = ffma2(bi[0], bi[0], eb);
      float2 gr = z2, gi = z2;
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        if (c > 0) {
          ea = ffma2(ai[c], ai[c], ffma2(ar[c], ar[c], ea));
          eb = ffma2(bi[c], bi[c], ffma2(br[c], br[c], eb));
        }
        gr = ffma2(bi[c], ai[c], ffma2(br[c], ar[c], gr));
        gi = ffma2(neg2(bi[c]), ar[c], ffma2(br[c], ai[c], gi));
      }
      vv[2 * q] = hsum(ea);
      vv[2 * q + 1] = hsum(eb);
      vv[U + 2 * q] = hsum(gr);
      vv[U + 2 * q + 1] = hsum(gi);
    }
    group_reduce_scatter<G>(vv, k);
    int zero_user = -1;
    float* sf = reinterpret_cast<float*>(ss);
    float* gf = reinterpret_cast<float*>(gp);
    // unnormalised rows, normalisation in the scalars (see dl_reg_f32):
    // x -= q_u (h_u^H x - s_u) h_u, q_u = 1/||h_u||^2
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
        const int gi2 = idx - U, pr = gi2 >> 1;
        if (gi2 & 1) {
          gf[pr * 4 + 1] = vv[i];
          gf[pr * 4 + 2] = -vv[i];
        } else {
          gf[pr * 4 + 0] = vv[i];
          gf[pr * 4 + 3] = vv[i];
        }
      }
    }
    __syncwarp();

    float2 xr[NP], xi[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) xr[c] = xi[c] = z2;
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp) {
        const int j0 = 2 * jp, j1 = 2 * jp + 1;
        float2 ar[NP], ai[NP], br[NP], bi[NP];
        SplitCols<JR, NP, G>::get(j0, hr, hi, hs, k, ar, ai);
        SplitCols<JR, NP, G>::get(j1, hr, hi, hs, k, br, bi);
        const float4 S0 = ss[j0], S1 = ss[j1], GG = gp[jp];
        float2 a0 = z2, c0 = z2, a1 = z2, c1 = z2;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          a0 = ffma2(ai[c], xi[c], ffma2(ar[c], xr[c], a0));
          c0 = ffma2(neg2(ai[c]), xr[c], ffma2(ar[c], xi[c], c0));
          a1 = ffma2(bi[c], xi[c], ffma2(br[c], xr[c], a1));
          c1 = ffma2(neg2(bi[c]), xr[c], ffma2(br[c], xi[c], c1));
        }
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
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1) {
            d0 = fadd2(d0, shfl_xor2(d0, o));
            d1 = fadd2(d1, shfl_xor2(d1, o));
          }
        }
        // r_u = q_u (h_u^H x - s_u) ; x -= r_u h_u   (precode.cpp:89-94 on unnormalised rows)
        const float2 r0 = ffma2(S0.z, d0, make_float2(-S0.x, -S0.y));
        d1 = ffma2(-r0.x, make_float2(GG.x, GG.y), d1);
        d1 = ffma2(-r0.y, make_float2(GG.z, GG.w), d1);
        const float2 r1 = ffma2(S1.z, d1, make_float2(-S1.x, -S1.y));
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          xr[c] = ffma2(r0.y, ai[c], ffma2(-r0.x, ar[c], xr[c]));
          xi[c] = ffma2(-r0.y, ar[c], ffma2(-r0.x, ai[c], xi[c]));
          xr[c] = ffma2(r1.y, bi[c], ffma2(-r1.x, br[c], xr[c]));
          xi[c] = ffma2(-r1.y, br[c], ffma2(-r1.x, bi[c], xi[c]));
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
      float2 vr[NP], vi[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) vr[c] = vi[c] = z2;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float2 ar[NP], ai[NP];
        SplitCols<JR, NP, G>::get(j, hr, hi, hs, k, ar, ai);
        const float2 sj = sraw[j];
        const float cr = sj.x, ci = sj.y;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          vr[c] = ffma2(-ci, ai[c], ffma2(cr, ar[c], vr[c]));
          vi[c] = ffma2(ci, ar[c], ffma2(cr, ai[c], vi[c]));
        }
      }
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

}  // namespace dcdg
