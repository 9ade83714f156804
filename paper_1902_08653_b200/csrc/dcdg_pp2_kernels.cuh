// Uplink fp32 CD with TWO problems per lane group (the north-star tile).
//
// ul_reg_f32 (dcdg_reg_kernels.cuh) gives each problem G = 8 lanes: a lane
// holds 4 antenna rows x U columns of ONE problem, so the only parallelism
// inside a warp is SIMT across its 4 problems, and every coordinate block is
// one dependency chain (dot -> 3-level butterfly -> scalar update -> rank-1
// update -> next dot).  At 204 registers the SM keeps 2 such warps per
// scheduler, and the kernel is bound by that chain (ncu: issue-active 44%,
// FMA pipe 55%, stalls on fixed-latency waits and shuffle results).
//
// Here a group of 16 lanes holds two problems: lane k keeps row pair k
// (rows 2k, 2k+1) of BOTH problems' tiles, the same 128 registers of channel.
// Each lane therefore runs two independent chains, interleaved by the
// compiler, at the same warp count.  The block reduction is split by problem:
//   1. xor 8: lanes 0-7 keep problem 0's partials and send problem 1's, lanes
//      8-15 the reverse (a reduce-scatter level: 4 shuffles);
//   2. xor 4, 2, 1: butterfly inside each 8-lane half (12 shuffles), so lanes
//      0-7 hold problem 0's full dots and lanes 8-15 problem 1's;
//   3. each half runs ITS problem's scalar update (pair-Gram correction,
//      x_j' = m_j d_j + n_j x_j, dx) -- no redundant scalar work;
//   4. xor 8: the halves swap their dx (4 shuffles); both problems' rank-1
//      updates follow.
// Same sweep order, same coordinate pairs and pair-Gram correction as
// ul_reg_f32 (detect.cpp:97-108); only the summation order of the dots
// differs (rounding).  Staging, scalar blocks and the output are ul_reg_f32's
// with NPW = 4 problems per warp (group g holds problems 2g, 2g + 1 of the set).
#pragma once

#include "dcdg_device.cuh"
#include "dcdg_reg_kernels.cuh"

namespace dcdg {

// 1: reduce-scatter by problem (one chain, each half updates one problem);
// 0: a full butterfly per problem, two independent chains
#ifndef DCDG_PP2_SPLIT
#define DCDG_PP2_SPLIT 0
#endif

template <int BC, int U, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB)
    ul_pp2_f32(const float2* __restrict__ H, const float2* __restrict__ Y, int P, int K, float kappa,
               float2* __restrict__ X) {
  constexpr int G = 16, PP = 2, NPW = 4, LB = 2, T = 1;
  constexpr int R = BC / G, NP = R / 2;
  static_assert(BC % (2 * G) == 0 && U % 16 == 0, "shape: row pairs per lane, U a multiple of the group");
  constexpr int TILE_B = BC * U * 8, Y_B = BC * 8, SLOT_B = Slot<TILE_B, Y_B, NPW>::kBytes;
  constexpr int SCAL_B = ul_scal_bytes(U, LB);
  using L = CtaSmem<SLOT_B, SCAL_B, NPW, W>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  const int own = (k >> 3) & 1;  // the problem whose scalar update this lane runs
  unsigned char* slot = smem + warp * SLOT_B;
  float4* mnx[PP];
  float4* gb[PP];
#pragma unroll
  for (int pp = 0; pp < PP; ++pp) {
    mnx[pp] = reinterpret_cast<float4*>(smem + L::kScalOff + (warp * NPW + PP * g + pp) * SCAL_B);
    gb[pp] = mnx[pp] + U;
  }
  float4* mnx_own = own ? mnx[1] : mnx[0];
  const float4* gb_own = own ? gb[1] : gb[0];
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
    float2 hr[PP][U][NP], hi[PP][U][NP], rr[PP][NP], ri[PP][NP];
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const float4* t4 = reinterpret_cast<const float4*>(slot + (PP * g + pp) * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const float4 v = t4[j * (BC / 2) + c * G + k];
          hr[pp][j][c] = pair(v.x, v.z);
          hi[pp][j][c] = pair(v.y, v.w);
        }
      const float4* y4 = reinterpret_cast<const float4*>(slot + NPW * TILE_B + (PP * g + pp) * Y_B);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = y4[c * G + k];
        rr[pp][c] = pair(v.x, v.z);
        ri[pp][c] = pair(v.y, v.w);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);

    // ---- per-problem scalars: ||h_j||^2 (detect.cpp:86-90) and the pair Grams
    // G_{2q+1,2q} = h_{2q+1}^H h_{2q}, reduce-scattered over the 16 lanes
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      constexpr int NV = ((U + G - 1) / G) * G;
      float v[NV];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float2 e = fmul2(hr[pp][j][0], hr[pp][j][0]);
        e = ffma2(hi[pp][j][0], hi[pp][j][0], e);
#pragma unroll
        for (int c = 1; c < NP; ++c) e = ffma2(hi[pp][j][c], hi[pp][j][c], ffma2(hr[pp][j][c], hr[pp][j][c], e));
        v[j] = hsum(e);
      }
#pragma unroll
      for (int j = U; j < NV; ++j) v[j] = 0.f;
      group_reduce_scatter<G>(v, k);
#pragma unroll
      for (int i = 0; i < NV / G; ++i) {
        const int idx = k * (NV / G) + i;
        const float m = __fdividef(1.f, v[i] + kappa);  // m_j = 1/(||h_j||^2 + N0/Ex)
        if (idx < U) mnx[pp][idx] = make_float4(m, m * v[i], 0.f, 0.f);
      }
    }
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      constexpr int NG0 = 2 * (U / LB) * T;
      constexpr int NG = ((NG0 + G - 1) / G) * G;
      float v[NG];
#pragma unroll
      for (int e = NG0; e < NG; ++e) v[e] = 0.f;
#pragma unroll
      for (int q = 0; q < U / LB; ++q) {
        const int ja = q * LB + 1, jb = q * LB;
        float2 gr = z2, gi = z2;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          gr = ffma2(hi[pp][ja][c], hi[pp][jb][c], ffma2(hr[pp][ja][c], hr[pp][jb][c], gr));
          gi = ffma2(neg2(hi[pp][ja][c]), hr[pp][jb][c], ffma2(hr[pp][ja][c], hi[pp][jb][c], gi));
        }
        v[2 * q] = hsum(gr);
        v[2 * q + 1] = hsum(gi);
      }
      group_reduce_scatter<G>(v, k);
      float* gf = reinterpret_cast<float*>(gb[pp]);
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

    // ---- K sweeps over the users in ascending order, coordinate pairs
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int q = 0; q < U / LB; ++q) {
        float2 d[PP][LB];
#pragma unroll
        for (int pp = 0; pp < PP; ++pp)
#pragma unroll
          for (int a = 0; a < LB; ++a) {  // h_j^H r (cdotc, detect.cpp:100), both against the same r
            const int j = q * LB + a;
            float2 ar = z2, ai = z2;
#pragma unroll
            for (int c = 0; c < NP; ++c) {
              ar = ffma2(hi[pp][j][c], ri[pp][c], ffma2(hr[pp][j][c], rr[pp][c], ar));
              ai = ffma2(neg2(hi[pp][j][c]), rr[pp][c], ffma2(hr[pp][j][c], ri[pp][c], ai));
            }
            d[pp][a] = make_float2(hsum(ar), hsum(ai));
          }
#if DCDG_PP2_SPLIT
        // 1. reduce-scatter by problem across the halves
        float2 e[LB];
#pragma unroll
        for (int a = 0; a < LB; ++a) {
          const float2 keep = own ? d[1][a] : d[0][a];
          const float2 send = own ? d[0][a] : d[1][a];
          e[a] = fadd2(keep, shfl_xor2(send, 8));
        }
        // 2. butterfly inside the half: every lane of the half gets the sums
#pragma unroll
        for (int o = 4; o > 0; o >>= 1)
#pragma unroll
          for (int a = 0; a < LB; ++a) e[a] = fadd2(e[a], shfl_xor2(e[a], o));
        // 3. the half's own problem: x_j' = m_j h_j^H r + n_j x_j, dx = x_j' - x_j
        float2 dx[LB];
#pragma unroll
        for (int a = 0; a < LB; ++a) {
          const int j = q * LB + a;
          const float4 A = mnx_own[j];
          if (a == 1) {  // h_j^H (r - dx_0 h_{j-1}) = h_j^H r - dx_0 G_{j,j-1}
            const float4 Gab = gb_own[q];
            e[1] = ffma2(-dx[0].x, make_float2(Gab.x, Gab.y), e[1]);
            e[1] = ffma2(-dx[0].y, make_float2(Gab.z, Gab.w), e[1]);
          }
          const float2 xo = make_float2(A.z, A.w);
          const float2 xn = ffma2(A.x, e[a], fmul2(A.y, xo));
          dx[a] = fadd2(xn, neg2(xo));
          *reinterpret_cast<float2*>(&mnx_own[j].z) = xn;  // every lane of the half stores the same value
        }
        // 4. swap dx between the halves, then both problems' rank-1 updates
        float2 dxp[PP][LB];
#pragma unroll
        for (int a = 0; a < LB; ++a) {
          const float2 other = shfl_xor2(dx[a], 8);
          dxp[0][a] = own ? other : dx[a];
          dxp[1][a] = own ? dx[a] : other;
        }
#else
        // independent chains: each problem's dots by a full 16-lane butterfly,
        // its scalar update on every lane (the two problems interleave)
        float2 dxp[PP][LB];
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
          for (int pp = 0; pp < PP; ++pp)
#pragma unroll
            for (int a = 0; a < LB; ++a) d[pp][a] = fadd2(d[pp][a], shfl_xor2(d[pp][a], o));
#pragma unroll
        for (int pp = 0; pp < PP; ++pp)
#pragma unroll
          for (int a = 0; a < LB; ++a) {
            const int j = q * LB + a;
            const float4 A = mnx[pp][j];
            if (a == 1) {  // h_j^H (r - dx_0 h_{j-1}) = h_j^H r - dx_0 G_{j,j-1}
              const float4 Gab = gb[pp][q];
              d[pp][1] = ffma2(-dxp[pp][0].x, make_float2(Gab.x, Gab.y), d[pp][1]);
              d[pp][1] = ffma2(-dxp[pp][0].y, make_float2(Gab.z, Gab.w), d[pp][1]);
            }
            const float2 xo = make_float2(A.z, A.w);
            const float2 xn = ffma2(A.x, d[pp][a], fmul2(A.y, xo));
            dxp[pp][a] = fadd2(xn, neg2(xo));
            *reinterpret_cast<float2*>(&mnx[pp][j].z) = xn;  // every lane of the group stores the same value
          }
#endif
#pragma unroll
        for (int pp = 0; pp < PP; ++pp)
#pragma unroll
          for (int a = 0; a < LB; ++a) {  // r -= dx_j h_j   (caxpy, detect.cpp:104)
            const int j = q * LB + a;
#pragma unroll
            for (int c = 0; c < NP; ++c) {
              rr[pp][c] = ffma2(dxp[pp][a].y, hi[pp][j][c], ffma2(-dxp[pp][a].x, hr[pp][j][c], rr[pp][c]));
              ri[pp][c] = ffma2(-dxp[pp][a].y, hr[pp][j][c], ffma2(-dxp[pp][a].x, hi[pp][j][c], ri[pp][c]));
            }
          }
      }
    }
    __syncwarp();
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const int p = set * NPW + PP * g + pp;
      if (p < P) {
        float4* xo = reinterpret_cast<float4*>(X + static_cast<size_t>(p) * U);
#pragma unroll
        for (int i = k; i < U / 2; i += G) {
          const float4 u0 = mnx[pp][2 * i], u1 = mnx[pp][2 * i + 1];
          xo[i] = make_float4(u0.z, u0.w, u1.z, u1.w);
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace dcdg
