// CD detect / precode kernels for sm_100a.
//
// Mapping ("register-resident sub-warp" kernels, the hot path):
//   * G consecutive lanes own one (subcarrier, cluster) problem; a warp holds
//     NPW = 32/G problems.  Lane k of a group owns R = B_c/G antenna rows:
//     row chunks q*G + k (chunk = 2 complex fp32 / 4 complex fp16 = 16 B), so
//     every 16-B load of a group is contiguous (coalesced global traffic,
//     conflict-free 128-B shared-memory phases).
//   * The whole B_c x U channel tile lives in registers for the K sweeps
//     (B_c*U/G complex per lane, 128 regs at the target shape); the residual
//     r (uplink) or beamformer x (downlink) stays in registers too.
//   * Each coordinate update is a local R-row complex dot, a log2(G)-step
//     xor-butterfly over the group, a scalar update replicated in every lane
//     (bitwise identical across the group) and a local rank-1 axpy.
//   * Tiles are staged HBM -> shared memory by one cp.async.bulk (TMA 1-D)
//     per warp and set, completing on a per-warp mbarrier; the next set's
//     copy is issued as soon as the current set is in registers, so the HBM
//     stream overlaps the whole sweep computation.  Warps are persistent
//     (grid sized to the SM count x occupancy).
// Reference algorithms: uplink Alg. 1 = cd_detect (src/detect.cpp:67-110);
// downlink Alg. 2 = cd_precode + power_scale (src/precode.cpp:52-111).
#pragma once

#include "dcdg_device.cuh"

namespace dcdg {

// Per-warp staging slot for NPW problems: [NPW tiles][NPW vectors] + mbarrier.
template <int TILE_B, int VEC_B, int NPW>
struct Slot {
  static constexpr int kBytes = NPW * (TILE_B + VEC_B);
};

// Issue the bulk copies of set `set` (problems [set*NPW, set*NPW + n)).
// `vec` holds per-problem vectors (uplink y) or, for the downlink, the symbol
// vectors of the subcarriers the set touches (vec_per_problem == false).
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

// ===========================================================================
// Uplink, fp32 storage + fp32 math
// ===========================================================================
template <int BC, int U, int G, int W>
__global__ void __launch_bounds__(32 * W) ul_reg_f32(const float2* __restrict__ H, const float2* __restrict__ Y,
                                                     int P, int K, float kappa, float2* __restrict__ X) {
  static_assert(32 % G == 0 && BC % (2 * G) == 0, "shape");
  constexpr int NPW = 32 / G, R = BC / G, CH = R / 2;
  constexpr int TILE_B = BC * U * 8, Y_B = BC * 8, SLOT_B = Slot<TILE_B, Y_B, NPW>::kBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + W * SLOT_B) + warp;
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
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    float hr[U][R], hi[U][R], rr[R], ri[R];
    {
      const float4* t4 = reinterpret_cast<const float4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const float4 v = t4[j * (BC / 2) + c * G + k];
          hr[j][2 * c] = v.x;
          hi[j][2 * c] = v.y;
          hr[j][2 * c + 1] = v.z;
          hi[j][2 * c + 1] = v.w;
        }
      const float4* y4 = reinterpret_cast<const float4*>(slot + NPW * TILE_B + g * Y_B);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const float4 v = y4[c * G + k];
        rr[2 * c] = v.x;
        ri[2 * c] = v.y;
        rr[2 * c + 1] = v.z;
        ri[2 * c + 1] = v.w;
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);

    // m_j = 1/(||h_j||^2 + N0/Ex), n_j = m_j ||h_j||^2   (detect.cpp:84-90)
    float m[U], n[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      float e = 0.f;
#pragma unroll
      for (int q = 0; q < R; ++q) e = fmaf(hi[j][q], hi[j][q], fmaf(hr[j][q], hr[j][q], e));
      e = gsum<G>(e);
      m[j] = __frcp_rn(e + kappa);
      n[j] = m[j] * e;
    }
    float xr[U], xi[U];
#pragma unroll
    for (int j = 0; j < U; ++j) xr[j] = xi[j] = 0.f;
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        // h_j^H r  (cdotc, detect.cpp:100)
        float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          a0 = fmaf(hr[j][q], rr[q], a0);
          a1 = fmaf(hi[j][q], ri[q], a1);
          b0 = fmaf(hr[j][q], ri[q], b0);
          b1 = fmaf(hi[j][q], rr[q], b1);
        }
        const float dr = gsum<G>(a0 + a1);
        const float di = gsum<G>(b0 - b1);
        // x_j' = m_j h_j^H r + n_j x_j ; dx = x_j' - x_j   (detect.cpp:100-103)
        const float nxr = fmaf(m[j], dr, n[j] * xr[j]);
        const float nxi = fmaf(m[j], di, n[j] * xi[j]);
        const float dxr = nxr - xr[j], dxi = nxi - xi[j];
        xr[j] = nxr;
        xi[j] = nxi;
        // r -= dx h_j   (caxpy, detect.cpp:104)
#pragma unroll
        for (int q = 0; q < R; ++q) {
          rr[q] = fmaf(-dxr, hr[j][q], fmaf(dxi, hi[j][q], rr[q]));
          ri[q] = fmaf(-dxr, hi[j][q], fmaf(-dxi, hr[j][q], ri[q]));
        }
      }
    }
    const int p = set * NPW + g;
    if (p < P) {
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (j % G == k) X[static_cast<size_t>(p) * U + j] = make_float2(xr[j], xi[j]);
    }
  }
}

// ===========================================================================
// Uplink, fp16 storage + half2 math (the paper's half-precision path)
// In registers each lane keeps row PAIRS in planar half2 form
// (re_i, re_i+1), (im_i, im_i+1): a complex MAC over two rows is 2 HFMA2
// instead of 4 FFMA per row.  Dots accumulate in half2 per lane, the group
// reduction moves one packed (re, im) half2 per shuffle, scalar updates run
// in fp32.
// ===========================================================================
template <int BC, int U, int G, int W>
__global__ void __launch_bounds__(32 * W) ul_reg_f16(const __half2* __restrict__ H, const __half2* __restrict__ Y,
                                                     int P, int K, float kappa, __half2* __restrict__ X) {
  static_assert(32 % G == 0 && BC % (4 * G) == 0, "shape");
  constexpr int NPW = 32 / G, R = BC / G, CH = R / 4, NP = R / 2;
  constexpr int TILE_B = BC * U * 4, Y_B = BC * 4, SLOT_B = Slot<TILE_B, Y_B, NPW>::kBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + W * SLOT_B) + warp;
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
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    __half2 hre[U][NP], him[U][NP], rre[NP], rim[NP];
    {
      const uint4* t4 = reinterpret_cast<const uint4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 v = t4[j * (BC / 4) + c * G + k];
          const __half2 a = u32_as_h2(v.x), b = u32_as_h2(v.y), cc = u32_as_h2(v.z), d = u32_as_h2(v.w);
          hre[j][2 * c] = __lows2half2(a, b);
          him[j][2 * c] = __highs2half2(a, b);
          hre[j][2 * c + 1] = __lows2half2(cc, d);
          him[j][2 * c + 1] = __highs2half2(cc, d);
        }
      const uint4* y4 = reinterpret_cast<const uint4*>(slot + NPW * TILE_B + g * Y_B);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const uint4 v = y4[c * G + k];
        const __half2 a = u32_as_h2(v.x), b = u32_as_h2(v.y), cc = u32_as_h2(v.z), d = u32_as_h2(v.w);
        rre[2 * c] = __lows2half2(a, b);
        rim[2 * c] = __highs2half2(a, b);
        rre[2 * c + 1] = __lows2half2(cc, d);
        rim[2 * c + 1] = __highs2half2(cc, d);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Y, set + nw, P, NPW, TILE_B, Y_B, true, 1, pol);

    float m[U], n[U];
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
      const float e = gsum<G>(f.x + f.y);
      m[j] = __frcp_rn(e + kappa);
      n[j] = m[j] * e;
    }
    float xr[U], xi[U];
#pragma unroll
    for (int j = 0; j < U; ++j) xr[j] = xi[j] = 0.f;
    const __half2 z2 = __float2half2_rn(0.f);
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        __half2 ar = z2, ai = z2, br = z2, bi = z2;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          ar = __hfma2(hre[j][q], rre[q], ar);
          ai = __hfma2(him[j][q], rim[q], ai);
          br = __hfma2(hre[j][q], rim[q], br);
          bi = __hfma2(him[j][q], rre[q], bi);
        }
        const __half2 re2 = __hadd2(ar, ai), im2 = __hsub2(br, bi);
        const __half2 d = gsum_h2<G>(__hadd2(__lows2half2(re2, im2), __highs2half2(re2, im2)));
        const float2 df = __half22float2(d);
        const float nxr = fmaf(m[j], df.x, n[j] * xr[j]);
        const float nxi = fmaf(m[j], df.y, n[j] * xi[j]);
        const float dxr = nxr - xr[j], dxi = nxi - xi[j];
        xr[j] = nxr;
        xi[j] = nxi;
        const __half2 ndr = __float2half2_rn(-dxr), pdi = __float2half2_rn(dxi), ndi = __float2half2_rn(-dxi);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          rre[q] = __hfma2(ndr, hre[j][q], __hfma2(pdi, him[j][q], rre[q]));
          rim[q] = __hfma2(ndr, him[j][q], __hfma2(ndi, hre[j][q], rim[q]));
        }
      }
    }
    const int p = set * NPW + g;
    if (p < P) {
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (j % G == k) X[static_cast<size_t>(p) * U + j] = __floats2half2_rn(xr[j], xi[j]);
    }
  }
}

// ===========================================================================
// Downlink, fp32.  Rows h_u of the dual problem are the uplink columns
// (conj_rows, precode.cpp:19-27); they are normalised in registers
// (p_u = 1/||h_u||, precode.cpp:69-87), the K dual sweeps update the local
// beamformer rows, then power_scale (precode.cpp:101-111) and the cluster's
// effective-gain share Re(s^H H_dl,c x_c) = Re((H_c s)^H x_c).
// ===========================================================================
template <int BC, int U, int G, int W, bool GAIN>
__global__ void __launch_bounds__(32 * W)
    dl_reg_f32(const float2* __restrict__ H, const float2* __restrict__ Sy, int P, int C, int K, float rho_c,
               float2* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status) {
  static_assert(32 % G == 0 && BC % (2 * G) == 0, "shape");
  constexpr int NPW = 32 / G, R = BC / G, CH = R / 2;
  constexpr int TILE_B = BC * U * 8, S_B = U * 8, SLOT_B = Slot<TILE_B, S_B, NPW>::kBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + W * SLOT_B) + warp;
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
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const int p = set * NPW + g;
    float hr[U][R], hi[U][R], sr[U], si[U];
    {
      const float4* t4 = reinterpret_cast<const float4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const float4 v = t4[j * (BC / 2) + c * G + k];
          hr[j][2 * c] = v.x;
          hi[j][2 * c] = v.y;
          hr[j][2 * c + 1] = v.z;
          hi[j][2 * c + 1] = v.w;
        }
      const int sidx = (min(p, P - 1)) / C - (set * NPW) / C;
      const float2* s2 = reinterpret_cast<const float2*>(slot + NPW * TILE_B) + sidx * U;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const float2 v = s2[j];
        sr[j] = v.x;
        si[j] = v.y;
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Sy, set + nw, P, NPW, TILE_B, S_B, false, C, pol);

    // v = H_c s (unnormalised rows) for the gain share
    float vr[R], vi[R];
    if (GAIN) {
#pragma unroll
      for (int q = 0; q < R; ++q) vr[q] = vi[q] = 0.f;
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int q = 0; q < R; ++q) {
          vr[q] = fmaf(sr[j], hr[j][q], fmaf(-si[j], hi[j][q], vr[q]));
          vi[q] = fmaf(sr[j], hi[j][q], fmaf(si[j], hr[j][q], vi[q]));
        }
    }
    // p_u = 1/||h_u||; h_u *= p_u; s_u *= p_u   (precode.cpp:69-87)
    bool zero_row = false;
    int zero_user = 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      float e = 0.f;
#pragma unroll
      for (int q = 0; q < R; ++q) e = fmaf(hi[j][q], hi[j][q], fmaf(hr[j][q], hr[j][q], e));
      e = gsum<G>(e);
      if (e == 0.f && !zero_row) {
        zero_row = true;
        zero_user = j;
      }
      const float pj = __frcp_rn(__fsqrt_rn(e));
#pragma unroll
      for (int q = 0; q < R; ++q) {
        hr[j][q] *= pj;
        hi[j][q] *= pj;
      }
      sr[j] *= pj;
      si[j] *= pj;
    }
    float xr[R], xi[R];
#pragma unroll
    for (int q = 0; q < R; ++q) xr[q] = xi[q] = 0.f;
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        // resid = h_u^H x - s_u ; x -= resid h_u   (precode.cpp:89-94)
        float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          a0 = fmaf(hr[j][q], xr[q], a0);
          a1 = fmaf(hi[j][q], xi[q], a1);
          b0 = fmaf(hr[j][q], xi[q], b0);
          b1 = fmaf(hi[j][q], xr[q], b1);
        }
        const float rsr = gsum<G>(a0 + a1) - sr[j];
        const float rsi = gsum<G>(b0 - b1) - si[j];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          xr[q] = fmaf(-rsr, hr[j][q], fmaf(rsi, hi[j][q], xr[q]));
          xi[q] = fmaf(-rsr, hi[j][q], fmaf(-rsi, hr[j][q], xi[q]));
        }
      }
    }
    // power_scale to rho_c = rho / sqrt(C)   (precode.cpp:101-111,155)
    float e = 0.f;
#pragma unroll
    for (int q = 0; q < R; ++q) e = fmaf(xi[q], xi[q], fmaf(xr[q], xr[q], e));
    e = gsum<G>(e);
    const float gsc = rho_c > 0.f ? rho_c / __fsqrt_rn(e) : 1.f;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      xr[q] *= gsc;
      xi[q] *= gsc;
    }
    float gq = 0.f;
    if (GAIN) {
#pragma unroll
      for (int q = 0; q < R; ++q) gq = fmaf(vr[q], xr[q], fmaf(vi[q], xi[q], gq));
      gq = gsum<G>(gq);
    }
    if (p < P) {
      if (k == 0) {
        if (zero_row) record_status(status, p, ST_ZERO_ROW, zero_user);
        else if (e == 0.f && rho_c > 0.f) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
        if (GAIN) gain_part[p] = gq;
      }
      float4* x4 = reinterpret_cast<float4*>(X + static_cast<size_t>(p) * BC);
#pragma unroll
      for (int c = 0; c < CH; ++c)
        x4[c * G + k] = make_float4(xr[2 * c], xi[2 * c], xr[2 * c + 1], xi[2 * c + 1]);
    }
  }
}

// ===========================================================================
// Downlink, fp16 storage + half2 math
// ===========================================================================
template <int BC, int U, int G, int W, bool GAIN>
__global__ void __launch_bounds__(32 * W)
    dl_reg_f16(const __half2* __restrict__ H, const __half2* __restrict__ Sy, int P, int C, int K, float rho_c,
               __half2* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status) {
  static_assert(32 % G == 0 && BC % (4 * G) == 0, "shape");
  constexpr int NPW = 32 / G, R = BC / G, CH = R / 4, NP = R / 2;
  constexpr int TILE_B = BC * U * 4, S_B = U * 4, SLOT_B = Slot<TILE_B, S_B, NPW>::kBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  unsigned char* slot = smem + warp * SLOT_B;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + W * SLOT_B) + warp;
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
  for (; set < nsets; set += nw) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const int p = set * NPW + g;
    __half2 hre[U][NP], him[U][NP];
    float sr[U], si[U];
    {
      const uint4* t4 = reinterpret_cast<const uint4*>(slot + g * TILE_B);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 v = t4[j * (BC / 4) + c * G + k];
          const __half2 a = u32_as_h2(v.x), b = u32_as_h2(v.y), cc = u32_as_h2(v.z), d = u32_as_h2(v.w);
          hre[j][2 * c] = __lows2half2(a, b);
          him[j][2 * c] = __highs2half2(a, b);
          hre[j][2 * c + 1] = __lows2half2(cc, d);
          him[j][2 * c + 1] = __highs2half2(cc, d);
        }
      const int sidx = (min(p, P - 1)) / C - (set * NPW) / C;
      const __half2* s2 = reinterpret_cast<const __half2*>(slot + NPW * TILE_B) + sidx * U;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const float2 v = __half22float2(s2[j]);
        sr[j] = v.x;
        si[j] = v.y;
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && set + nw < nsets) issue_set(slot, bar, H, Sy, set + nw, P, NPW, TILE_B, S_B, false, C, pol);

    const __half2 z2 = __float2half2_rn(0.f);
    __half2 vre[NP], vim[NP];
    if (GAIN) {
#pragma unroll
      for (int q = 0; q < NP; ++q) vre[q] = vim[q] = z2;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const __half2 s_r = __float2half2_rn(sr[j]), s_i = __float2half2_rn(si[j]), n_i = __float2half2_rn(-si[j]);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          vre[q] = __hfma2(s_r, hre[j][q], __hfma2(n_i, him[j][q], vre[q]));
          vim[q] = __hfma2(s_r, him[j][q], __hfma2(s_i, hre[j][q], vim[q]));
        }
      }
    }
    bool zero_row = false;
    int zero_user = 0;
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
      const float e = gsum<G>(f.x + f.y);
      if (e == 0.f && !zero_row) {
        zero_row = true;
        zero_user = j;
      }
      const float pj = __frcp_rn(__fsqrt_rn(e));
      const __half2 p2 = __float2half2_rn(pj);
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        hre[j][q] = __hmul2(p2, hre[j][q]);
        him[j][q] = __hmul2(p2, him[j][q]);
      }
      sr[j] *= pj;
      si[j] *= pj;
    }
    __half2 xre[NP], xim[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) xre[q] = xim[q] = z2;
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        __half2 ar = z2, ai = z2, br = z2, bi = z2;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          ar = __hfma2(hre[j][q], xre[q], ar);
          ai = __hfma2(him[j][q], xim[q], ai);
          br = __hfma2(hre[j][q], xim[q], br);
          bi = __hfma2(him[j][q], xre[q], bi);
        }
        const __half2 re2 = __hadd2(ar, ai), im2 = __hsub2(br, bi);
        const __half2 d = gsum_h2<G>(__hadd2(__lows2half2(re2, im2), __highs2half2(re2, im2)));
        const float2 df = __half22float2(d);
        const float rsr = df.x - sr[j], rsi = df.y - si[j];
        const __half2 ndr = __float2half2_rn(-rsr), pdi = __float2half2_rn(rsi), ndi = __float2half2_rn(-rsi);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          xre[q] = __hfma2(ndr, hre[j][q], __hfma2(pdi, him[j][q], xre[q]));
          xim[q] = __hfma2(ndr, him[j][q], __hfma2(ndi, hre[j][q], xim[q]));
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
      if (k == 0) {
        if (zero_row) record_status(status, p, ST_ZERO_ROW, zero_user);
        else if (e == 0.f && rho_c > 0.f) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
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
  }
}

// ===========================================================================
// Generic kernels: any B_c, U (one warp per problem, fp32 math).  Used for
// shapes without a register-resident specialisation and for fp16 shapes
// whose B_c is not a multiple of 4G.  Residual / beamformer and scalars live
// in shared memory; lane l owns rows l, l+32, ...
// ===========================================================================
template <typename T>
__global__ void __launch_bounds__(128) ul_generic(const T* __restrict__ H, const T* __restrict__ Y, int P, int BC,
                                                  int U, int K, float kappa, T* __restrict__ X) {
  extern __shared__ float2 gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (p >= P) return;
  float2* r = gsm + warp * (BC + 2 * U);
  float2* x = r + BC;
  float2* mn = x + U;
  const T* h = H + static_cast<size_t>(p) * BC * U;
  for (int i = lane; i < BC; i += 32) r[i] = ldc(Y, static_cast<size_t>(p) * BC + i);
  for (int j = 0; j < U; ++j) {
    float e = 0.f;
    for (int i = lane; i < BC; i += 32) {
      const float2 v = ldc(h, static_cast<size_t>(j) * BC + i);
      e = fmaf(v.y, v.y, fmaf(v.x, v.x, e));
    }
    e = warp_sum(e);
    if (lane == 0) {
      const float m = __frcp_rn(e + kappa);
      mn[j] = make_float2(m, m * e);
      x[j] = make_float2(0.f, 0.f);
    }
  }
  __syncwarp();
  for (int t = 0; t < K; ++t)
    for (int j = 0; j < U; ++j) {
      float dr = 0.f, di = 0.f;
      for (int i = lane; i < BC; i += 32) {
        const float2 hv = ldc(h, static_cast<size_t>(j) * BC + i);
        const float2 rv = r[i];
        dr = fmaf(hv.x, rv.x, fmaf(hv.y, rv.y, dr));
        di = fmaf(hv.x, rv.y, fmaf(-hv.y, rv.x, di));
      }
      dr = warp_sum(dr);
      di = warp_sum(di);
      const float2 mnj = mn[j], xo = x[j];
      const float nxr = fmaf(mnj.x, dr, mnj.y * xo.x), nxi = fmaf(mnj.x, di, mnj.y * xo.y);
      const float dxr = nxr - xo.x, dxi = nxi - xo.y;
      __syncwarp();
      if (lane == 0) x[j] = make_float2(nxr, nxi);
      for (int i = lane; i < BC; i += 32) {
        const float2 hv = ldc(h, static_cast<size_t>(j) * BC + i);
        float2 rv = r[i];
        rv.x = fmaf(-dxr, hv.x, fmaf(dxi, hv.y, rv.x));
        rv.y = fmaf(-dxr, hv.y, fmaf(-dxi, hv.x, rv.y));
        r[i] = rv;
      }
      __syncwarp();
    }
  for (int j = lane; j < U; j += 32) stc(X, static_cast<size_t>(p) * U + j, x[j]);
}

template <typename T, bool GAIN>
__global__ void __launch_bounds__(128)
    dl_generic(const T* __restrict__ H, const T* __restrict__ Sy, int P, int C, int BC, int U, int K, float rho_c,
               T* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status) {
  extern __shared__ float2 gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (p >= P) return;
  float2* x = gsm + warp * (BC + 2 * U);
  float2* sb = x + BC;  // normalised targets
  float* pn = reinterpret_cast<float*>(sb + U);  // row normalisers
  const T* h = H + static_cast<size_t>(p) * BC * U;
  const T* s = Sy + static_cast<size_t>(p / C) * U;
  int zero_user = -1;
  for (int j = 0; j < U; ++j) {
    float e = 0.f;
    for (int i = lane; i < BC; i += 32) {
      const float2 v = ldc(h, static_cast<size_t>(j) * BC + i);
      e = fmaf(v.y, v.y, fmaf(v.x, v.x, e));
    }
    e = warp_sum(e);
    if (e == 0.f && zero_user < 0) zero_user = j;
    const float pj = __frcp_rn(__fsqrt_rn(e));
    if (lane == 0) {
      const float2 sv = ldc(s, j);
      sb[j] = make_float2(sv.x * pj, sv.y * pj);
      pn[j] = pj;
    }
  }
  for (int i = lane; i < BC; i += 32) x[i] = make_float2(0.f, 0.f);
  __syncwarp();
  for (int t = 0; t < K; ++t)
    for (int j = 0; j < U; ++j) {
      const float pj = pn[j];
      float dr = 0.f, di = 0.f;
      for (int i = lane; i < BC; i += 32) {
        float2 hv = ldc(h, static_cast<size_t>(j) * BC + i);
        hv.x *= pj;
        hv.y *= pj;
        const float2 xv = x[i];
        dr = fmaf(hv.x, xv.x, fmaf(hv.y, xv.y, dr));
        di = fmaf(hv.x, xv.y, fmaf(-hv.y, xv.x, di));
      }
      dr = warp_sum(dr) - sb[j].x;
      di = warp_sum(di) - sb[j].y;
      for (int i = lane; i < BC; i += 32) {
        float2 hv = ldc(h, static_cast<size_t>(j) * BC + i);
        hv.x *= pj;
        hv.y *= pj;
        float2 xv = x[i];
        xv.x = fmaf(-dr, hv.x, fmaf(di, hv.y, xv.x));
        xv.y = fmaf(-dr, hv.y, fmaf(-di, hv.x, xv.y));
        x[i] = xv;
      }
    }
  float e = 0.f;
  for (int i = lane; i < BC; i += 32) e = fmaf(x[i].y, x[i].y, fmaf(x[i].x, x[i].x, e));
  e = warp_sum(e);
  const float gsc = rho_c > 0.f ? rho_c / __fsqrt_rn(e) : 1.f;
  float gq = 0.f;
  for (int i = lane; i < BC; i += 32) {
    const float2 xv = make_float2(x[i].x * gsc, x[i].y * gsc);
    stc(X, static_cast<size_t>(p) * BC + i, xv);
    if (GAIN) {
      // v_i = sum_u s_u h_iu (unnormalised)
      float vr = 0.f, vi = 0.f;
      for (int j = 0; j < U; ++j) {
        const float2 hv = ldc(h, static_cast<size_t>(j) * BC + i);
        const float2 sv = ldc(s, j);
        vr = fmaf(sv.x, hv.x, fmaf(-sv.y, hv.y, vr));
        vi = fmaf(sv.x, hv.y, fmaf(sv.y, hv.x, vi));
      }
      gq = fmaf(vr, xv.x, fmaf(vi, xv.y, gq));
    }
  }
  if (GAIN) gq = warp_sum(gq);
  if (lane == 0) {
    if (zero_user >= 0) record_status(status, p, ST_ZERO_ROW, zero_user);
    else if (e == 0.f && rho_c > 0.f) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
    if (GAIN) gain_part[p] = gq;
  }
}

// ===========================================================================
// Post-equalization variance (optimal fusion), one warp per problem:
// A = I + (Ex/N0) H^H H (Gram, detect.cpp:21-28,118-121); Cholesky A = L L^H
// (numerics.cpp:45-58); sigma^2 = (Ex/U) tr(A^-1) = (Ex/U) ||L^-1||_F^2
// (the reference sums U Cholesky solves, detect.cpp:122-129).
// Shared memory per warp: A/L [U][U] + Z [U][U] complex fp32 (U <= 32).
// ===========================================================================
template <typename T>
__global__ void __launch_bounds__(128) post_eq_var(const T* __restrict__ H, int P, int BC, int U, float gam,
                                                   float ex_over_u, bool round_fp16, float* __restrict__ sigma2,
                                                   unsigned long long* __restrict__ status) {
  extern __shared__ float2 vsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (p >= P) return;
  float2* A = vsm + warp * (2 * U * U);  // column-major, lower triangle used
  float2* Z = A + U * U;
  const T* h = H + static_cast<size_t>(p) * BC * U;
  const int ntri = U * (U + 1) / 2;
  for (int e = lane; e < ntri; e += 32) {
    // e -> (i >= j): column j, row i
    int j = 0, rem = e;
    while (rem >= U - j) {
      rem -= U - j;
      ++j;
    }
    const int i = j + rem;
    float gr = 0.f, gi = 0.f;  // conj(h_i)^T h_j
    for (int b = 0; b < BC; ++b) {
      const float2 a = ldc(h, static_cast<size_t>(i) * BC + b);
      const float2 c = ldc(h, static_cast<size_t>(j) * BC + b);
      gr = fmaf(a.x, c.x, fmaf(a.y, c.y, gr));
      gi = fmaf(a.x, c.y, fmaf(-a.y, c.x, gi));
    }
    A[j * U + i] = make_float2((i == j ? 1.f : 0.f) + gam * gr, gam * gi);
  }
  __syncwarp();
  float maxdiag = 0.f;  // numerics.cpp:38-41 (pivot floor 1e-14 * max |A_jj|)
  for (int j = lane; j < U; j += 32) maxdiag = fmaxf(maxdiag, fabsf(A[j * U + j].x));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) maxdiag = fmaxf(maxdiag, __shfl_xor_sync(0xffffffffu, maxdiag, o));
  const float floor_ = 1e-14f * maxdiag;
  bool singular = false;
  // left-looking Cholesky, lanes parallel over rows i >= j
  for (int j = 0; j < U; ++j) {
    float d = A[j * U + j].x;
    for (int kk = 0; kk < j; ++kk) {
      const float2 l = A[kk * U + j];
      d -= l.x * l.x + l.y * l.y;
    }
    if (!(d > floor_)) singular = true;
    const float ljj = __fsqrt_rn(fmaxf(d, 1e-30f));
    for (int i = j + 1 + lane; i < U; i += 32) {
      float2 s = A[j * U + i];
      for (int kk = 0; kk < j; ++kk) {
        const float2 a = A[kk * U + i], b = A[kk * U + j];  // s -= L_ik conj(L_jk)
        s.x -= a.x * b.x + a.y * b.y;
        s.y -= a.y * b.x - a.x * b.y;
      }
      A[j * U + i] = make_float2(s.x / ljj, s.y / ljj);
    }
    __syncwarp();
    if (lane == 0) A[j * U + j] = make_float2(ljj, 0.f);
    __syncwarp();
  }
  // columns of L^-1: lane c solves L z = e_c (rows i >= c)
  float tr = 0.f;
  for (int c = lane; c < U; c += 32) {
    for (int i = c; i < U; ++i) {
      float sr = (i == c) ? 1.f : 0.f, si = 0.f;
      for (int kk = c; kk < i; ++kk) {
        const float2 l = A[kk * U + i], z = Z[c * U + kk];
        sr -= l.x * z.x - l.y * z.y;
        si -= l.x * z.y + l.y * z.x;
      }
      const float li = A[i * U + i].x;
      const float2 z = make_float2(sr / li, si / li);
      Z[c * U + i] = z;
      tr = fmaf(z.x, z.x, fmaf(z.y, z.y, tr));
    }
  }
  tr = warp_sum(tr);
  if (lane == 0) {
    float s2 = ex_over_u * tr;
    if (round_fp16) s2 = __half2float(__float2half_rn(s2));
    sigma2[p] = s2;
    if (singular) record_status(status, p, ST_SINGULAR, 0);
  }
}

// ===========================================================================
// Fusion (detect.cpp:132-145,180-187): one thread per (subcarrier, user),
// ascending cluster order.  Full fusion (C == C_total) reproduces the
// reference's weights; partial fusion (C < C_total, multi-GPU) emits
// sum_c w_c x_c with uniform w = 1/C_total, or sum_c x_c / sigma_c^2 plus the
// weight sum for the optimal cross-GPU normalisation.
// ===========================================================================
template <typename T>
__global__ void fuse_kernel(const T* __restrict__ XL, const float* __restrict__ sigma2, int S, int C, int C_total, int U,
                            bool optimal, float2* __restrict__ xhat, float* __restrict__ wsum,
                            unsigned long long* __restrict__ status) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(S) * U) return;
  const long long s = idx / U;
  const int u = static_cast<int>(idx - s * U);
  const bool full = C == C_total;
  float2 acc = make_float2(0.f, 0.f);
  if (!optimal) {
    const float w = 1.f / static_cast<float>(C_total);
    for (int c = 0; c < C; ++c) {
      const float2 v = ldc(XL, (static_cast<size_t>(s) * C + c) * U + u);
      acc.x = fmaf(w, v.x, acc.x);
      acc.y = fmaf(w, v.y, acc.y);
    }
  } else {
    float total = 0.f;
    bool bad = false;
    for (int c = 0; c < C; ++c) {
      const float v = sigma2[s * C + c];
      if (!(v > 0.f) || !isfinite(v)) bad = true;
      total += 1.f / v;
    }
    if (bad && u == 0) record_status(status, s * C, ST_BAD_VARIANCE, 0);
    for (int c = 0; c < C; ++c) {
      const float w = full ? (1.f / sigma2[s * C + c]) / total : 1.f / sigma2[s * C + c];
      const float2 v = ldc(XL, (static_cast<size_t>(s) * C + c) * U + u);
      acc.x = fmaf(w, v.x, acc.x);
      acc.y = fmaf(w, v.y, acc.y);
    }
    if (!full && wsum && u == 0) wsum[s] = total;
  }
  xhat[idx] = acc;
}

__global__ void fuse_finalize_kernel(float2* __restrict__ xhat, const float* __restrict__ wsum, int S, int U) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(S) * U) return;
  const float w = wsum[idx / U];
  xhat[idx] = make_float2(xhat[idx].x / w, xhat[idx].y / w);
}

template <typename T>
__global__ void gain_reduce_kernel(const float* __restrict__ part, const T* __restrict__ Sy, int S, int C, int U,
                                   float* __restrict__ gain) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= S) return;
  float se = 0.f;
  for (int u = 0; u < U; ++u) {
    const float2 v = ldc(Sy, static_cast<size_t>(s) * U + u);
    se = fmaf(v.y, v.y, fmaf(v.x, v.x, se));
  }
  float num = 0.f;
  for (int c = 0; c < C; ++c) num += part[s * C + c];
  gain[s] = se > 0.f ? num / se : 0.f;
}

template <typename T>
__global__ void power_scale_kernel(T* __restrict__ X, int P, int n, float rho, unsigned long long* __restrict__ status) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (p >= P) return;
  T* x = X + static_cast<size_t>(p) * n;
  float e = 0.f;
  for (int i = lane; i < n; i += 32) {
    const float2 v = ldc(x, i);
    e = fmaf(v.y, v.y, fmaf(v.x, v.x, e));
  }
  e = warp_sum(e);
  if (e == 0.f) {
    if (lane == 0) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
    return;
  }
  const float g = rho / __fsqrt_rn(e);
  for (int i = lane; i < n; i += 32) {
    const float2 v = ldc(x, i);
    stc(x, i, make_float2(v.x * g, v.y * g));
  }
}

__global__ void fusion_weights_kernel(const float* __restrict__ s2, int S, int C, float* __restrict__ w,
                                      unsigned long long* __restrict__ status) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= S) return;
  float total = 0.f;
  bool bad = false;
  for (int c = 0; c < C; ++c) {
    const float v = s2[s * C + c];
    if (!(v > 0.f) || !isfinite(v)) bad = true;
    total += 1.f / v;
  }
  if (bad) record_status(status, s * C, ST_BAD_VARIANCE, 0);
  for (int c = 0; c < C; ++c) w[s * C + c] = (1.f / s2[s * C + c]) / total;
}

__global__ void round_fp16_kernel(float* __restrict__ x, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    x[i] = __half2float(__float2half_rn(x[i]));
}

__global__ void f32_to_f16_kernel(const float* __restrict__ src, __half* __restrict__ dst, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = __float2half_rn(src[i]);
}

__global__ void f16_to_f32_kernel(const __half* __restrict__ src, float* __restrict__ dst, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = __half2float(src[i]);
}

}  // namespace dcdg
