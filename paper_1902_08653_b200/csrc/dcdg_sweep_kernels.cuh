// Device-side batch synthesis and the matched-filter baselines: what a GPU
// BER sweep needs around the CD kernels.
//
// Synthesis restates make_batch + run_uplink_round's observation
// (src/cluster.cpp:80-105,142-145; gen_rayleigh / modulate / awgn,
// src/mimo.cpp:16-26,124-163) with a counter-based generator so every element
// is an independent function of (seed, purpose, trial, index):
//   H_{b,u} ~ CN(0, 1)                   purpose CHANNEL, index b*ceil(U/2) + u/2
//   payload bits of user u (MSB first)   purpose BITS,    index u
//   uplink noise n_b ~ CN(0, N0)         purpose NOISE_UL, index b
//   downlink noise at user u ~ CN(0, N0) purpose NOISE_DL, index u
// with b the global antenna row (cluster c, row i: b = c*B_c + i), so a
// centralized layout (C = 1, B_c = B) sees the same channel as any cluster
// split, and every method and sweep count of a sweep sees identical
// realizations (the harness keys trials by (SNR index, trial) as
// harness.cpp:176 does).  The streams differ from the reference's
// mt19937_64 streams; BER-level results are compared statistically, while the
// bit-exact parity of the detection path itself is tested on the reference's
// own batches.
//
// Philox-4x32-10: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
// easy as 1, 2, 3", SC'11 (the published round function and Weyl constants).
#pragma once

#include "dcdg_aux_kernels.cuh"

namespace dcdg {

enum RngPurposeDev : uint32_t { RNG_CHANNEL = 1, RNG_BITS = 2, RNG_NOISE_UL = 3, RNG_NOISE_DL = 4 };

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ U4 draw(uint64_t seed, uint32_t purpose, uint64_t trial, uint32_t index) {
  return philox4x32_10(U4{index, purpose, static_cast<uint32_t>(trial), static_cast<uint32_t>(trial >> 32)},
                       static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

// Two uniforms in (0, 1) -> one complex normal with E|z|^2 = var (Box-Muller;
// the reference's cgaussian(var) draws N(0, var/2) per axis, rng.cpp).
__device__ __forceinline__ float2 cgauss(uint32_t a, uint32_t b, float var) {
  const float u1 = (static_cast<float>(a) + 0.5f) * 2.3283064365386963e-10f;
  const float u2 = (static_cast<float>(b) + 0.5f) * 2.3283064365386963e-10f;
  const float r = sqrtf(-var * __logf(u1));  // sqrt(-2 ln u1) * sqrt(var/2)
  float sn, cs;
  __sincosf(6.283185307179586f * u2, &sn, &cs);
  return make_float2(r * cs, r * sn);
}

__device__ __forceinline__ unsigned payload_label(uint64_t seed, uint64_t trial, int u, int bps) {
  const uint32_t w = draw(seed, RNG_BITS, trial, static_cast<uint32_t>(u)).x;
  unsigned label = 0;
  for (int k = 0; k < bps; ++k) label = (label << 1) | ((w >> k) & 1u);  // bit k of the symbol = (w >> k) & 1
  return label;
}

// One thread per (subcarrier, global antenna row).  Writes the channel tiles
// [S][C][U][B_c] (column-major per tile), the receive samples y = H x + n
// [S][C][B_c] (Y may be NULL), and for rows b < U the payload bits of user b
// [S][U*bps] (one byte per bit, MSB first), the transmitted symbol [S][U]
// (SYM may be NULL) and the downlink receiver noise [S][U] (NDL may be NULL).
__global__ void __launch_bounds__(256) synth_kernel(int S, int C, int BC, int U, uint64_t seed, uint64_t first_trial,
                                                    float n0, unsigned order, double ex, float2* __restrict__ H,
                                                    float2* __restrict__ Y, uint8_t* __restrict__ bits,
                                                    float2* __restrict__ SYM, float2* __restrict__ NDL) {
  __shared__ Qam q;
  __shared__ float lv[8];
  if (threadIdx.x == 0) {
    q = make_qam(order, ex);
    for (int i = 0; i < q.levels; ++i) lv[i] = static_cast<float>(q.level[i]);
  }
  __syncthreads();
  const int B = C * BC, bps = 2 * q.axis_bits, UH = (U + 1) / 2;
  const long long n = static_cast<long long>(S) * B;
  for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long s = idx / B;
    const int b = static_cast<int>(idx - s * B);
    const int c = b / BC, i = b - c * BC;
    const uint64_t trial = first_trial + static_cast<uint64_t>(s);
    float2 acc = make_float2(0.f, 0.f);
    float2* hcol = H + (static_cast<size_t>(s) * C + c) * U * BC + i;
    for (int jp = 0; jp < UH; ++jp) {
      const U4 r = draw(seed, RNG_CHANNEL, trial, static_cast<uint32_t>(b * UH + jp));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * jp + h;
        if (j >= U) break;
        const float2 hv = h ? cgauss(r.z, r.w, 1.f) : cgauss(r.x, r.y, 1.f);
        hcol[static_cast<size_t>(j) * BC] = hv;
        if (Y) {
          const unsigned lab = payload_label(seed, trial, j, bps);
          const float xr = lv[lab >> q.axis_bits], xi = lv[lab & (q.levels - 1)];
          acc.x = fmaf(hv.x, xr, fmaf(-hv.y, xi, acc.x));
          acc.y = fmaf(hv.x, xi, fmaf(hv.y, xr, acc.y));
        }
      }
    }
    if (Y) {
      const U4 r = draw(seed, RNG_NOISE_UL, trial, static_cast<uint32_t>(b));
      const float2 nv = cgauss(r.x, r.y, n0);
      Y[(static_cast<size_t>(s) * C + c) * BC + i] = make_float2(acc.x + nv.x, acc.y + nv.y);
    }
    if (b < U) {
      const uint32_t w = draw(seed, RNG_BITS, trial, static_cast<uint32_t>(b)).x;
      unsigned lab = 0;
      for (int k = 0; k < bps; ++k) {
        const unsigned bit = (w >> k) & 1u;
        bits[(static_cast<size_t>(s) * U + b) * bps + k] = static_cast<uint8_t>(bit);
        lab = (lab << 1) | bit;
      }
      if (SYM) SYM[static_cast<size_t>(s) * U + b] = make_float2(lv[lab >> q.axis_bits], lv[lab & (q.levels - 1)]);
      if (NDL) {
        const U4 r = draw(seed, RNG_NOISE_DL, trial, static_cast<uint32_t>(b));
        NDL[static_cast<size_t>(s) * U + b] = cgauss(r.x, r.y, n0);
      }
    }
  }
}

// Matched-filter uplink baseline (mf_detect, detect.cpp:191-218), one warp per
// subcarrier, lane u: x_u = sum_c h_cu^H y_c / sum_c ||h_cu||^2.
__global__ void __launch_bounds__(128) mf_detect_kernel(const float2* __restrict__ H, const float2* __restrict__ Y,
                                                        int S, int C, int BC, int U, float2* __restrict__ X,
                                                        unsigned long long* __restrict__ status) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long s = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (s >= S || lane >= U) return;
  float cr = 0.f, ci = 0.f, e = 0.f;
  for (int c = 0; c < C; ++c) {
    const float2* h = H + ((static_cast<size_t>(s) * C + c) * U + lane) * BC;
    const float2* y = Y + (static_cast<size_t>(s) * C + c) * BC;
    float pr = 0.f, pi = 0.f, pe = 0.f;  // per-cluster partials, summed in cluster order as the reference
    for (int i = 0; i < BC; ++i) {
      const float2 hv = __ldg(h + i), yv = __ldg(y + i);
      pr = fmaf(hv.x, yv.x, fmaf(hv.y, yv.y, pr));
      pi = fmaf(hv.x, yv.y, fmaf(-hv.y, yv.x, pi));
      pe = fmaf(hv.x, hv.x, fmaf(hv.y, hv.y, pe));
    }
    cr += pr;
    ci += pi;
    e += pe;
  }
  if (e == 0.f) record_status(status, s, ST_MF_ZERO_ENERGY, lane);
  X[static_cast<size_t>(s) * U + lane] = make_float2(cr / e, ci / e);
}

// Matched-filter downlink baseline (mf_precode, precode.cpp:171-202), one
// warp per (subcarrier, cluster): x_c = rho_c v / ||v||, v = H_c s (the
// cluster's conjugate-transposed downlink block applied to s).
__global__ void __launch_bounds__(128) mf_precode_kernel(const float2* __restrict__ H, const float2* __restrict__ Sy,
                                                         int P, int C, int BC, int U, float rho_c,
                                                         float2* __restrict__ X, unsigned long long* __restrict__ status) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (p >= P) return;
  const float2* h = H + static_cast<size_t>(p) * U * BC;
  const float2* sv = Sy + static_cast<size_t>(p / C) * U;
  float2* x = X + static_cast<size_t>(p) * BC;
  float e = 0.f;
  for (int i = lane; i < BC; i += 32) {
    float vr = 0.f, vi = 0.f;
    for (int u = 0; u < U; ++u) {
      const float2 hv = __ldg(h + static_cast<size_t>(u) * BC + i), su = __ldg(sv + u);
      vr = fmaf(hv.x, su.x, fmaf(-hv.y, su.y, vr));
      vi = fmaf(hv.x, su.y, fmaf(hv.y, su.x, vi));
    }
    x[i] = make_float2(vr, vi);
    e = fmaf(vr, vr, fmaf(vi, vi, e));
  }
  e = warp_sum(e);
  if (e == 0.f) {
    if (lane == 0) record_status(status, p, ST_MF_ZERO_BEAMFORMER, static_cast<uint32_t>(p % C));
    return;
  }
  const float g = rho_c / __fsqrt_rn(e);
  for (int i = lane; i < BC; i += 32) {
    const float2 v = x[i];
    x[i] = make_float2(v.x * g, v.y * g);
  }
}

}  // namespace dcdg
