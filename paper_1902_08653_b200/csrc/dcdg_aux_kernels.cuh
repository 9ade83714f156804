// Generic (any-shape) CD kernels, the post-equalization variance, fusion,
// gain reduction, power scaling and format conversion kernels.
#pragma once

#include "dcdg_device.cuh"

namespace dcdg {

// ===========================================================================
// Generic kernels: any B_c, U (one warp per problem, fp32 math).  Used for
// shapes without a register-resident specialisation and for fp16 shapes
// whose B_c is not a multiple of 4G.  Residual / beamformer and scalars live
// in shared memory; lane l owns rows l, l+32, ...
// ===========================================================================
//
// TRACE (the SweepObserver debug path, detect.hpp:28-36): after every
// coordinate update of problem 0 the iterate x and the residual r are dumped
// to xt[(t U + j) U ..] and rt[(t U + j) B_c ..] (fp32 complex), the values the
// reference hands to observer->after_update (detect.cpp:106, precode.cpp:95).
template <typename T, bool TRACE = false>
__global__ void __launch_bounds__(128) ul_generic(const T* __restrict__ H, const T* __restrict__ Y, int P, int BC,
                                                  int U, int K, float kappa, T* __restrict__ X,
                                                  float2* __restrict__ xt = nullptr, float2* __restrict__ rt = nullptr) {
  extern __shared__ float2 gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (p >= P) return;
  float2* r = gsm + warp * (BC + 2 * U);
  float2* x = r + BC;
  float2* mn = x + U;
  const T* h = H + static_cast<size_t>(p) * BC * U;
  for (int i = lane; i < BC; i += 32) r[i] = ldv(Y + static_cast<size_t>(p) * BC, i);
  for (int j = 0; j < U; ++j) {
    float e = 0.f;
    for (int i = lane; i < BC; i += 32) {
      const float2 v = ldv(h + static_cast<size_t>(j) * BC, i);
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
        const float2 hv = ldv(h + static_cast<size_t>(j) * BC, i);
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
        const float2 hv = ldv(h + static_cast<size_t>(j) * BC, i);
        float2 rv = r[i];
        rv.x = fmaf(-dxr, hv.x, fmaf(dxi, hv.y, rv.x));
        rv.y = fmaf(-dxr, hv.y, fmaf(-dxi, hv.x, rv.y));
        r[i] = rv;
      }
      __syncwarp();
      if (TRACE && p == 0) {
        const size_t e = static_cast<size_t>(t) * U + j;
        for (int i = lane; i < U; i += 32) xt[e * U + i] = x[i];
        for (int i = lane; i < BC; i += 32) rt[e * BC + i] = r[i];
      }
    }
  for (int j = lane; j < U; j += 32) stc(X, static_cast<size_t>(p) * U + j, x[j]);
}

// TRACE: the beamformer x after every update of problem 0 to xt[(t U + j) B_c ..]
// (precode.cpp:95 hands the observer x and an empty residual).
template <typename T, bool GAIN, bool TRACE = false>
__global__ void __launch_bounds__(128)
    dl_generic(const T* __restrict__ H, const T* __restrict__ Sy, int P, int C, int BC, int U, int K, float rho_c,
               T* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status,
               float2* __restrict__ xt = nullptr) {
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
      const float2 v = ldv(h + static_cast<size_t>(j) * BC, i);
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
        float2 hv = ldv(h + static_cast<size_t>(j) * BC, i);
        hv.x *= pj;
        hv.y *= pj;
        const float2 xv = x[i];
        dr = fmaf(hv.x, xv.x, fmaf(hv.y, xv.y, dr));
        di = fmaf(hv.x, xv.y, fmaf(-hv.y, xv.x, di));
      }
      dr = warp_sum(dr) - sb[j].x;
      di = warp_sum(di) - sb[j].y;
      for (int i = lane; i < BC; i += 32) {
        float2 hv = ldv(h + static_cast<size_t>(j) * BC, i);
        hv.x *= pj;
        hv.y *= pj;
        float2 xv = x[i];
        xv.x = fmaf(-dr, hv.x, fmaf(di, hv.y, xv.x));
        xv.y = fmaf(-dr, hv.y, fmaf(-di, hv.x, xv.y));
        x[i] = xv;
        if (TRACE && p == 0) xt[(static_cast<size_t>(t) * U + j) * BC + i] = xv;  // each lane its own rows
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
        const float2 hv = ldv(h + static_cast<size_t>(j) * BC, i);
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
// The Gram is computed from row chunks of the tile staged in shared memory
// (column stride PR+1 complex: conflict-free), each lane accumulating a 4x2
// block of entries with packed FFMA2 (rows broadcast, columns pre-swapped).
// Shared memory per warp: staged chunk [U][PR+1] + A/L [U][U] + Z [U][U]
// complex fp32 (U <= 32).
// ===========================================================================
constexpr int kPevRows = 32;  // rows staged per chunk

__host__ __device__ constexpr int pev_smem_per_warp(int U) {
  return (U * (kPevRows + 1) + 2 * U * U) * 8;
}

// One warp per problem; MODE selects what the Gram/Cholesky serves:
//   kPev  (post_eq_variance, detect.cpp:112-130): one tile per problem,
//         A = I + gam*G, out[p] = scale * tr(A^-1);
//   kBias (mmse_bias_factors, detect.cpp:227-242): the NT = C cluster tiles of a
//         subcarrier stacked (full-H Gram), A = kappa*I + G,
//         out[p*U + u] = 1 - kappa * [A^-1]_uu.
// UT > 0: U == UT at compile time (register-resident Cholesky/inverse);
// BT > 0: B_c == BT at compile time (vectorised staging, unrolled Gram).
//   kSolve (lmmse_exact, detect.cpp:54-65): NT stacked tiles, A = kappa*I + G,
//         x = A^-1 H^H y by forward/back substitution, xo[p*U + u];
//   kZf   (zf_exact + power_scale, precode.cpp:31-50,101-111): A = G,
//         w = A^-1 s, x = H w over the NT tiles scaled to ||x|| = scale,
//         xo[(p*NT + t)*B_c + i].
enum GramMode { kPev = 0, kBias = 1, kSolve = 2, kZf = 3 };

// Cholesky solve A w = b with L in shared memory (Lat(i, k) = L_ik, real
// diagonal): lane i < U holds b_i on entry and returns w_i.  Column-oriented
// forward (L z = b) and back (L^H w = z) substitution, one broadcast per step.
template <typename LF>
__device__ __forceinline__ float2 chol_solve(LF Lat, float2 bi, int U, int lane) {
  float2 zi = make_float2(0.f, 0.f);
  for (int j = 0; j < U; ++j) {
    const float ljj = Lat(j, j).x;
    const float2 zj = make_float2(__shfl_sync(0xffffffffu, bi.x, j) / ljj, __shfl_sync(0xffffffffu, bi.y, j) / ljj);
    if (lane == j) zi = zj;
    if (lane > j && lane < U) {  // b_i -= L_ij z_j
      const float2 l = Lat(lane, j);
      bi.x -= l.x * zj.x - l.y * zj.y;
      bi.y -= l.x * zj.y + l.y * zj.x;
    }
  }
  float2 wi = make_float2(0.f, 0.f);
  for (int j = U - 1; j >= 0; --j) {
    const float ljj = Lat(j, j).x;
    const float2 wj = make_float2(__shfl_sync(0xffffffffu, zi.x, j) / ljj, __shfl_sync(0xffffffffu, zi.y, j) / ljj);
    if (lane == j) wi = wj;
    if (lane < j) {  // z_i -= conj(L_ji) w_j
      const float2 l = Lat(j, lane);
      zi.x -= l.x * wj.x + l.y * wj.y;
      zi.y -= l.x * wj.y - l.y * wj.x;
    }
  }
  return wi;
}

// Right-hand side and output stage of the solve modes (after the Cholesky).
template <typename T, int MODE, typename LF>
__device__ __forceinline__ void solve_emit(LF Lat, const T* __restrict__ H, const T* __restrict__ V, long long p, int NT,
                                           int BC, int U, float scale, bool singular, float2* __restrict__ xo,
                                           unsigned long long* __restrict__ status, int lane) {
  float2 b = make_float2(0.f, 0.f);
  if (lane < U) {
    if (MODE == kSolve) {  // b_u = sum_t h_tu^H y_t   (cdotc, detect.cpp:61-63)
      for (int t = 0; t < NT; ++t) {
        const T* h = H + ((static_cast<size_t>(p) * NT + t) * U + lane) * BC;
        const T* y = V + (static_cast<size_t>(p) * NT + t) * BC;
        for (int i = 0; i < BC; ++i) {
          const float2 hv = ldv(h, i), yv = ldv(y, i);
          b.x = fmaf(hv.x, yv.x, fmaf(hv.y, yv.y, b.x));
          b.y = fmaf(hv.x, yv.y, fmaf(-hv.y, yv.x, b.y));
        }
      }
    } else {
      b = ldc(V, static_cast<size_t>(p) * U + lane);
    }
  }
  const float2 w = chol_solve(Lat, b, U, lane);
  if (singular && lane == 0) record_status(status, p, MODE == kSolve ? ST_SINGULAR : ST_RANK_DEFICIENT, 0);
  if (MODE == kSolve) {
    if (lane < U) xo[static_cast<size_t>(p) * U + lane] = w;
    return;
  }
  // x = H w (x_i = sum_u H_iu w_u, precode.cpp:45-48), then power_scale
  float e = 0.f;
  for (int t = 0; t < NT; ++t) {
    const T* h = H + (static_cast<size_t>(p) * NT + t) * U * BC;
    float2* x = xo + (static_cast<size_t>(p) * NT + t) * BC;
    for (int i0 = 0; i0 < BC; i0 += 32) {
      const int i = i0 + lane;
      float xr = 0.f, xi = 0.f;
      for (int u = 0; u < U; ++u) {
        const float wr = __shfl_sync(0xffffffffu, w.x, u), wi = __shfl_sync(0xffffffffu, w.y, u);
        if (i < BC) {
          const float2 hv = ldv(h + static_cast<size_t>(u) * BC, i);
          xr = fmaf(hv.x, wr, fmaf(-hv.y, wi, xr));
          xi = fmaf(hv.x, wi, fmaf(hv.y, wr, xi));
        }
      }
      if (i < BC) {
        x[i] = make_float2(xr, xi);
        e = fmaf(xr, xr, fmaf(xi, xi, e));
      }
    }
  }
  if (scale <= 0.f) return;  // raw zf_exact beamformer (no power_scale)
  e = warp_sum(e);
  if (e == 0.f) {
    if (lane == 0 && !singular) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
    return;
  }
  const float g = scale / __fsqrt_rn(e);  // power_scale(x, rho), precode.cpp:101-111
  for (int t = 0; t < NT; ++t) {
    float2* x = xo + (static_cast<size_t>(p) * NT + t) * BC;
    for (int i = lane; i < BC; i += 32) {
      const float2 v = x[i];
      x[i] = make_float2(v.x * g, v.y * g);
    }
  }
}

// (the solve modes return after the Cholesky; the inverse that follows is
// dead code in those instantiations)
#pragma nv_diag_suppress 128
template <typename T, int UT, int BT, int MODE>
__global__ void __launch_bounds__(128) gram_chol(const T* __restrict__ H, int P, int NT, int BC_, int U_, float a0,
                                                 float a1, float scale, bool round_fp16, float* __restrict__ out,
                                                 unsigned long long* __restrict__ status,
                                                 const T* __restrict__ V = nullptr, float2* __restrict__ xo = nullptr) {
  extern __shared__ float2 vsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (p >= P) return;
  const int BC = BT > 0 ? BT : BC_;
  const int U = UT > 0 ? UT : U_;
  constexpr int PR = kPevRows;
  float2* Hs = vsm + warp * (U * (PR + 1) + 2 * U * U);  // staged rows, column-major, stride PR+1
  float2* A = Hs + U * (PR + 1);                          // column-major, lower triangle used
  float2* Z = A + U * U;
  // 4x2 entry blocks: block id = lane + 32t, (ib, jb) = (id / njb, id % njb)
  const int nib = (U + 3) / 4, njb = (U + 1) / 2, nblk = nib * njb;
  float2 acc[4][4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[t][r][0] = acc[t][r][1] = make_float2(0.f, 0.f);
  for (int tile = 0; tile < NT; ++tile) {
  const T* h = H + (static_cast<size_t>(p) * NT + tile) * BC * U;
  for (int b0 = 0; b0 < BC; b0 += PR) {
    const int rows = min(PR, BC - b0);
    if (BT == PR && sizeof(T) == 8) {
      // whole fp32 tile in one chunk: 16-B loads, two rows per load
      const float4* t4 = reinterpret_cast<const float4*>(h);
#pragma unroll
      for (int i = 0; i < (BT > 0 ? BT * (UT > 0 ? UT : 1) / 64 : 1); ++i) {
        const int idx = lane + 32 * i;
        const int j = idx / (PR / 2), rr = idx - j * (PR / 2);
        const float4 v = __ldg(t4 + idx);
        Hs[j * (PR + 1) + 2 * rr] = make_float2(v.x, v.y);
        Hs[j * (PR + 1) + 2 * rr + 1] = make_float2(v.z, v.w);
      }
    } else {
      for (int idx = lane; idx < rows * U; idx += 32) {
        const int j = idx / rows, b = idx - j * rows;
        Hs[j * (PR + 1) + b] = ldv(h + static_cast<size_t>(j) * BC, b0 + b);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int id = lane + 32 * t;
      if (id < nblk) {
        const int i0 = 4 * (id / njb), j0 = 2 * (id % njb);
#pragma unroll 8
        for (int b = 0; b < (BT == PR ? PR : rows); ++b) {
          float2 a[4], c[2], cs[2];
#pragma unroll
          for (int r = 0; r < 4; ++r) a[r] = (i0 + r < U) ? Hs[(i0 + r) * (PR + 1) + b] : make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            c[q] = (j0 + q < U) ? Hs[(j0 + q) * (PR + 1) + b] : make_float2(0.f, 0.f);
            cs[q] = make_float2(c[q].y, -c[q].x);
          }
          // conj(a) c = a.x (c.x, c.y) + a.y (c.y, -c.x)
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 2; ++q) acc[t][r][q] = ffma2(a[r].y, cs[q], ffma2(a[r].x, c[q], acc[t][r][q]));
        }
      }
    }
    __syncwarp();
  }
  }  // tiles
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int id = lane + 32 * t;
    if (id < nblk) {
      const int i0 = 4 * (id / njb), j0 = 2 * (id % njb);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int i = i0 + r, j = j0 + q;
          if (i < U && j < U && i >= j)  // A = a0 I + a1 G
            A[j * U + i] = make_float2((i == j ? a0 : 0.f) + a1 * acc[t][r][q].x, a1 * acc[t][r][q].y);
        }
    }
  }
  __syncwarp();
  float maxdiag = 0.f;  // numerics.cpp:38-41 (pivot floor 1e-14 * max |A_jj|)
  for (int j = lane; j < U; j += 32) maxdiag = fmaxf(maxdiag, fabsf(A[j * U + j].x));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) maxdiag = fmaxf(maxdiag, __shfl_xor_sync(0xffffffffu, maxdiag, o));
  // The reference's floor is ~45 fp64 ulps of the largest pivot.  The
  // regularised Grams (kPev, kBias, kSolve: A = a0 I + a1 G, positive definite
  // by construction) keep it; the unregularised ZF Gram takes the same 45 ulps
  // in fp32, where an exactly rank-deficient G leaves a ~1e-7 rounding residue.
  const float floor_ = (MODE == kZf ? 45.f * 1.1920929e-7f : 1e-14f) * maxdiag;
  bool singular = false;
  float tr = 0.f;
  if (UT > 0) {
    // Register-resident path (U == UT): lane i holds row i of A and of L;
    // finished rows of L are published row-major in Z for broadcast reads.
    constexpr int N = UT > 0 ? UT : 1;
    float2 a[N], l[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      a[k] = (lane < N && k <= lane) ? A[k * N + lane] : make_float2(0.f, 0.f);
      l[k] = make_float2(0.f, 0.f);
    }
    float2* Lr = Z;  // row-major L
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (lane == j) {  // d_j = A_jj - sum_k |L_jk|^2 ; L_jj = sqrt(d_j)   (numerics.cpp:47-52)
        float d = a[j].x;
#pragma unroll
        for (int k = 0; k < j; ++k) d -= l[k].x * l[k].x + l[k].y * l[k].y;
        if (!(d > floor_)) singular = true;
        l[j] = make_float2(__fsqrt_rn(fmaxf(d, 1e-30f)), 0.f);
#pragma unroll
        for (int k = 0; k <= j; ++k) Lr[j * N + k] = l[k];
      }
      __syncwarp();
      if (lane > j && lane < N) {  // L_ij = (A_ij - sum_{k<j} L_ik conj(L_jk)) / L_jj   (numerics.cpp:53-56)
        float sr = a[j].x, si = a[j].y;
#pragma unroll
        for (int k = 0; k < j; ++k) {
          const float2 b = Lr[j * N + k];
          sr -= l[k].x * b.x + l[k].y * b.y;
          si -= l[k].y * b.x - l[k].x * b.y;
        }
        const float inv = __frcp_rn(Lr[j * N + j].x);
        l[j] = make_float2(sr * inv, si * inv);
      }
    }
    __syncwarp();
    singular = __any_sync(0xffffffffu, singular);  // pivot j was tested by lane j only
    if constexpr (MODE >= kSolve) {  // Lr holds every row of L (row j published at step j)
      solve_emit<T, MODE>([&](int i, int k) { return Lr[i * N + k]; }, H, V, p, NT, BC, U, scale, singular, xo,
                          status, lane);
      return;
    }
    // X = L^{-1}: lane c holds column c; row i: X_ic = -(sum_{k=c}^{i-1} L_ik X_kc) / L_ii
    float2 x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float linv = __frcp_rn(Lr[i * N + i].x);
      float sr = 0.f, si = 0.f;
#pragma unroll
      for (int k = 0; k < i; ++k) {
        const float2 lk = Lr[i * N + k];
        const float2 xk = x[k];  // zero above the diagonal (k < c)
        sr += lk.x * xk.x - lk.y * xk.y;
        si += lk.x * xk.y + lk.y * xk.x;
      }
      float2 xi;
      if (lane == i) xi = make_float2(linv, 0.f);
      else if (lane < i) xi = make_float2(-sr * linv, -si * linv);
      else xi = make_float2(0.f, 0.f);
      x[i] = xi;
      tr = fmaf(xi.x, xi.x, fmaf(xi.y, xi.y, tr));
    }
  } else {
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
  if constexpr (MODE >= kSolve) {
    solve_emit<T, MODE>([&](int i, int k) { return A[k * U + i]; }, H, V, p, NT, BC, U, scale, singular, xo, status,
                        lane);
    return;
  }
  // columns of L^-1: lane c solves L z = e_c (rows i >= c)
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
  }
  if (MODE == kBias) {  // lane u holds [A^-1]_uu = ||column u of L^-1||^2
    if (lane < U) out[p * U + lane] = 1.f - a0 * tr;
    if (lane == 0 && singular) record_status(status, p, ST_SINGULAR, 0);
    return;
  }
  tr = warp_sum(tr);
  if (lane == 0) {
    float s2 = scale * tr;
    if (round_fp16) s2 = __half2float(__float2half_rn(s2));
    out[p] = s2;
    if (singular) record_status(status, p, ST_SINGULAR, 0);
  }
}

// ===========================================================================
// Post-equalization variance for U = 16, two problems per warp (optimal
// fusion, detect.cpp:112-130).  The Gram of each problem uses the whole warp
// (lane = one 4x2 block of the 16x16 Gram, tiles staged in shared memory as in
// gram_chol); the factorisation then runs both problems at once, one half-warp
// each: lane (h, i) holds row i of A_h in registers, the left-looking Cholesky
// publishes finished rows of L_h row-major in shared memory, and lane (h, c)
// accumulates column c of L_h^{-1} (tr A^-1 = ||L^-1||_F^2, summed over the
// half).  gram_chol's factorisation keeps half the warp idle at U = 16; here
// every lane works, so the scalar Cholesky/inverse stream serves two problems.
// ===========================================================================
#ifndef DCDG_PEV_SWEEP  // factorisation: 1 = sweep operator, 0 = Cholesky + triangular inverse
#define DCDG_PEV_SWEEP 0  // lab switch: the sweep operator measured slower here (profiles/lab/README.md)
#endif
#ifndef DCDG_PEV_TRI  // lower-triangle-only Gram (lab switch: measured slower for fp32, see below)
#define DCDG_PEV_TRI 0
#endif
template <typename T, int BT>
__global__ void __launch_bounds__(128) pev16_pair_kernel(const T* __restrict__ H, int P, float gam, float scale,
                                                         bool round_fp16, float* __restrict__ out,
                                                         unsigned long long* __restrict__ status) {
  constexpr int N = 16, PR = BT;  // users, staged rows
  extern __shared__ float2 psm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2* Hs = psm + warp * (2 * N * (PR + 1) + 2 * N * N);  // 2 staged tiles, column stride PR+1
  float2* A = Hs + 2 * N * (PR + 1);                        // 2 x [16][16] column-major (lower used)
  float2* Lr = Hs;                                          // 2 x [16][16] row-major L, over the tiles
  const long long p0 = (static_cast<long long>(blockIdx.x) * 4 + warp) * 2;
  if (p0 >= P) return;
  // ---- stage both tiles (the second clamped to P-1 when P is odd)
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const long long p = min(p0 + t, static_cast<long long>(P) - 1);
    const T* h = H + static_cast<size_t>(p) * BT * N;
    float2* hs = Hs + t * N * (PR + 1);
    if constexpr (sizeof(T) == 8 && BT % 2 == 0) {
      const float4* t4 = reinterpret_cast<const float4*>(h);
#pragma unroll
      for (int i = 0; i < BT * N / 64; ++i) {
        const int idx = lane + 32 * i;
        const int j = idx / (BT / 2), rr = idx - j * (BT / 2);
        const float4 v = __ldg(t4 + idx);
        hs[j * (PR + 1) + 2 * rr] = make_float2(v.x, v.y);
        hs[j * (PR + 1) + 2 * rr + 1] = make_float2(v.z, v.w);
      }
    } else if constexpr (sizeof(T) == 4 && BT % 4 == 0) {
      // fp16 row-pair planar tile: one 16-B load = rows 4q..4q+3 of a column
      // as {re0, re1, im0, im1, re2, re3, im2, im3}
      const uint4* t4 = reinterpret_cast<const uint4*>(h);
#pragma unroll
      for (int i = 0; i < BT * N / 128; ++i) {
        const int idx = lane + 32 * i;
        const int j = idx / (BT / 4), q = idx - j * (BT / 4);
        const uint4 v = __ldg(t4 + idx);
        const float2 re01 = __half22float2(u32_as_h2(v.x)), im01 = __half22float2(u32_as_h2(v.y));
        const float2 re23 = __half22float2(u32_as_h2(v.z)), im23 = __half22float2(u32_as_h2(v.w));
        float2* dst = hs + j * (PR + 1) + 4 * q;
        dst[0] = make_float2(re01.x, im01.x);
        dst[1] = make_float2(re01.y, im01.y);
        dst[2] = make_float2(re23.x, im23.x);
        dst[3] = make_float2(re23.y, im23.y);
      }
    } else {
      for (int idx = lane; idx < BT * N; idx += 32) {
        const int j = idx / BT, b = idx - j * BT;
        hs[j * (PR + 1) + b] = ldv(h + static_cast<size_t>(j) * BT, b);
      }
    }
  }
  __syncwarp();
#if DCDG_PEV_TRI
  // ---- Grams, lower triangles only (detect.cpp:118-121 reads i >= j): both
  // problems at once.  Lanes 0-23: half of an off-diagonal 4x4 block (4x2,
  // 6 blocks per problem); lanes 24-31: the left 4x2 of a diagonal 4x4 block;
  // lanes 0-7 also the bottom-right 2x2 of a diagonal block.  24 FFMA2 per
  // staged row on the busiest lanes instead of 2 x 16 for two full Grams.
  // Bitwise-identical variances, but 0.452 vs 0.428 ms (fp32) and 0.421 vs
  // 0.427 ms (fp16) per 134 400 problems: the factorisation chain, not the
  // Gram, bounds this kernel, and the mixed-problem loads conflict in banks.
  {
    constexpr int kOffI[6] = {1, 2, 2, 3, 3, 3}, kOffJ[6] = {0, 0, 1, 0, 1, 2};
    int t1, i1, j1;
    if (lane < 24) {
      const int idx = lane % 12, bp = idx >> 1;
      t1 = lane / 12;
      i1 = 4 * kOffI[bp];
      j1 = 4 * kOffJ[bp] + 2 * (idx & 1);
    } else {
      t1 = (lane - 24) >> 2;
      i1 = j1 = 4 * ((lane - 24) & 3);
    }
    const int t2 = (lane & 7) >> 2, d2 = 4 * (lane & 3) + 2;  // 2x2 unit (rows/cols d2, d2+1) of problem t2
    const float2* h1 = Hs + t1 * N * (PR + 1);
    const float2* h2 = Hs + t2 * N * (PR + 1);
    float2 pa[4][2], qa[4][2], pb[2][2], qb[2][2];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q) pa[r][q] = qa[r][q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q) pb[r][q] = qb[r][q] = make_float2(0.f, 0.f);
#pragma unroll 8
    for (int b = 0; b < PR; ++b) {
      float2 a[4], c[2], a2[2];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = h1[(i1 + r) * (PR + 1) + b];
#pragma unroll
      for (int q = 0; q < 2; ++q) c[q] = h1[(j1 + q) * (PR + 1) + b];
#pragma unroll
      for (int r = 0; r < 2; ++r) a2[r] = h2[(d2 + r) * (PR + 1) + b];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          pa[r][q] = ffma2(a[r].x, c[q], pa[r][q]);
          qa[r][q] = ffma2(a[r].y, c[q], qa[r][q]);
        }
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          pb[r][q] = ffma2(a2[r].x, a2[q], pb[r][q]);
          qb[r][q] = ffma2(a2[r].y, a2[q], qb[r][q]);
        }
    }
    float2* A1 = A + t1 * N * N;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int i = i1 + r, j = j1 + q;
        const float gr = pa[r][q].x + qa[r][q].y, gi = pa[r][q].y - qa[r][q].x;
        if (i >= j) A1[j * N + i] = make_float2((i == j ? 1.f : 0.f) + gam * gr, gam * gi);
      }
    if (lane < 8) {
      float2* A2 = A + t2 * N * N;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int q = 0; q <= r; ++q) {
          const int i = d2 + r, j = d2 + q;
          const float gr = pb[r][q].x + qb[r][q].y, gi = pb[r][q].y - qb[r][q].x;
          A2[j * N + i] = make_float2((i == j ? 1.f : 0.f) + gam * gr, gam * gi);
        }
    }
  }
#else
  // ---- Grams: lane -> 4x2 block (rows 4*ib.., columns 2*jb..) of G_t; A_t = I + gam G_t
  const int i0 = 4 * (lane >> 3), j0 = 2 * (lane & 7);
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const float2* hs = Hs + t * N * (PR + 1);
    // conj(a) c = (a.x c.x + a.y c.y, a.x c.y - a.y c.x): accumulate
    // P = sum a.x (c.x, c.y) and Q = sum a.y (c.x, c.y), combine once per entry
    float2 pa[4][2], qa[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q) pa[r][q] = qa[r][q] = make_float2(0.f, 0.f);
#pragma unroll 8
    for (int b = 0; b < PR; ++b) {
      float2 a[4], c[2];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = hs[(i0 + r) * (PR + 1) + b];
#pragma unroll
      for (int q = 0; q < 2; ++q) c[q] = hs[(j0 + q) * (PR + 1) + b];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          pa[r][q] = ffma2(a[r].x, c[q], pa[r][q]);
          qa[r][q] = ffma2(a[r].y, c[q], qa[r][q]);
        }
    }
    float2* At = A + t * N * N;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int i = i0 + r, j = j0 + q;
        const float gr = pa[r][q].x + qa[r][q].y, gi = pa[r][q].y - qa[r][q].x;
        if (i >= j)  // detect.cpp:118-121
          At[j * N + i] = make_float2((i == j ? 1.f : 0.f) + gam * gr, gam * gi);
      }
  }
#endif
  __syncwarp();  // the staged tiles are dead from here: Lr reuses their space
#if DCDG_PEV_SWEEP
  // ---- tr A^-1 by the sweep operator, half-warp h = problem p0 + h, lane i =
  // row i of A (full Hermitian row, upper part conj of the stored lower part).
  // Pivot kk in ascending order, its row broadcast through shared memory as
  // (a_kk,j, i a_kk,j) pairs:  d = a_kk,kk;  a_ij -= (a_i,kk / d) a_kk,j;
  // a_i,kk <- a_i,kk / d;  a_kk,j <- a_kk,j / d;  a_kk,kk <- -1/d.  After the
  // 16 pivots the rows hold -A^-1.  The pivots are the Cholesky pivots of
  // hermitian_solve, so the reference's singularity test applies unchanged
  // (numerics.cpp:38-41,55-56); every update is independent (no dot-product
  // chains), two FFMA2 per complex update.
  const int hf = lane >> 4, i = lane & 15;
  const float2* Ah = A + hf * N * N;
  float4* prow = reinterpret_cast<float4*>(Lr) + hf * 2 * N;  // 2 alternating rows of N (a, i a) pairs
  float2 a[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float2 v = (j <= i) ? Ah[j * N + i] : Ah[i * N + j];
    a[j] = (j <= i) ? v : make_float2(v.x, -v.y);
  }
  float maxdiag = 0.f;
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (i == j) maxdiag = fabsf(a[j].x);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) maxdiag = fmaxf(maxdiag, __shfl_xor_sync(0xffffffffu, maxdiag, o));
  const float floor_ = 1e-14f * maxdiag;  // numerics.cpp:38-41,55-56
  bool singular = false;
  __syncwarp();  // every lane has its row: the staged tiles' space now carries the pivot rows
#pragma unroll
  for (int kk = 0; kk < N; ++kk) {
    float4* slot = prow + (kk & 1) * N;
    if (i == kk) {
#pragma unroll
      for (int j = 0; j < N; ++j) slot[j] = make_float4(a[j].x, a[j].y, -a[j].y, a[j].x);
    }
    __syncwarp();
    const float d = slot[kk].x;
    if (!(d > floor_)) singular = true;
    const float inv = __frcp_rn(d);
    const bool piv = (i == kk);
    const float2 f = piv ? make_float2(1.f - inv, 0.f) : fmul2(inv, a[kk]);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (j == kk) continue;
      const float4 v = slot[j];
      a[j] = ffma2(-f.x, make_float2(v.x, v.y), a[j]);
      a[j] = ffma2(-f.y, make_float2(v.z, v.w), a[j]);
    }
    a[kk] = piv ? make_float2(-inv, 0.f) : f;
  }
  float tr = 0.f;
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (i == j) tr = -a[j].x;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
#else
  // ---- factorisation, half-warp h = problem p0 + h, lane i = row i
  const int hf = lane >> 4, i = lane & 15;
  const float2* Ah = A + hf * N * N;
  float2* Lh = Lr + hf * N * N;
  float maxdiag = fabsf(Ah[i * N + i].x);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) maxdiag = fmaxf(maxdiag, __shfl_xor_sync(0xffffffffu, maxdiag, o));
  const float floor_ = 1e-14f * maxdiag;  // numerics.cpp:38-41,55-56
  // complex products in packed fp32x2: u conj(b) = b.x (u.x, u.y) + b.y (u.y, -u.x)
  // and L x = L.x (x.x, x.y) + L.y (-x.y, x.x), with the swizzled copies kept
  // next to each register value (lw, xw) and the shared-memory operand broadcast
  float2 a[N], l[N], lw[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    a[k] = (k <= i) ? Ah[k * N + i] : make_float2(0.f, 0.f);
    l[k] = lw[k] = make_float2(0.f, 0.f);
  }
  bool singular = false;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    if (i == j) {  // d_j = A_jj - sum_k |L_jk|^2 ; L_jj = sqrt(d_j)   (numerics.cpp:47-52)
      float2 e = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < j; ++k) e = ffma2(l[k], l[k], e);
      const float d = a[j].x - hsum(e);
      if (!(d > floor_)) singular = true;
      l[j] = make_float2(__fsqrt_rn(fmaxf(d, 1e-30f)), 0.f);
      lw[j] = make_float2(0.f, -l[j].x);
#pragma unroll
      for (int k = 0; k <= j; ++k) Lh[j * N + k] = l[k];
    }
    __syncwarp();
    if (i > j) {  // L_ij = (A_ij - sum_{k<j} L_ik conj(L_jk)) / L_jj   (numerics.cpp:53-56)
      float2 sv = a[j];
#pragma unroll
      for (int k = 0; k < j; ++k) {
        const float2 bk = Lh[j * N + k];
        sv = ffma2(-bk.x, l[k], sv);
        sv = ffma2(-bk.y, lw[k], sv);
      }
      const float inv = __frcp_rn(Lh[j * N + j].x);
      l[j] = fmul2(inv, sv);
      lw[j] = make_float2(l[j].y, -l[j].x);
    }
  }
  __syncwarp();
  // X = L^-1: lane (h, c) holds column c; X_ic = -(sum_{k=c}^{i-1} L_ik X_kc) / L_ii
  const int c = i;
  float tr = 0.f;
  float2 x[N], xw[N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    const float linv = __frcp_rn(Lh[r * N + r].x);
    float2 sv = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < r; ++k) {  // x[k] is zero above the diagonal (k < c)
      const float2 lk = Lh[r * N + k];
      sv = ffma2(lk.x, x[k], sv);
      sv = ffma2(lk.y, xw[k], sv);
    }
    float2 v;
    if (c == r) v = make_float2(linv, 0.f);
    else if (c < r) v = fmul2(-linv, sv);
    else v = make_float2(0.f, 0.f);
    x[r] = v;
    xw[r] = make_float2(-v.y, v.x);
    tr = fmaf(v.x, v.x, fmaf(v.y, v.y, tr));
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
#endif
  const unsigned sing = __ballot_sync(0xffffffffu, singular);
  const long long p = p0 + hf;
  if (i == 0 && p < P) {
    float s2 = scale * tr;
    if (round_fp16) s2 = __half2float(__float2half_rn(s2));
    out[p] = s2;
    if ((sing >> (16 * hf)) & 0xffffu) record_status(status, p, ST_SINGULAR, 0);
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
  griddep_wait();  // launched as a programmatic dependent of the CD kernel
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(S) * U) return;
  const long long s = idx / U;
  const int u = static_cast<int>(idx - s * U);
  const bool full = C == C_total;
  const T* xs = XL + static_cast<size_t>(s) * C * U + u;
  // the estimates of a chunk of clusters are loaded together (independent
  // loads in flight), then accumulated in ascending cluster order
  constexpr int CH = 8;
  float2 acc = make_float2(0.f, 0.f);
  if (!optimal) {
    const float w = 1.f / static_cast<float>(C_total);
    for (int c0 = 0; c0 < C; c0 += CH) {
      float2 v[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) v[i] = c0 + i < C ? ldc(xs, static_cast<size_t>(c0 + i) * U) : make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < CH; ++i)
        if (c0 + i < C) {
          acc.x = fmaf(w, v[i].x, acc.x);
          acc.y = fmaf(w, v[i].y, acc.y);
        }
    }
  } else {
    const float* sg = sigma2 + s * C;
    float total = 0.f;
    bool bad = false;
    for (int c0 = 0; c0 < C; c0 += CH) {
      float v[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) v[i] = c0 + i < C ? __ldg(sg + c0 + i) : 1.f;
#pragma unroll
      for (int i = 0; i < CH; ++i)
        if (c0 + i < C) {
          if (!(v[i] > 0.f) || !isfinite(v[i])) bad = true;
          total += 1.f / v[i];
        }
    }
    // keyed at the subcarrier's LAST cluster: a cluster's own error (e.g. a
    // singular variance) outranks it, as the reference's workers throw before
    // fusion_weights runs (detect.cpp:160-176)
    if (bad && u == 0) record_status(status, s * C + C - 1, ST_BAD_VARIANCE, 0);
    for (int c0 = 0; c0 < C; c0 += CH) {
      float2 v[CH];
      float q[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        v[i] = c0 + i < C ? ldc(xs, static_cast<size_t>(c0 + i) * U) : make_float2(0.f, 0.f);
        q[i] = c0 + i < C ? __ldg(sg + c0 + i) : 1.f;
      }
#pragma unroll
      for (int i = 0; i < CH; ++i)
        if (c0 + i < C) {
          const float w = full ? (1.f / q[i]) / total : 1.f / q[i];
          acc.x = fmaf(w, v[i].x, acc.x);
          acc.y = fmaf(w, v[i].y, acc.y);
        }
    }
    if (!full && wsum && u == 0) wsum[s] = total;
  }
  xhat[idx] = acc;
}

// ===========================================================================
// Fused cross-GPU exchange (see XMap in dcdg_device.cuh).
// xchg_put_kernel: for shapes whose CD kernel has no exchange epilogue, and for
// the optimal-fusion variances: copy this rank's per-cluster rows into the
// owners' windows, then signal (last CTA).
// xchg_fuse_kernel: on the owner, wait until every rank has published this
// epoch, then the reference's ascending-cluster fusion over the gathered
// [S_own][C_total] estimates — the arithmetic of fuse_kernel with C == C_total,
// so the result is bitwise that of a single GPU holding every cluster.
// ===========================================================================
template <typename T>
__global__ void xchg_put_kernel(const T* __restrict__ XL, const float* __restrict__ sigma2, long long P, XMap m) {
  const long long n = P * m.U;
  const int parity = static_cast<int>(xchg_epoch(m) & 1);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n + (sigma2 ? P : 0);
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (i < n) {
      const long long p = i / m.U;
      const int u = static_cast<int>(i - p * m.U);
      reinterpret_cast<T*>(xchg_x_dst(m, static_cast<int>(p), parity))[u] = XL[i];
    } else {
      const long long p = i - n;
      const long long s = p / m.C_local;
      const int c = static_cast<int>(p - s * m.C_local);
      const int owner = static_cast<int>(s / m.S_own);
      const long long s_in = s - static_cast<long long>(owner) * m.S_own;
      float* dst = reinterpret_cast<float*>(m.win[owner] + kXchgFlagBytes + parity * m.buf_bytes + m.sig_off);
      dst[s_in * m.C_total + m.c0 + c] = sigma2[p];
    }
  }
  xchg_cta_done(m);
}

__device__ __forceinline__ float2 ldcg_c(const float2* p, size_t i) { return __ldcg(p + i); }
__device__ __forceinline__ float2 ldcg_c(const __half2* p, size_t i) { return __half22float2(__ldcg(p + i)); }

template <typename T>
__global__ void xchg_fuse_kernel(const unsigned char* __restrict__ win, const unsigned long long* __restrict__ epoch_dev,
                                 int world, long long buf_bytes, long long sig_off, int S_own, int C_total, int U,
                                 bool optimal, long long timeout_ns, float2* __restrict__ xhat,
                                 unsigned long long* __restrict__ status) {
  // one system-scope acquire per block; the grid is sized to the SMs and
  // strides over the (subcarrier, user) outputs
  const unsigned long long epoch = xchg_epoch(epoch_dev);
  const int parity = static_cast<int>(epoch & 1);
  if (!xchg_block_wait(win, 0, world, epoch, timeout_ns, status)) return;
  const unsigned char* buf = win + kXchgFlagBytes + parity * buf_bytes;
  const T* XL = reinterpret_cast<const T*>(buf);
  const float* sigma2 = reinterpret_cast<const float*>(buf + sig_off);
  const long long n = static_cast<long long>(S_own) * U;
  for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long s = idx / U;
    const int u = static_cast<int>(idx - s * U);
    float2 acc = make_float2(0.f, 0.f);
    if (!optimal) {
      const float w = 1.f / static_cast<float>(C_total);
      for (int c = 0; c < C_total; ++c) {
        const float2 v = ldcg_c(XL, (static_cast<size_t>(s) * C_total + c) * U + u);
        acc.x = fmaf(w, v.x, acc.x);
        acc.y = fmaf(w, v.y, acc.y);
      }
    } else {
      float total = 0.f;
      bool bad = false;
      for (int c = 0; c < C_total; ++c) {
        const float v = __ldcg(sigma2 + s * C_total + c);
        if (!(v > 0.f) || !isfinite(v)) bad = true;
        total += 1.f / v;
      }
      if (bad && u == 0) record_status(status, s * C_total + C_total - 1, ST_BAD_VARIANCE, 0);  // see fuse_kernel
      for (int c = 0; c < C_total; ++c) {
        const float w = (1.f / __ldcg(sigma2 + s * C_total + c)) / total;
        const float2 v = ldcg_c(XL, (static_cast<size_t>(s) * C_total + c) * U + u);
        acc.x = fmaf(w, v.x, acc.x);
        acc.y = fmaf(w, v.y, acc.y);
      }
    }
    xhat[idx] = acc;
  }
}

// Downlink (decentralized_cd_precode, precode.cpp:136-169, across GPUs):
// xchg_symbols_push_kernel (root): store the centre's symbol batch into the
// symbol region of every rank's window (the centre -> cluster broadcast as
// NVLink stores), then publish kSlotSymbols.  Each rank's DL kernel then reads
// its symbols from its own window after xchg_wait_kernel.
template <typename T>
__global__ void xchg_symbols_push_kernel(const T* __restrict__ s, long long n, XMap m) {
  const int parity = static_cast<int>(xchg_epoch(m) & 1);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const T v = s[i];
    for (int q = 0; q < m.world; ++q)
      reinterpret_cast<T*>(m.win[q] + kXchgFlagBytes + parity * m.buf_bytes)[i] = v;
  }
  xchg_cta_done(m);
}

__global__ void xchg_wait_kernel(const unsigned char* __restrict__ win, int slot0, int n,
                                 const unsigned long long* __restrict__ epoch_dev, long long timeout_ns,
                                 unsigned long long* __restrict__ status) {
  xchg_block_wait(win, slot0, n, xchg_epoch(epoch_dev), timeout_ns, status);
}

// Each call advances the window's batch epoch on the device before its
// kernels read it (one sequence for both directions).
__global__ void xchg_advance_kernel(unsigned long long* __restrict__ epoch_dev) { *epoch_dev += 1ull; }

// The symbols of this call's parity buffer, copied out of the window for the
// precoder (whose input pointer cannot depend on a device-side epoch).
__global__ void xchg_symbols_fetch_kernel(const unsigned char* __restrict__ win,
                                          const unsigned long long* __restrict__ epoch_dev, long long buf_bytes,
                                          long long n16, uint4* __restrict__ dst) {
  const int parity = static_cast<int>(xchg_epoch(epoch_dev) & 1);
  const uint4* src = reinterpret_cast<const uint4*>(win + kXchgFlagBytes + parity * buf_bytes);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = __ldcg(src + i);
}

// Every rank's per-cluster gain shares Re(s^H H_dl,c x_c) gathered into every
// window as [S][C_total] (kSlotGain + rank published when done).
__global__ void xchg_gain_put_kernel(const float* __restrict__ gain_part, long long P, XMap m) {
  const int parity = static_cast<int>(xchg_epoch(m) & 1);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long s = i / m.C_local;
    const int c = static_cast<int>(i - s * m.C_local);
    const float v = gain_part[i];
    for (int q = 0; q < m.world; ++q)
      reinterpret_cast<float*>(m.win[q] + kXchgFlagBytes + parity * m.buf_bytes + m.sig_off)[s * m.C_total + m.c0 + c] = v;
  }
  xchg_cta_done(m);
}

// Wait for every rank's gain shares, then assemble_blocks' effective gain
// (precode.cpp:123-131) with gain_reduce_kernel's arithmetic over all C_total
// clusters in ascending order: bitwise the single-GPU gain.
template <typename T>
__global__ void xchg_gain_fuse_kernel(const unsigned char* __restrict__ win,
                                      const unsigned long long* __restrict__ epoch_dev, int world,
                                      long long buf_bytes, long long gain_off, int S, int C_total, int U,
                                      long long timeout_ns, float* __restrict__ gain,
                                      unsigned long long* __restrict__ status) {
  const unsigned long long epoch = xchg_epoch(epoch_dev);
  const int parity = static_cast<int>(epoch & 1);
  if (!xchg_block_wait(win, kSlotGain, world, epoch, timeout_ns, status)) return;
  if (!gain) return;
  const unsigned char* buf = win + kXchgFlagBytes + parity * buf_bytes;
  const T* Sy = reinterpret_cast<const T*>(buf);
  const float* part = reinterpret_cast<const float*>(buf + gain_off);
  for (long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; s < S;
       s += static_cast<long long>(gridDim.x) * blockDim.x) {
    float se = 0.f;
    for (int u = 0; u < U; ++u) {
      const float2 v = ldcg_c(Sy, static_cast<size_t>(s) * U + u);
      se = fmaf(v.y, v.y, fmaf(v.x, v.x, se));
    }
    float num = 0.f;
    for (int c = 0; c < C_total; ++c) num += __ldcg(part + s * C_total + c);
    gain[s] = se > 0.f ? num / se : 0.f;
  }
}

// dcdg_status_enqueue: the device status word into pinned host memory
__global__ void status_mirror_kernel(const unsigned long long* __restrict__ st, unsigned long long* host_word) {
  *reinterpret_cast<volatile unsigned long long*>(host_word) = *st;
}

__global__ void fuse_finalize_kernel(float2* __restrict__ xhat, const float* __restrict__ wsum, int S, int U) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(S) * U) return;
  const float w = wsum[idx / U];
  xhat[idx] = make_float2(xhat[idx].x / w, xhat[idx].y / w);
}

// Effective gain per subcarrier (precode.cpp:123-131): a block stages the
// symbols and gain shares of kGainSubs subcarriers with coalesced loads (rows
// padded by one complex against bank conflicts), then one thread per
// subcarrier runs the ascending-order sums.
constexpr int kGainSubs = 32;
inline size_t gain_reduce_smem(int U, int C) {
  return static_cast<size_t>(kGainSubs) * (U + 1) * sizeof(float2) + static_cast<size_t>(kGainSubs) * C * sizeof(float);
}

template <typename T>
__global__ void gain_reduce_kernel(const float* __restrict__ part, const T* __restrict__ Sy, int S, int C, int U,
                                   float* __restrict__ gain) {
  extern __shared__ float2 gsh[];  // [kGainSubs][U + 1] symbols, then [kGainSubs][C] shares
  float* psh = reinterpret_cast<float*>(gsh + kGainSubs * (U + 1));
  griddep_wait();  // launched as a programmatic dependent of the CD kernel
  const long long s0 = static_cast<long long>(blockIdx.x) * kGainSubs;
  const int ns = S - s0 < kGainSubs ? static_cast<int>(S - s0) : kGainSubs;
  for (int i = threadIdx.x; i < ns * U; i += blockDim.x) {
    const int r = i / U, u = i - r * U;
    gsh[r * (U + 1) + u] = ldc(Sy, static_cast<size_t>(s0) * U + i);
  }
  for (int i = threadIdx.x; i < ns * C; i += blockDim.x) psh[i] = __ldg(part + s0 * C + i);
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= ns) return;
  float se = 0.f;
  for (int u = 0; u < U; ++u) {
    const float2 v = gsh[t * (U + 1) + u];
    se = fmaf(v.y, v.y, fmaf(v.x, v.x, se));
  }
  float num = 0.f;
  for (int c = 0; c < C; ++c) num += psh[t * C + c];
  gain[s0 + t] = se > 0.f ? num / se : 0.f;
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
  if (bad) record_status(status, s * C + C - 1, ST_BAD_VARIANCE, 0);  // see fuse_kernel
  for (int c = 0; c < C; ++c) w[s * C + c] = (1.f / s2[s * C + c]) / total;
}

// ===========================================================================
// Hard decisions (§8f): Gray square QAM exactly as Constellation::qam builds
// it (mimo.cpp:64-109), nearest point by brute force in fp64 with the
// reference's arithmetic and strict '<' so distance ties go to the lowest
// label (Constellation::slice, mimo.cpp:111-122).
// ===========================================================================
struct Qam {
  double level[8];  // level_of_label
  int levels, axis_bits;
};

__device__ __forceinline__ Qam make_qam(unsigned order, double ex) {
  Qam q;
  q.levels = 2;
  int bits = 2;
  while (static_cast<unsigned>(q.levels * q.levels) < order) {
    q.levels <<= 1;
    bits += 2;
  }
  q.axis_bits = bits / 2;
  const double scale = sqrt(__ddiv_rn(3.0 * ex, 2.0 * (q.levels * q.levels - 1.0)));
  for (int pos = 0; pos < q.levels; ++pos)
    q.level[pos ^ (pos >> 1)] = __dmul_rn(scale, 2.0 * pos - (q.levels - 1.0));
  return q;
}

__device__ __forceinline__ unsigned slice_qam(const Qam& q, unsigned order, double yr, double yi) {
  unsigned best = 0;
  double best_d = 0.0;
  for (unsigned i = 0; i < order; ++i) {
    const double dr = __dsub_rn(yr, q.level[i >> q.axis_bits]);
    const double di = __dsub_rn(yi, q.level[i & (q.levels - 1)]);
    const double d = __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di));  // std::norm, no contraction
    if (i == 0 || d < best_d) {
      best_d = d;
      best = i;
    }
  }
  return best;
}

// labels[i] = slice(x[i] / beta[i])   (run_uplink_round's unbiasing, cluster.cpp:196-203)
template <typename T>
__global__ void slice_kernel(const T* __restrict__ x, const float* __restrict__ beta, long long n, unsigned order,
                             double ex, uint8_t* __restrict__ labels) {
  __shared__ Qam q;
  if (threadIdx.x == 0) q = make_qam(order, ex);
  __syncthreads();
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 v = ldc(x, i);
    double yr = v.x, yi = v.y;
    if (beta) {
      const double b = beta[i];
      yr = __ddiv_rn(yr, b);
      yi = __ddiv_rn(yi, b);
    }
    labels[i] = static_cast<uint8_t>(slice_qam(q, order, yr, yi));
  }
}

// errors += popcount(label ^ label(bits)) with bits MSB-first per symbol
// (demodulate_hard, mimo.cpp:141-150; BER tally cluster.cpp:203-206)
__global__ void bit_errors_kernel(const uint8_t* __restrict__ labels, const uint8_t* __restrict__ bits, long long n,
                                  int bps, unsigned long long* __restrict__ errors) {
  unsigned long long e = 0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (labels[i] == 0xff) {  // flagged downlink trial: half its bits count as errors (precode.cpp:219-223)
      e += static_cast<unsigned>(bps / 2);
      continue;
    }
    unsigned ref = 0;
    for (int k = 0; k < bps; ++k) ref = (ref << 1) | (bits[i * bps + k] & 1u);
    e += __popc(ref ^ labels[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0 && e) atomicAdd(errors, e);
}

// Downlink receive (downlink_receive_and_ber, precode.cpp:204-233), one warp
// per subcarrier with every cluster local: y0_u = sum_c h_{c,u}^H x_c,
// beta = Re(s^H y0)/||s||^2, y = y0 + noise, labels of y/beta; flagged when
// beta <= 0 or non-finite (the reference then counts half the bits wrong).
template <typename T>
__global__ void __launch_bounds__(128) dl_receive_kernel(const T* __restrict__ H, const T* __restrict__ X,
                                                         const T* __restrict__ Sy, const float2* __restrict__ noise,
                                                         int S, int C, int BC, int U, unsigned order, double ex,
                                                         uint8_t* __restrict__ labels, float* __restrict__ beta_out,
                                                         uint8_t* __restrict__ flagged) {
  __shared__ Qam q;
  if (threadIdx.x == 0) q = make_qam(order, ex);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long s = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (s >= S) return;
  float yr = 0.f, yi = 0.f;  // lane u: y0_u
  if (lane < U)
    for (int c = 0; c < C; ++c) {
      const T* h = H + ((static_cast<size_t>(s) * C + c) * U + lane) * BC;  // column u of tile c
      const T* x = X + (static_cast<size_t>(s) * C + c) * BC;
      for (int b = 0; b < BC; ++b) {
        const float2 hv = ldv(h, b), xv = ldc(x, b);
        yr = fmaf(hv.x, xv.x, fmaf(hv.y, xv.y, yr));
        yi = fmaf(hv.x, xv.y, fmaf(-hv.y, xv.x, yi));
      }
    }
  const float2 sv = lane < U ? ldc(Sy, static_cast<size_t>(s) * U + lane) : make_float2(0.f, 0.f);
  const float se = warp_sum(sv.x * sv.x + sv.y * sv.y);
  const float num = warp_sum(sv.x * yr + sv.y * yi);
  const float b = se > 0.f ? num / se : 0.f;
  const bool flag = !(b > 0.f) || !isfinite(b);
  if (lane == 0) {
    beta_out[s] = b;
    flagged[s] = flag;
  }
  if (lane < U) {
    if (noise) {
      const float2 nv = noise[static_cast<size_t>(s) * U + lane];
      yr += nv.x;
      yi += nv.y;
    }
    labels[static_cast<size_t>(s) * U + lane] =
        flag ? 0xff : static_cast<uint8_t>(slice_qam(q, order, __ddiv_rn(yr, b), __ddiv_rn(yi, b)));
  }
}

// Per-cluster effective-gain share of finished beamformers (assemble_blocks,
// precode.cpp:123-131): part[p] = Re(s^H H_dl,c x_c) = Re(sum_u conj(s_u) h_u^H x_c),
// one warp per problem, lane u.  Used where the precoding kernel saw a
// different s than the gain needs (fp16 messages_only: the clusters receive
// the rounded broadcast, the gain uses the centre's own s).
template <typename T>
__global__ void __launch_bounds__(128) gain_part_kernel(const T* __restrict__ H, const T* __restrict__ X,
                                                        const T* __restrict__ Sy, int P, int C, int BC, int U,
                                                        float* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = static_cast<long long>(blockIdx.x) * 4 + warp;
  if (p >= P) return;
  const long long s = p / C;
  const T* x = X + static_cast<size_t>(p) * BC;
  float acc = 0.f;
  for (int u = lane; u < U; u += 32) {
    const T* h = H + (static_cast<size_t>(p) * U + u) * BC;  // column u of the tile
    float yr = 0.f, yi = 0.f;
    for (int b = 0; b < BC; ++b) {
      const float2 hv = ldv(h, b), xv = ldc(x, b);
      yr = fmaf(hv.x, xv.x, fmaf(hv.y, xv.y, yr));
      yi = fmaf(hv.x, xv.y, fmaf(-hv.y, xv.x, yi));
    }
    const float2 sv = ldc(Sy, static_cast<size_t>(s) * U + u);
    acc = fmaf(sv.x, yr, fmaf(sv.y, yi, acc));
  }
  acc = warp_sum(acc);
  if (lane == 0) part[p] = acc;
}

__global__ void fill_kernel(float* __restrict__ x, long long n, float v) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    x[i] = v;
}

__global__ void round_fp16_kernel(float* __restrict__ x, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    x[i] = __half2float(__float2half_rn(x[i]));
}

// complex fp32 -> row-pair planar fp16 {re_a, re_b, im_a, im_b} and back
__global__ void f32_to_f16_pairs_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, long long npairs) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < npairs;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 v = src[i];  // re_a, im_a, re_b, im_b
    uint2 o;
    o.x = h2_as_u32(__floats2half2_rn(v.x, v.z));
    o.y = h2_as_u32(__floats2half2_rn(v.y, v.w));
    dst[i] = o;
  }
}

__global__ void f16_pairs_to_f32_kernel(const uint2* __restrict__ src, float4* __restrict__ dst, long long npairs) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < npairs;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 re = __half22float2(u32_as_h2(src[i].x)), im = __half22float2(u32_as_h2(src[i].y));
    dst[i] = make_float4(re.x, im.x, re.y, im.y);
  }
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
