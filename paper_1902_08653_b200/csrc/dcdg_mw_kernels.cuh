// Multi-warp register-resident CD kernels for large cluster tiles (B_c >= 128
// at U = 32, B_c >= 256 at U = 16): the channel tile no longer fits the
// registers of one warp, so one CTA of NW warps owns one problem at a time.
//
// Mapping
//   * Warp w owns the row stripe [w*RW, (w+1)*RW), RW = B_c/NW (64 or 128 rows,
//     i.e. 128 registers of channel per lane as in the single-warp kernels);
//     lane l owns row pairs c*32 + l of the stripe as planar float2 registers.
//   * Each warp stages its stripe itself: U column segments of RW complex (plus
//     its y segment, or the symbol vector for the downlink) by cp.async.bulk on
//     its own mbarrier, prefetching the CTA's next problem while it sweeps.
//   * Per coordinate block (LB = 2 or 4, see dcdg_reg_kernels.cuh) the LB
//     partial dot products of a warp (2*LB floats) are reduce-scattered over
//     the warp (6 shuffles for LB = 2 instead of a 20-shuffle butterfly), one
//     lane per value writes it to a double-buffered exchange row, and after one
//     CTA barrier every lane sums the NW rows in warp order (deterministic).  The scalar update
//     runs redundantly in every warp on its private scalar block, so no other
//     synchronisation is needed.
//   * Norms and block Grams are reduce-scattered per warp and summed across
//     warps through the same kind of exchange once per problem.
//
// Reference algorithms: cd_detect src/detect.cpp:67-110, cd_precode +
// power_scale src/precode.cpp:52-111, assemble_blocks src/precode.cpp:115-132.
#pragma once

#include "dcdg_reg_kernels.cuh"

namespace dcdg {

// Reduce-scatter NV values over a full warp, then finish the sum: afterwards
// lane l holds the warp-wide sum of value l / (32/NV).  log2(NV) halving rounds
// + log2(32/NV) single-value rounds.
template <int NV>
__device__ __forceinline__ float warp_scatter_sum(float (&v)[NV], int lane) {
  ReduceScatter<16, NV, NV>::run(v, lane);
  float s = v[0];
#pragma unroll
  for (int o = 16 / NV; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Shared-memory layout of one multi-warp CTA:
//   [NW staging slots][NW scalar blocks][xp: 2 x NW x NXP floats]
//   [xs: NW x NX floats][xe: NW float2][NW mbarriers]
// NXP: floats per warp per block exchange (2*LB); NX: floats per warp of the
// setup exchange (norms + block Grams, padded to a multiple of 32).
__host__ __device__ constexpr int mw_setup_floats(int U, int LB) {
  return (U + 2 * (U / LB) * (LB * (LB - 1) / 2) + 31) / 32 * 32;
}
template <int SLOT_B, int SCAL_B, int NW, int NX, int NXP = 4>
struct MwSmem {
  static constexpr int kScalOff = NW * SLOT_B;
  static constexpr int kXpOff = kScalOff + NW * SCAL_B;
  static constexpr int kXsOff = kXpOff + 2 * NW * NXP * 4;
  static constexpr int kXeOff = kXsOff + NW * NX * 4;
  static constexpr int kBarOff = (kXeOff + NW * 8 + 7) / 8 * 8;
  static constexpr int kBytes = kBarOff + NW * 8;
};

__host__ __device__ constexpr int ul_mw_slot_bytes(int BC, int U, int NW) { return (BC / NW) * (U + 1) * 8; }
__host__ __device__ constexpr int dl_mw_slot_bytes(int BC, int U, int NW) { return (BC / NW) * U * 8 + U * 8; }

// Issue this warp's stripe of problem p: U column segments of RW complex from
// the column-major tile + one vector segment (vbytes from vsrc).
template <int U, int RW, int BC>
__device__ __forceinline__ void issue_stripe(unsigned char* slot, uint64_t* bar, const float2* H, long long p, int w,
                                             const void* vsrc, int vbytes, int lane, uint64_t pol) {
  if (lane == 0) mbar_arrive_expect_tx(bar, static_cast<uint32_t>(U * RW * 8 + vbytes));
  __syncwarp();
  const float2* tile = H + static_cast<size_t>(p) * BC * U + static_cast<size_t>(w) * RW;
  for (int j = lane; j < U; j += 32) bulk_g2s(slot + j * RW * 8, tile + static_cast<size_t>(j) * BC, RW * 8, bar, pol);
  if (lane == 31) bulk_g2s(slot + U * RW * 8, vsrc, vbytes, bar, pol);
}

// Cross-warp sum of the per-warp setup vectors (NX = 2U floats each): lane l
// returns, for i < PER, the totals of values l*PER + i in warp order.
template <int NW, int PER>
__device__ __forceinline__ void setup_exchange(float (&v)[PER], float* xs, int warp, int lane, int NX) {
#pragma unroll
  for (int i = 0; i < PER; ++i) xs[warp * NX + lane * PER + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    float t = xs[lane * PER + i];
#pragma unroll
    for (int w = 1; w < NW; ++w) t += xs[w * NX + lane * PER + i];
    v[i] = t;
  }
}

// Exchange one reduce-scattered block of 4 dot-product floats; returns the
// CTA-wide sums (d0.re, d0.im, d1.re, d1.im).
template <int NW>
__device__ __forceinline__ float4 block_exchange(float s, float4* xp, int buf, int warp, int lane) {
  if ((lane & 7) == 0) reinterpret_cast<float*>(xp + buf * NW + warp)[lane >> 3] = s;
  __syncthreads();
  float4 d = xp[buf * NW];
#pragma unroll
  for (int w = 1; w < NW; ++w) {
    const float4 e = xp[buf * NW + w];
    d.x += e.x;
    d.y += e.y;
    d.z += e.z;
    d.w += e.w;
  }
  return d;
}

// Same for LB coordinates (2*LB floats per warp): d[a] = CTA-wide h_a^H r.
template <int NW, int LB>
__device__ __forceinline__ void block_exchange_lb(float s, float* xp, int buf, int warp, int lane, float2 (&d)[LB]) {
  constexpr int NV = 2 * LB, SP = 32 / NV;
  if (lane % SP == 0) xp[(buf * NW + warp) * NV + lane / SP] = s;
  __syncthreads();
  const float4* x4 = reinterpret_cast<const float4*>(xp + buf * NW * NV);
#pragma unroll
  for (int h = 0; h < LB / 2; ++h) {
    float4 t = x4[h];
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      const float4 e = x4[w * (NV / 4) + h];
      t.x += e.x;
      t.y += e.y;
      t.z += e.z;
      t.w += e.w;
    }
    d[2 * h] = make_float2(t.x, t.y);
    d[2 * h + 1] = make_float2(t.z, t.w);
  }
}

// ===========================================================================
// Uplink, fp32 (Alg. 1).  Scalar block per warp as in ul_reg_f32:
// float4 mnx[U] = (m_j, n_j, Re x_j, Im x_j), float4 gb[U/LB][LB(LB-1)/2] =
// block Grams (Re G, Im G, -Im G, Re G).
// ===========================================================================
template <int BC, int U, int NW, int MINB, int LB>
__global__ void __launch_bounds__(32 * NW, MINB)
    ul_mw_f32(const float2* __restrict__ H, const float2* __restrict__ Y, int P, int K, float kappa,
              float2* __restrict__ X) {
  constexpr int RW = BC / NW, NP = RW / 64, T = LB * (LB - 1) / 2;
  constexpr int NG0 = 2 * (U / LB) * T, NX = mw_setup_floats(U, LB), PER = NX / 32;
  static_assert(RW % 64 == 0 && U % 16 == 0 && NW <= 8 && (LB == 2 || LB == 4), "shape");
  constexpr int SLOT_B = ul_mw_slot_bytes(BC, U, NW), SCAL_B = ul_scal_bytes(U, LB);
  using L = MwSmem<SLOT_B, SCAL_B, NW, NX, 2 * LB>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* slot = smem + warp * SLOT_B;
  float4* mnx = reinterpret_cast<float4*>(smem + L::kScalOff + warp * SCAL_B);
  float4* gb = mnx + U;
  float* xp = reinterpret_cast<float*>(smem + L::kXpOff);
  float* xs = reinterpret_cast<float*>(smem + L::kXsOff);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff) + warp;
  const uint64_t pol = l2_evict_first_policy();
  long long p = blockIdx.x;
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (p < P) issue_stripe<U, RW, BC>(slot, bar, H, p, warp, Y + static_cast<size_t>(p) * BC + warp * RW, RW * 8, lane, pol);
  uint32_t phase = 0;
  const float2 z2 = make_float2(0.f, 0.f);
  for (; p < P; p += gridDim.x) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    float2 hr[U][NP], hi[U][NP], rr[NP], ri[NP];
    {
      const float4* t4 = reinterpret_cast<const float4*>(slot);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const float4 v = t4[j * (RW / 2) + c * 32 + lane];
          hr[j][c] = pair(v.x, v.z);
          hi[j][c] = pair(v.y, v.w);
        }
      const float4* y4 = reinterpret_cast<const float4*>(slot + U * RW * 8);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float4 v = y4[c * 32 + lane];
        rr[c] = pair(v.x, v.z);
        ri[c] = pair(v.y, v.w);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    {
      const long long pn = p + gridDim.x;
      if (pn < P)
        issue_stripe<U, RW, BC>(slot, bar, H, pn, warp, Y + static_cast<size_t>(pn) * BC + warp * RW, RW * 8, lane,
                                pol);
    }

    // ---- ||h_j||^2 (detect.cpp:86-90) and block Grams G_ab = h_a^H h_b (a > b)
    {
      float v[NX];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float2 e = fmul2(hr[j][0], hr[j][0]);
        e = ffma2(hi[j][0], hi[j][0], e);
#pragma unroll
        for (int c = 1; c < NP; ++c) e = ffma2(hi[j][c], hi[j][c], ffma2(hr[j][c], hr[j][c], e));
        v[j] = hsum(e);
      }
#pragma unroll
      for (int q = 0; q < U / LB; ++q)
#pragma unroll
        for (int a = 1; a < LB; ++a)
#pragma unroll
          for (int b = 0; b < a; ++b) {
            const int ja = q * LB + a, jb = q * LB + b, e = q * T + a * (a - 1) / 2 + b;
            float2 gr = z2, gi = z2;
#pragma unroll
            for (int c = 0; c < NP; ++c) {
              gr = ffma2(hi[ja][c], hi[jb][c], ffma2(hr[ja][c], hr[jb][c], gr));
              gi = ffma2(neg2(hi[ja][c]), hr[jb][c], ffma2(hr[ja][c], hi[jb][c], gi));
            }
            v[U + 2 * e] = hsum(gr);
            v[U + 2 * e + 1] = hsum(gi);
          }
#pragma unroll
      for (int i = U + NG0; i < NX; ++i) v[i] = 0.f;
      group_reduce_scatter<32>(v, lane);
      float t[PER];
#pragma unroll
      for (int i = 0; i < PER; ++i) t[i] = v[i];
      setup_exchange<NW, PER>(t, xs, warp, lane, NX);
      float* gf = reinterpret_cast<float*>(gb);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int idx = lane * PER + i;
        if (idx < U) {
          const float m = __fdividef(1.f, t[i] + kappa);  // m_j = 1/(||h_j||^2 + N0/Ex)
          mnx[idx] = make_float4(m, m * t[i], 0.f, 0.f);
        } else if (idx < U + NG0) {
          const int gi = idx - U, e = gi >> 1;
          if (gi & 1) {
            gf[e * 4 + 1] = t[i];
            gf[e * 4 + 2] = -t[i];
          } else {
            gf[e * 4 + 0] = t[i];
            gf[e * 4 + 3] = t[i];
          }
        }
      }
    }
    __syncwarp();

    // ---- K sweeps, users ascending, LB coordinates per CTA exchange
    for (int t = 0; t < K; ++t) {
#pragma unroll
      for (int q = 0; q < U / LB; ++q) {
        float vv[2 * LB];
#pragma unroll
        for (int a = 0; a < LB; ++a) {  // h_j^H r (cdotc, detect.cpp:100), all against the same r
          const int j = q * LB + a;
          float2 ar = z2, ai = z2;
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            ar = ffma2(hi[j][c], ri[c], ffma2(hr[j][c], rr[c], ar));
            ai = ffma2(neg2(hi[j][c]), rr[c], ffma2(hr[j][c], ri[c], ai));
          }
          vv[2 * a] = hsum(ar);
          vv[2 * a + 1] = hsum(ai);
        }
        const float s = warp_scatter_sum<2 * LB>(vv, lane);
        float2 d[LB];
        block_exchange_lb<NW, LB>(s, xp, (t * (U / LB) + q) & 1, warp, lane, d);
        float2 dx[LB];
#pragma unroll
        for (int a = 0; a < LB; ++a) {
          const int j = q * LB + a;
          const float4 A = mnx[j];
#pragma unroll
          for (int b = 0; b < a; ++b) {  // h_j^H (r - sum_{b<a} dx_b h_b)
            const float4 Gab = gb[q * T + a * (a - 1) / 2 + b];
            d[a] = ffma2(-dx[b].x, make_float2(Gab.x, Gab.y), d[a]);
            d[a] = ffma2(-dx[b].y, make_float2(Gab.z, Gab.w), d[a]);
          }
          // x_j' = m_j h_j^H r + n_j x_j ; dx = x_j' - x_j   (detect.cpp:100-103)
          const float2 xo = make_float2(A.z, A.w);
          const float2 xn = ffma2(A.x, d[a], fmul2(A.y, xo));
          dx[a] = fadd2(xn, neg2(xo));
          *reinterpret_cast<float2*>(&mnx[j].z) = xn;
        }
#pragma unroll
        for (int a = 0; a < LB; ++a) {  // r -= dx_j h_j   (caxpy, detect.cpp:104)
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
    if (warp == 0) {
      float4* xo = reinterpret_cast<float4*>(X + static_cast<size_t>(p) * U);
#pragma unroll
      for (int i = lane; i < U / 2; i += 32) {
        const float4 u0 = mnx[2 * i], u1 = mnx[2 * i + 1];
        xo[i] = make_float4(u0.z, u0.w, u1.z, u1.w);
      }
    }
    __syncthreads();  // exchange buffers are reused by the next problem
  }
}

// ===========================================================================
// Downlink, fp32 (Alg. 2 + power_scale + effective-gain share).  Scalar block
// per warp as in dl_reg_f32: float4 ss[U] = (Re s~, Im s~, p_u, ||h_u||),
// float4 gp[U/2] = normalised pair Grams, float2 sraw[U].
// ===========================================================================
template <int BC, int U, int NW, int MINB, bool GAIN>
__global__ void __launch_bounds__(32 * NW, MINB)
    dl_mw_f32(const float2* __restrict__ H, const float2* __restrict__ Sy, int P, int C, int K, float rho_c,
              float2* __restrict__ X, float* __restrict__ gain_part, unsigned long long* __restrict__ status) {
  constexpr int RW = BC / NW, NP = RW / 64, NX = 2 * U, PER = NX / 32;
  static_assert(RW % 64 == 0 && U % 16 == 0 && NW <= 8, "shape");
  constexpr int SLOT_B = dl_mw_slot_bytes(BC, U, NW), SCAL_B = dl_scal_bytes(U);
  static_assert(NX == mw_setup_floats(U, 2), "downlink setup layout");
  using L = MwSmem<SLOT_B, SCAL_B, NW, NX, 4>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* slot = smem + warp * SLOT_B;
  float4* ss = reinterpret_cast<float4*>(smem + L::kScalOff + warp * SCAL_B);
  float4* gp = ss + U;
  float2* sraw = reinterpret_cast<float2*>(gp + U / 2);
  float4* xp = reinterpret_cast<float4*>(smem + L::kXpOff);
  float* xs = reinterpret_cast<float*>(smem + L::kXsOff);
  float2* xe = reinterpret_cast<float2*>(smem + L::kXeOff);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff) + warp;
  const uint64_t pol = l2_evict_first_policy();
  long long p = blockIdx.x;
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (p < P) issue_stripe<U, RW, BC>(slot, bar, H, p, warp, Sy + static_cast<size_t>(p / C) * U, U * 8, lane, pol);
  uint32_t phase = 0;
  const float2 z2 = make_float2(0.f, 0.f);
  for (; p < P; p += gridDim.x) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    float2 hr[U][NP], hi[U][NP];
    {
      const float4* t4 = reinterpret_cast<const float4*>(slot);
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const float4 v = t4[j * (RW / 2) + c * 32 + lane];
          hr[j][c] = pair(v.x, v.z);
          hi[j][c] = pair(v.y, v.w);
        }
      const float4* s4 = reinterpret_cast<const float4*>(slot + U * RW * 8);
      float4* d4 = reinterpret_cast<float4*>(sraw);
#pragma unroll
      for (int i = lane; i < U / 2; i += 32) d4[i] = s4[i];
    }
    fence_proxy_async_smem();
    __syncwarp();
    {
      const long long pn = p + gridDim.x;
      if (pn < P)
        issue_stripe<U, RW, BC>(slot, bar, H, pn, warp, Sy + static_cast<size_t>(pn / C) * U, U * 8, lane, pol);
    }

    // ---- row norms and raw pair Grams (precode.cpp:69-87), summed over warps
    float t[PER];
    {
      float v[NX];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float2 e = fmul2(hr[j][0], hr[j][0]);
        e = ffma2(hi[j][0], hi[j][0], e);
#pragma unroll
        for (int c = 1; c < NP; ++c) e = ffma2(hi[j][c], hi[j][c], ffma2(hr[j][c], hr[j][c], e));
        v[j] = hsum(e);
      }
#pragma unroll
      for (int i = 0; i < U / 2; ++i) {
        float2 gr = z2, gi = z2;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          gr = ffma2(hi[2 * i + 1][c], hi[2 * i][c], ffma2(hr[2 * i + 1][c], hr[2 * i][c], gr));
          gi = ffma2(neg2(hi[2 * i + 1][c]), hr[2 * i][c], ffma2(hr[2 * i + 1][c], hi[2 * i][c], gi));
        }
        v[U + 2 * i] = hsum(gr);
        v[U + 2 * i + 1] = hsum(gi);
      }
      group_reduce_scatter<32>(v, lane);
#pragma unroll
      for (int i = 0; i < PER; ++i) t[i] = v[i];
      setup_exchange<NW, PER>(t, xs, warp, lane, NX);
    }
    int zero_user = -1;
    float* sf = reinterpret_cast<float*>(ss);
    float* gf = reinterpret_cast<float*>(gp);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int idx = lane * PER + i;
      if (idx < U) {
        if (t[i] == 0.f && zero_user < 0) zero_user = idx;
        const float pinv = rsqrtf(t[i]);
        sf[idx * 4 + 2] = pinv;  // p_u = 1/||h_u||
        sf[idx * 4 + 3] = t[i] * pinv;
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int idx = lane * PER + i;
      if (idx < U) {
        const float2 s = sraw[idx];
        const float pj = sf[idx * 4 + 2];
        sf[idx * 4] = s.x * pj;  // s~_u = p_u s_u
        sf[idx * 4 + 1] = s.y * pj;
      } else {
        const int gi = idx - U, pr = gi >> 1;
        const float val = t[i] * (sf[(2 * pr + 1) * 4 + 2] * sf[(2 * pr) * 4 + 2]);  // G~ = p_a p_b G
        if (gi & 1) {
          gf[pr * 4 + 1] = val;
          gf[pr * 4 + 2] = -val;
        } else {
          gf[pr * 4 + 0] = val;
          gf[pr * 4 + 3] = val;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {  // normalise the rows held in registers
      const float pj = sf[j * 4 + 2];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        hr[j][c] = fmul2(pj, hr[j][c]);
        hi[j][c] = fmul2(pj, hi[j][c]);
      }
    }
    __syncwarp();

    float2 xr[NP], xi[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) xr[c] = xi[c] = z2;
    int buf = 0;
    for (int it = 0; it < K; ++it) {
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp) {
        const int j0 = 2 * jp, j1 = 2 * jp + 1;
        float2 a0 = z2, c0 = z2, a1 = z2, c1 = z2;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          a0 = ffma2(hi[j0][c], xi[c], ffma2(hr[j0][c], xr[c], a0));
          c0 = ffma2(neg2(hi[j0][c]), xr[c], ffma2(hr[j0][c], xi[c], c0));
          a1 = ffma2(hi[j1][c], xi[c], ffma2(hr[j1][c], xr[c], a1));
          c1 = ffma2(neg2(hi[j1][c]), xr[c], ffma2(hr[j1][c], xi[c], c1));
        }
        float vv[4] = {hsum(a0), hsum(c0), hsum(a1), hsum(c1)};
        const float s = warp_scatter_sum<4>(vv, lane);
        const float4 d = block_exchange<NW>(s, xp, buf, warp, lane);
        buf ^= 1;
        const float4 S0 = ss[j0], S1 = ss[j1], GG = gp[jp];
        // resid_u = h~_u^H x - s~_u ; x -= resid_u h~_u   (precode.cpp:89-94)
        const float2 r0 = make_float2(d.x - S0.x, d.y - S0.y);
        float2 d1 = make_float2(d.z, d.w);
        d1 = ffma2(-r0.x, make_float2(GG.x, GG.y), d1);
        d1 = ffma2(-r0.y, make_float2(GG.z, GG.w), d1);
        const float2 r1 = fadd2(d1, make_float2(-S1.x, -S1.y));
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          xr[c] = ffma2(r0.y, hi[j0][c], ffma2(-r0.x, hr[j0][c], xr[c]));
          xi[c] = ffma2(-r0.y, hr[j0][c], ffma2(-r0.x, hi[j0][c], xi[c]));
          xr[c] = ffma2(r1.y, hi[j1][c], ffma2(-r1.x, hr[j1][c], xr[c]));
          xi[c] = ffma2(-r1.y, hr[j1][c], ffma2(-r1.x, hi[j1][c], xi[c]));
        }
      }
    }
    // ||x||^2 and the raw gain share Re(v^H x), v = sum_u s_u ||h_u|| h~_u,
    // summed over the warps in one exchange; both scale linearly with gsc
    float2 e2 = fmul2(xr[0], xr[0]);
    e2 = ffma2(xi[0], xi[0], e2);
#pragma unroll
    for (int c = 1; c < NP; ++c) e2 = ffma2(xi[c], xi[c], ffma2(xr[c], xr[c], e2));
    float eq[2] = {hsum(e2), 0.f};
    if (GAIN) {
      float2 vr[NP], vi[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) vr[c] = vi[c] = z2;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const float2 sj = sraw[j];
        const float nj = ss[j].w;
        const float cr = sj.x * nj, ci = sj.y * nj;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          vr[c] = ffma2(-ci, hi[j][c], ffma2(cr, hr[j][c], vr[c]));
          vi[c] = ffma2(ci, hr[j][c], ffma2(cr, hi[j][c], vi[c]));
        }
      }
      float2 q2 = fmul2(vr[0], xr[0]);
      q2 = ffma2(vi[0], xi[0], q2);
#pragma unroll
      for (int c = 1; c < NP; ++c) q2 = ffma2(vi[c], xi[c], ffma2(vr[c], xr[c], q2));
      eq[1] = hsum(q2);
    }
    {
      const float sum = warp_scatter_sum<2>(eq, lane);  // lanes 0-15: ||x||^2, 16-31: gain share
      if ((lane & 15) == 0) reinterpret_cast<float*>(xe + warp)[lane >> 4] = sum;
    }
    __syncthreads();
    float2 tot = xe[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      tot.x += xe[w].x;
      tot.y += xe[w].y;
    }
    // power_scale to rho_c = rho / sqrt(C)   (precode.cpp:101-111,155); rho_c == 0: raw beamformer
    const float e = tot.x;
    const float gsc = rho_c > 0.f ? rho_c / __fsqrt_rn(e) : 1.f;
    if (warp == 0) {
      if (zero_user >= 0) record_status(status, p, ST_ZERO_ROW, zero_user);
      if (lane == 0) {
        if (e == 0.f && rho_c > 0.f) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
        if (GAIN) gain_part[p] = gsc * tot.y;
      }
    }
    float4* x4 = reinterpret_cast<float4*>(X + static_cast<size_t>(p) * BC + warp * RW);
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      const float2 a = fmul2(gsc, xr[c]), b = fmul2(gsc, xi[c]);
      x4[c * 32 + lane] = make_float4(a.x, b.x, a.y, b.y);
    }
    __syncthreads();  // exchange buffers are reused by the next problem
  }
}

}  // namespace dcdg
