// Gram-space uplink CD on the tensor cores — fp16 storage, fp32 arithmetic.
//
// Alg. 1 (detect.cpp:67-110) touches the channel only through inner products
// h_j^H r with r = y - H x, so it can run in the U-dimensional space of the
// matched filter c = H^H r = z - G x  (z = H^H y, G = H^H H):
//     d_j = c_j;  x_j' = m_j d_j + n_j x_j;  dx = x_j' - x_j;
//     r -= dx h_j   <=>   c_k -= dx G_kj  for every k.
// Same sweep order, same updates; only rounding differs.  The B_c-long work
// (G and z, 20 mma per problem) goes to the tensor cores (mma.sync
// m16n8k16, fp16 in, fp32 accumulate: exact products of the stored fp16
// values), and each coordinate update becomes a broadcast of dx and a
// U-long fp32 update of c spread over the problem's lanes.  The half2 sweep
// kernel (dcdg_reg_kernels.cuh) stays the kernel that mirrors the paper's
// half-precision arithmetic; this one is more accurate (fp32 arithmetic on
// the stored fp16 values) and faster on B200 (0.098 vs 0.112 ms per 134 400
// problems, profiles/lab/README.md).
//
// The contraction axis is the memory order of a column.  An fp16 column of
// the row-pair planar layout is W = {re_0, re_1, im_0, im_1, re_2, ...}; then
//     sum_p W_m[p] W_n[p]  = Re(h_m^H h_n),
//     sum_p W_m[p] W'_n[p] = Im(h_m^H h_n),  W' = {im_0, im_1, -re_0, -re_1, ...}
// (and likewise z with y), so the fragments are the stored words: W' is one
// lane-pair exchange and a sign flip of the same registers.
//
// Staging: a 2-D TMA (cp.async.bulk.tensor, 128-B swizzle) brings the set's
// NPW x U columns of 128 B into shared memory so that the ldmatrix row reads
// are bank-conflict free; y by a 1-D bulk copy; both on one mbarrier.  The
// next set's copy is issued as soon as the Grams are built, so it overlaps
// the sweeps.
//
// Mapping: one warp per CTA (persistent), NPW = 4 problems per set.  The
// tensor-core phase runs problem by problem over the whole warp and hands
// each problem's G (through a padded shared-memory transit buffer) to its 8
// sweep lanes: lane k keeps rows 2k, 2k+1 of G in registers and owns
// c_{2k}, c_{2k+1}, x_{2k}, x_{2k+1}; coordinates go in pairs owned by one
// lane (the second dot corrected with G_{2k+1,2k}, one shuffle round per pair).
#pragma once

#include <cuda.h>

#include "dcdg_device.cuh"

namespace dcdg {

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}


// W' word of this lane from the W fragment word: lane t holds word t of a
// 16-B chunk {re pair, im pair, re pair, im pair}; W' swaps each (re, im)
// word pair and negates the new odd word.
__device__ __forceinline__ uint32_t swap_neg(uint32_t w, int t) {
  const uint32_t o = __shfl_xor_sync(0xffffffffu, w, 1);
  return (t & 1) ? (o ^ 0x80008000u) : o;
}

__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int U, int NPW>
struct GramSmem {
  static_assert(U == 16, "Gram kernel: U = 16");
  static constexpr int kRowB = 128;                 // one fp16 column of B_c = 32 antennas
  static constexpr int kSlotB = NPW * U * kRowB;    // TMA box: NPW*U rows of 128 B (1024-B aligned)
  static constexpr int kYOff = kSlotB;              // NPW y vectors, 128 B each
  // pivot rows of the fused variance (SIG): [problem][2][U/2] float4
  static constexpr int kGOff = kYOff + NPW * 128;
  static constexpr int kZOff = kGOff + NPW * U * 16;  // z: [problem][j] float2
  static constexpr int kBarOff = kZOff + NPW * U * 8;
  static constexpr int kBcOff = kBarOff + 16;       // sweep broadcast slots: [NPW][2] float4
  static constexpr int kBytes = kBcOff + NPW * 32;
  static constexpr int kAlloc = kBytes + 1024;      // slack to align the swizzled slot to 1024 B
};

// Gram fragments by 8-B loads in a (re, im)-paired k-order (1) or ldmatrix
// plus a lane-pair shuffle for W' (0)
#ifndef DCDG_GRAM_LDS64
#define DCDG_GRAM_LDS64 1
#endif
#ifndef DCDG_GRAM_SMEM_BCAST
#define DCDG_GRAM_SMEM_BCAST 0
#endif
// The pair's two updates from its owner lane (base + jp) to the problem's 8
// lanes: four shuffles (default), or (DCDG_GRAM_SMEM_BCAST=1) one 16-B store
// by the owner into an alternating shared-memory slot and one 16-B broadcast
// load.  The slot won by ~1% while the Gram rows went through a separate
// transit buffer; with the slot transit the shuffles win by 1-2%
// (profiles/lab/README.md).
__device__ __forceinline__ float4 pair_bcast(float4 v, int JP, int k, int base, float4* slots) {
#if DCDG_GRAM_SMEM_BCAST
  float4* sl = slots + (JP & 1);
  if (k == JP) *sl = v;
  __syncwarp();
  return *sl;
#else
  (void)k;
  (void)slots;
  return make_float4(__shfl_sync(0xffffffffu, v.x, base + JP), __shfl_sync(0xffffffffu, v.y, base + JP),
                     __shfl_sync(0xffffffffu, v.z, base + JP), __shfl_sync(0xffffffffu, v.w, base + JP));
#endif
}


// Tensor-core phase of a set (shared by the uplink and downlink kernels): the
// Gram G = H^H H (and, with Z, the matched filter z = H^H y) of each of the
// NPW problems, from the swizzled TMA slot, handed through the slot itself
// (each problem's consumed rows) to the problem's 8 sweep lanes: lane k of
// problem q gets rows 2k and 2k+1 of G (and z_{2k}, z_{2k+1}).
template <int U, int NPW, bool Z>
__device__ __forceinline__ void gram_tc_phase(unsigned char* sm, uint32_t sbase, int lane, float (&g0r)[U],
                                              float (&g0i)[U], float (&g1r)[U], float (&g1i)[U], float (&cr)[2],
                                              float (&ci)[2]) {
  using L = GramSmem<U, NPW>;
  const int g = lane >> 2, t = lane & 3;  // mma fragment coordinates
  const int q = lane >> 3, k = lane & 7;
  // ldmatrix row of this lane: matrix mi = lane/8 -> users (mi&1)*8 + lane%8, chunk half mi>>1
  const int lu = ((lane >> 3) & 1) * 8 + (lane & 7), lch = lane >> 4;
  float2* zbuf = reinterpret_cast<float2*>(sm + L::kZOff);
#pragma unroll
  for (int pl = 0; pl < NPW; ++pl) {
    float gr[2][4] = {}, gi[2][4] = {}, zz[4] = {};
#if !DCDG_GRAM_LDS64
    const int row = pl * U + lu;
#endif
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t a[4];
#if DCDG_GRAM_LDS64
      // k-order: thread t of k-step ks takes row pair 4ks + t, its (re, im)
      // word pair in one 8-B load per user (k 2t, 2t+1 = re pair, k 2t+8, 2t+9
      // = im pair), so W' = (im, -re) is a register swap and a sign flip
      {
        const int row0 = pl * U + g, row1 = row0 + 8, ch = 2 * ks + (t >> 1), off = (t & 1) * 8;
        const uint2 u0 = *reinterpret_cast<const uint2*>(sm + row0 * L::kRowB + ((ch ^ (row0 & 7)) << 4) + off);
        const uint2 u1 = *reinterpret_cast<const uint2*>(sm + row1 * L::kRowB + ((ch ^ (row1 & 7)) << 4) + off);
        a[0] = u0.x;
        a[1] = u1.x;
        a[2] = u0.y;
        a[3] = u1.y;
      }
      (void)lu;
      (void)lch;
      mma_f16f32(gr[0], a, a[0], a[2]);
      mma_f16f32(gr[1], a, a[1], a[3]);
      mma_f16f32(gi[0], a, a[2], a[0] ^ 0x80008000u);
      mma_f16f32(gi[1], a, a[3], a[1] ^ 0x80008000u);
      if (Z) {
        // B = [Y, Y', 0 ...]: column g = 0 is y, g = 1 = (im, -re), same k-order
        uint32_t y0 = 0, y1 = 0;
        if (g < 2) {
          const uint2 yv = reinterpret_cast<const uint2*>(sm + L::kYOff + pl * 128)[4 * ks + t];
          y0 = g ? yv.y : yv.x;
          y1 = g ? (yv.x ^ 0x80008000u) : yv.y;
        }
        mma_f16f32(zz, a, y0, y1);
      }
#else
      const int ch = 2 * ks + lch;
      ldsm_x4(a, sbase + row * L::kRowB + ((ch ^ (row & 7)) << 4));
      // B = W: n-tile 0 (users 0-7) = (a0, a2), n-tile 1 (users 8-15) = (a1, a3)
      mma_f16f32(gr[0], a, a[0], a[2]);
      mma_f16f32(gr[1], a, a[1], a[3]);
      mma_f16f32(gi[0], a, swap_neg(a[0], t), swap_neg(a[2], t));
      mma_f16f32(gi[1], a, swap_neg(a[1], t), swap_neg(a[3], t));
      if (Z) {
        // B = [Y, Y', 0 ...]: column g = 0 is y, g = 1 its swapped/negated words
        uint32_t y0 = 0, y1 = 0;
        if (g < 2) {
          const uint32_t* yw = reinterpret_cast<const uint32_t*>(sm + L::kYOff + pl * 128);
          const int w = g ? (t ^ 1) : t;
          const uint32_t sg = (g && (t & 1)) ? 0x80008000u : 0u;
          y0 = yw[(2 * ks) * 4 + w] ^ sg;
          y1 = yw[(2 * ks + 1) * 4 + w] ^ sg;
        }
        mma_f16f32(zz, a, y0, y1);
      }
#endif
    }
    // problem pl's rows of the slot are consumed: its G goes there, swizzled
    // [k][chunk j ^ k][rows 2k, 2k+1] (2048 B, conflict-free 16-B reads), and
    // all four problems' rows are read back in one pass after the loop
    // (0.096 -> 0.087 ms uplink, 0.103 -> 0.095 ms downlink against a
    // separate transit buffer read problem by problem, profiles/lab/README.md)
    __syncwarp();
    unsigned char* tb = sm + pl * (U * L::kRowB);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = nt * 8 + 2 * t + h, k0 = g >> 1, k1 = (g >> 1) + 4;
        *reinterpret_cast<float2*>(tb + k0 * (U * 16) + ((j ^ k0) << 4) + (g & 1) * 8) =
            make_float2(gr[nt][h], gi[nt][h]);
        *reinterpret_cast<float2*>(tb + k1 * (U * 16) + ((j ^ k1) << 4) + (g & 1) * 8) =
            make_float2(gr[nt][2 + h], gi[nt][2 + h]);
      }
    if (Z && t == 0) {
      zbuf[pl * U + g] = make_float2(zz[0], zz[1]);
      zbuf[pl * U + g + 8] = make_float2(zz[2], zz[3]);
    }
  }
  __syncwarp();
  {
    const unsigned char* mine = sm + q * (U * L::kRowB) + k * (U * 16);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const float4 v = *reinterpret_cast<const float4*>(mine + ((j ^ k) << 4));
      g0r[j] = v.x;
      g0i[j] = v.y;
      g1r[j] = v.z;
      g1i[j] = v.w;
    }
    if (Z) {
      const float4 zv = reinterpret_cast<const float4*>(zbuf + q * U)[k];
      cr[0] = zv.x;
      ci[0] = zv.y;
      cr[1] = zv.z;
      ci[1] = zv.w;
    }
  }
}

#ifndef DCDG_GRAM_SIG_CPAIRS
#define DCDG_GRAM_SIG_CPAIRS 0  // lab: column-pair FFMA2 sweep operator here, 0.268 -> 0.296 ms (slower)
#endif
template <int U, int NPW, int MINB, bool SIG = false>
__global__ void __launch_bounds__(32, MINB)
    ul_gram_f16(const __grid_constant__ CUtensorMap tmH, const __half2* __restrict__ Y, int P, int K, float kappa,
                __half2* __restrict__ X, float* __restrict__ sigma2, float gam, float scale,
                unsigned long long* __restrict__ status) {
  static_assert(NPW == 4, "a set is 4 problems of 8 sweep lanes");
  using L = GramSmem<U, NPW>;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  unsigned char* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::kBarOff);
  const int lane = threadIdx.x & 31;
  const int q = lane >> 3, k = lane & 7;  // sweep: problem q of the set; lane k owns users 2k, 2k+1
  const int nsets = (P + NPW - 1) / NPW;
  int set = blockIdx.x;
  const uint64_t pol = l2_evict_first_policy();
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int s) {
    const int p0 = s * NPW;
    const int n = min(NPW, P - p0);
    mbar_arrive_expect_tx(bar, static_cast<uint32_t>(L::kSlotB + n * 128));
    tma_load_2d(sm, &tmH, 0, p0 * U, bar, pol);
    bulk_g2s(sm + L::kYOff, reinterpret_cast<const unsigned char*>(Y) + static_cast<size_t>(p0) * 128, n * 128, bar,
             pol);
  };
  if (lane == 0 && set < nsets) issue(set);
  uint32_t phase = 0;
  for (; set < nsets; set += gridDim.x) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    // rows 2k, 2k+1 of this lane's problem's G (fp32, registers) and c = z
    float g0r[U], g0i[U], g1r[U], g1i[U];
    float cr[2], ci[2];
    // ---------------- tensor-core phase: G and z of each problem, handed to its 8 sweep lanes
    gram_tc_phase<U, NPW, true>(sm, sbase, lane, g0r, g0i, g1r, g1i, cr, ci);
    fence_proxy_async_all();
    __syncwarp();
    if (lane == 0 && set + static_cast<int>(gridDim.x) < nsets) issue(set + gridDim.x);

    // ---------------- sweep phase: 8 lanes per problem, c = H^H r in fp32,
    // coordinates in pairs (2jp, 2jp+1) owned by lane jp: the pair's second
    // dot is corrected locally with G_{2jp+1,2jp}, both dx go out in one
    // shuffle round.
    float xr[2] = {0.f, 0.f}, xi[2] = {0.f, 0.f}, mm[2], nn[2];
    {
      float e[2];
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp)
        if (k == jp) {
          e[0] = g0r[2 * jp];      // G_{2k,2k}
          e[1] = g1r[2 * jp + 1];  // G_{2k+1,2k+1}
        }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mm[h] = __fdividef(1.f, e[h] + kappa);  // m_j = 1/(||h_j||^2 + N0/Ex)   (detect.cpp:86-90)
        nn[h] = mm[h] * e[h];                   // n_j = m_j ||h_j||^2
      }
    }
    const int base = lane & ~7;
    float4* bslots = reinterpret_cast<float4*>(sm + L::kBcOff) + 2 * q;
    for (int sw = 0; sw < K; ++sw) {
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp) {
        const int j0 = 2 * jp, j1 = 2 * jp + 1;
        // candidate on every lane from its own pair; the owner's (lane jp) is the update
        // x_j' = m_j d_j + n_j x_j, dx = x_j' - x_j   (detect.cpp:100-103)
        const float n0r = fmaf(mm[0], cr[0], nn[0] * xr[0]), n0i = fmaf(mm[0], ci[0], nn[0] * xi[0]);
        const float d0r = n0r - xr[0], d0i = n0i - xi[0];
        float c1r = cr[1], c1i = ci[1];
        csub_mul(c1r, c1i, d0r, d0i, g1r[j0], g1i[j0]);  // d_{j+1} = c_{j+1} - dx_j G_{j+1,j}
        const float n1r = fmaf(mm[1], c1r, nn[1] * xr[1]), n1i = fmaf(mm[1], c1i, nn[1] * xi[1]);
        const float d1r = n1r - xr[1], d1i = n1i - xi[1];
        const float4 bv = pair_bcast(make_float4(d0r, d0i, d1r, d1i), jp, k, base, bslots);
        const float a0r = bv.x, a0i = bv.y, a1r = bv.z, a1i = bv.w;
        if (k == jp) {
          xr[0] = n0r;
          xi[0] = n0i;
          xr[1] = n1r;
          xi[1] = n1i;
        }
        // r -= dx_j h_j + dx_{j+1} h_{j+1}  <=>  c_k -= dx_j G_kj + dx_{j+1} G_k,j+1
        csub_mul(cr[0], ci[0], a0r, a0i, g0r[j0], g0i[j0]);
        csub_mul(cr[0], ci[0], a1r, a1i, g0r[j1], g0i[j1]);
        csub_mul(cr[1], ci[1], a0r, a0i, g1r[j0], g1i[j0]);
        csub_mul(cr[1], ci[1], a1r, a1i, g1r[j1], g1i[j1]);
      }
    }
    const int p = set * NPW + q;
    if (p < P) {
      uint2 w;
      w.x = h2_as_u32(__floats2half2_rn(xr[0], xi[0]));
      w.y = h2_as_u32(__floats2half2_rn(xr[1], xi[1]));
      reinterpret_cast<uint2*>(X + static_cast<size_t>(p) * U)[k] = w;
    }
    if constexpr (SIG) {
      // optimal fusion: sigma^2 from the same Gram (the transit buffer is free
      // until the next set's tensor-core phase); rounded to the fp16 wire
      // format as the reference rounds the messages (detect.cpp:170-173)
      bool singular = false;
      float4* prow = reinterpret_cast<float4*>(sm + L::kGOff) + q * U;
#if DCDG_SIG_COLS
      // columns 2k, 2k+1 of the Hermitian A = I + gam G are the conjugated
      // rows this lane holds: forward elimination (gram_trace_inverse_cols)
      float2 Cr[U], Ci[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        Cr[i] = make_float2(fmaf(gam, g0r[i], i == 2 * k ? 1.f : 0.f), fmaf(gam, g1r[i], i == 2 * k + 1 ? 1.f : 0.f));
        Ci[i] = make_float2(-gam * g0i[i], -gam * g1i[i]);
      }
      const float tr = gram_trace_inverse_cols<U>(Cr, Ci, k, prow, singular);
#elif DCDG_GRAM_SIG_CPAIRS
      // A = I + gam G as column pairs, then the FFMA2 sweep operator (as ul_reg_f32's fused variance)
      float2 R0r[U / 2], R0i[U / 2], R1r[U / 2], R1i[U / 2];
#pragma unroll
      for (int jq = 0; jq < U / 2; ++jq) {
        R0r[jq] = make_float2(fmaf(gam, g0r[2 * jq], jq == k ? 1.f : 0.f), gam * g0r[2 * jq + 1]);
        R0i[jq] = make_float2(gam * g0i[2 * jq], gam * g0i[2 * jq + 1]);
        R1r[jq] = make_float2(gam * g1r[2 * jq], fmaf(gam, g1r[2 * jq + 1], jq == k ? 1.f : 0.f));
        R1i[jq] = make_float2(gam * g1i[2 * jq], gam * g1i[2 * jq + 1]);
      }
      const float tr = gram_trace_inverse_cpairs<U>(R0r, R0i, R1r, R1i, k, prow, singular);
#else
      const float tr = gram_trace_inverse<U>(g0r, g0i, g1r, g1i, k, gam, prow, singular);
#endif
      const unsigned sing = __ballot_sync(0xffffffffu, singular);
      if (p < P && k == 0) {
        sigma2[p] = __half2float(__float2half_rn(scale * tr));
        if ((sing >> (8 * q)) & 0xffu) record_status(status, p, ST_SINGULAR, 0);
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 16-B read-only global load, no L1 allocation, with an L2 eviction policy
__device__ __forceinline__ uint4 ldg_nc_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

#ifndef DCDG_DL_GRAM_PREFETCH
#define DCDG_DL_GRAM_PREFETCH 0  // lab switch, measured slower (profiles/lab/README.md)
#endif
__device__ __forceinline__ uint4 ldg_nc_l1(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// Gram-space downlink CD (Alg. 2 / Eq. 5, precode.cpp:52-99 on raw rows, as
// dl_reg_f16): every iterate is x = H a (a in C^U), so the dual update reads
// the channel only through w = H^H x = G a:
//     rho_u = q_u (w_u - s_u);  a_u -= rho_u;  w_k -= rho_u G_ku  for every k,
// with q_u = 1/||h_u||^2.  G comes from the tensor cores exactly as in the
// uplink kernel; the sweeps keep w and a in fp32 on the problem's 8 lanes
// (pairs of coordinates, the second corrected with G_{2k+1,2k}).  After the
// sweeps x = H a is formed on the CUDA cores from the problem's tile re-read
// from L2 (the TMA brought it in with evict-normal priority; the slot already
// holds the next set), then ||x||^2 gives power_scale (precode.cpp:101-111)
// and Re(s^H w) the effective-gain share (precode.cpp:123-131).
template <int U, int NPW, int MINB, bool GAIN>
__global__ void __launch_bounds__(32, MINB)
    dl_gram_f16(const __grid_constant__ CUtensorMap tmH, const __half2* __restrict__ H, const __half2* __restrict__ Sy,
                int P, int C, int K, float rho_c, __half2* __restrict__ X, float* __restrict__ gain_part,
                unsigned long long* __restrict__ status) {
  static_assert(NPW == 4, "a set is 4 problems of 8 sweep lanes");
  constexpr int BC = 32;
  using L = GramSmem<U, NPW>;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  unsigned char* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::kBarOff);
  const int lane = threadIdx.x & 31;
  const int q = lane >> 3, k = lane & 7;  // sweep: problem q of the set; lane k owns users 2k, 2k+1
  const int nsets = (P + NPW - 1) / NPW;
  int set = blockIdx.x;
  const uint64_t pol_keep = l2_evict_normal_policy(), pol_last_use = l2_evict_first_policy();
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int s) {
    mbar_arrive_expect_tx(bar, static_cast<uint32_t>(L::kSlotB));
    tma_load_2d(sm, &tmH, 0, s * NPW * U, bar, pol_keep);
  };
  if (lane == 0 && set < nsets) issue(set);
  uint32_t phase = 0;
  float4* abuf = reinterpret_cast<float4*>(sm + L::kYOff);  // a of the set's problems: [q][k] (a_2k, a_2k+1)
  for (; set < nsets; set += gridDim.x) {
    const int p = set * NPW + q;
    // s_{2k}, s_{2k+1} of the problem's subcarrier, in flight during the tensor-core phase
    uint32_t sw0 = 0, sw1 = 0;
    if (p < P) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(Sy + static_cast<size_t>(p / C) * U) + k);
      sw0 = v.x;
      sw1 = v.y;
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    float g0r[U], g0i[U], g1r[U], g1i[U];
    float unused_r[2], unused_i[2];
    gram_tc_phase<U, NPW, false>(sm, sbase, lane, g0r, g0i, g1r, g1i, unused_r, unused_i);
    fence_proxy_async_all();
    __syncwarp();
    if (lane == 0 && set + static_cast<int>(gridDim.x) < nsets) issue(set + gridDim.x);

    // ---------------- sweep phase (dual coordinates in fp32)
    float e[2];
#pragma unroll
    for (int jp = 0; jp < U / 2; ++jp)
      if (k == jp) {
        e[0] = g0r[2 * jp];      // ||h_2k||^2
        e[1] = g1r[2 * jp + 1];  // ||h_2k+1||^2
      }
    float qv[2], sqr[2], sqi[2];
    {
      const float2 s0 = __half22float2(u32_as_h2(sw0)), s1 = __half22float2(u32_as_h2(sw1));
      qv[0] = __frcp_rn(e[0]);
      qv[1] = __frcp_rn(e[1]);
      sqr[0] = qv[0] * s0.x;  // q_u s_u: the normalised symbol scaled by 1/||h_u|| (precode.cpp:80-87)
      sqi[0] = qv[0] * s0.y;
      sqr[1] = qv[1] * s1.x;
      sqi[1] = qv[1] * s1.y;
    }
    float ar[2] = {0.f, 0.f}, ai[2] = {0.f, 0.f}, wr[2] = {0.f, 0.f}, wi[2] = {0.f, 0.f};
    const int base = lane & ~7;
    float4* bslots = reinterpret_cast<float4*>(sm + L::kBcOff) + 2 * q;
    for (int sw = 0; sw < K; ++sw) {
#if DCDG_DL_GRAM_PREFETCH
      if (sw == K - 1 && p < P) {  // the tile's columns 2k, 2k+1 (one 128-B line each) into L1 for x = H a
        const char* hl = reinterpret_cast<const char*>(H) + static_cast<size_t>(p) * U * BC * 4 + (2 * k) * BC * 4;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(hl));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(hl + BC * 4));
      }
#endif
#pragma unroll
      for (int jp = 0; jp < U / 2; ++jp) {
        const int j0 = 2 * jp, j1 = 2 * jp + 1;
        // rho_u = q_u h_u^H x - q_u s_u  (precode.cpp:89-94, raw rows); the owner's (lane jp) is the update
        const float r0r = fmaf(qv[0], wr[0], -sqr[0]), r0i = fmaf(qv[0], wi[0], -sqi[0]);
        float f1r = wr[1], f1i = wi[1];
        csub_mul(f1r, f1i, r0r, r0i, g1r[j0], g1i[j0]);  // w_{j+1} after x -= rho_j h_j
        const float r1r = fmaf(qv[1], f1r, -sqr[1]), r1i = fmaf(qv[1], f1i, -sqi[1]);
        const float4 bv = pair_bcast(make_float4(r0r, r0i, r1r, r1i), jp, k, base, bslots);
        const float b0r = bv.x, b0i = bv.y, b1r = bv.z, b1i = bv.w;
        if (k == jp) {
          ar[0] -= r0r;
          ai[0] -= r0i;
          ar[1] -= r1r;
          ai[1] -= r1i;
        }
        // x -= rho_j h_j + rho_{j+1} h_{j+1}  <=>  w_k -= rho_j G_kj + rho_{j+1} G_k,j+1
        csub_mul(wr[0], wi[0], b0r, b0i, g0r[j0], g0i[j0]);
        csub_mul(wr[0], wi[0], b1r, b1i, g0r[j1], g0i[j1]);
        csub_mul(wr[1], wi[1], b0r, b0i, g1r[j0], g1i[j0]);
        csub_mul(wr[1], wi[1], b1r, b1i, g1r[j1], g1i[j1]);
      }
    }
    // ---------------- x = H a: lane k forms antennas 4k..4k+3 (its 16-B chunk of every column)
    abuf[q * (U / 2) + k] = make_float4(ar[0], ai[0], ar[1], ai[1]);
    __syncwarp();
    // antenna pairs (4k, 4k+1) and (4k+2, 4k+3) as packed fp32x2: the row-pair
    // planar tile words convert straight into FFMA2 operands
    float2 xr2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}, xi2[2] = {xr2[0], xr2[0]};
    if (p < P) {
      const unsigned char* hp = reinterpret_cast<const unsigned char*>(H) + static_cast<size_t>(p) * U * BC * 4 + k * 16;
      uint4 hv[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        hv[u] = DCDG_DL_GRAM_PREFETCH ? ldg_nc_l1(hp + u * BC * 4, pol_last_use) : ldg_nc_hint(hp + u * BC * 4, pol_last_use);
#pragma unroll
      for (int u2 = 0; u2 < U / 2; ++u2) {
        const float4 av = abuf[q * (U / 2) + u2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint4 v = hv[2 * u2 + h];
          const float aR = h ? av.z : av.x, aI = h ? av.w : av.y;
          const float2 hr[2] = {__half22float2(u32_as_h2(v.x)), __half22float2(u32_as_h2(v.z))};
          const float2 hi[2] = {__half22float2(u32_as_h2(v.y)), __half22float2(u32_as_h2(v.w))};
#pragma unroll
          for (int b = 0; b < 2; ++b) {  // x += h a: (hr ar - hi ai, hr ai + hi ar)
            xr2[b] = ffma2(aR, hr[b], ffma2(-aI, hi[b], xr2[b]));
            xi2[b] = ffma2(aI, hr[b], ffma2(aR, hi[b], xi2[b]));
          }
        }
      }
    }
    const float xr[4] = {xr2[0].x, xr2[0].y, xr2[1].x, xr2[1].y}, xi[4] = {xi2[0].x, xi2[0].y, xi2[1].x, xi2[1].y};
    float en = 0.f;
#pragma unroll
    for (int b = 0; b < 4; ++b) en = fmaf(xr[b], xr[b], fmaf(xi[b], xi[b], en));
    const float nrm = gsum<8>(en);
    const float gsc = rho_c > 0.f ? rho_c / __fsqrt_rn(nrm) : 1.f;  // power_scale, rho_c = rho/sqrt(C)
    float gq = 0.f;
    if (GAIN) {
      const float2 s0 = __half22float2(u32_as_h2(sw0)), s1 = __half22float2(u32_as_h2(sw1));
      // Re(s^H H^H x) = Re(s^H w), w = G a tracked through the sweeps
      gq = gsc * gsum<8>(fmaf(s0.x, wr[0], fmaf(s0.y, wi[0], fmaf(s1.x, wr[1], s1.y * wi[1]))));
    }
    if (p < P) {
      if (e[0] == 0.f)
        record_status(status, p, ST_ZERO_ROW, 2 * k);
      else if (e[1] == 0.f)
        record_status(status, p, ST_ZERO_ROW, 2 * k + 1);
      if (k == 0) {
        if (nrm == 0.f && rho_c > 0.f) record_status(status, p, ST_ZERO_BEAMFORMER, 0);
        if (GAIN) gain_part[p] = gq;
      }
      uint4 v;  // the precoder is interleaved complex (re, im) per antenna, antennas 4k..4k+3
      v.x = h2_as_u32(__floats2half2_rn(gsc * xr[0], gsc * xi[0]));
      v.y = h2_as_u32(__floats2half2_rn(gsc * xr[1], gsc * xi[1]));
      v.z = h2_as_u32(__floats2half2_rn(gsc * xr[2], gsc * xi[2]));
      v.w = h2_as_u32(__floats2half2_rn(gsc * xr[3], gsc * xi[3]));
      reinterpret_cast<uint4*>(X + static_cast<size_t>(p) * BC)[k] = v;
    }
    __syncwarp();  // abuf is rewritten by the next set
  }
}

}  // namespace dcdg
