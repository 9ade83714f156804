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

__device__ __forceinline__ void mma_f16f32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
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
  // one problem's G in transit from the mma fragments to the sweep lanes:
  // [k][col j][rows 2k, 2k+1] float2, k-stride padded 16 B (conflict-free)
  static constexpr int kGStride = U * 16 + 16;
  static constexpr int kGOff = kYOff + NPW * 128;
  static constexpr int kZOff = kGOff + (U / 2) * kGStride;  // z: [j] float2
  static constexpr int kBarOff = kZOff + U * 8;
  static constexpr int kBytes = kBarOff + 16;
  static constexpr int kAlloc = kBytes + 1024;      // slack to align the swizzled slot to 1024 B
};

// complex c -= a * b
__device__ __forceinline__ void csub_mul(float& cr, float& ci, float ar, float ai, float br, float bi) {
  cr = fmaf(-ar, br, fmaf(ai, bi, cr));
  ci = fmaf(-ar, bi, fmaf(-ai, br, ci));
}

template <int U, int NPW, int MINB>
__global__ void __launch_bounds__(32, MINB)
    ul_gram_f16(const __grid_constant__ CUtensorMap tmH, const __half2* __restrict__ Y, int P, int K, float kappa,
                __half2* __restrict__ X) {
  static_assert(NPW == 4, "a set is 4 problems of 8 sweep lanes");
  using L = GramSmem<U, NPW>;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  unsigned char* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::kBarOff);
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;  // mma fragment coordinates
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
  // ldmatrix row of this lane: matrix mi = lane/8 -> users (mi&1)*8 + lane%8, chunk half mi>>1
  const int lu = ((lane >> 3) & 1) * 8 + (lane & 7), lch = lane >> 4;
  unsigned char* gbuf = sm + L::kGOff;
  float2* zbuf = reinterpret_cast<float2*>(sm + L::kZOff);
  for (; set < nsets; set += gridDim.x) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    // rows 2k, 2k+1 of this lane's problem's G (fp32, registers) and c = z
    float g0r[U], g0i[U], g1r[U], g1i[U];
    float cr[2], ci[2];
    // ---------------- tensor-core phase: G and z of each problem, handed to its 8 sweep lanes
#pragma unroll
    for (int pl = 0; pl < NPW; ++pl) {
      float gr[2][4] = {}, gi[2][4] = {}, zz[4] = {};
      const int row = pl * U + lu;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t a[4];
        const int ch = 2 * ks + lch;
        ldsm_x4(a, sbase + row * L::kRowB + ((ch ^ (row & 7)) << 4));
        // B = W: n-tile 0 (users 0-7) = (a0, a2), n-tile 1 (users 8-15) = (a1, a3)
        mma_f16f32(gr[0], a, a[0], a[2]);
        mma_f16f32(gr[1], a, a[1], a[3]);
        mma_f16f32(gi[0], a, swap_neg(a[0], t), swap_neg(a[2], t));
        mma_f16f32(gi[1], a, swap_neg(a[1], t), swap_neg(a[3], t));
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
      __syncwarp();  // the previous problem's lanes have read the transit buffer
      // C fragments: (row g, cols 2t, 2t+1) and (row g+8, same cols) of each n-tile
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = nt * 8 + 2 * t + h;
          // row g -> (k = g/2, r = g%2); row g+8 -> (k = g/2 + 4, r = g%2)
          *reinterpret_cast<float2*>(gbuf + (g >> 1) * L::kGStride + j * 16 + (g & 1) * 8) =
              make_float2(gr[nt][h], gi[nt][h]);
          *reinterpret_cast<float2*>(gbuf + ((g >> 1) + 4) * L::kGStride + j * 16 + (g & 1) * 8) =
              make_float2(gr[nt][2 + h], gi[nt][2 + h]);
        }
      if (t == 0) {
        zbuf[g] = make_float2(zz[0], zz[1]);
        zbuf[g + 8] = make_float2(zz[2], zz[3]);
      }
      __syncwarp();
      if (q == pl) {
        const unsigned char* mine = gbuf + k * L::kGStride;
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(mine + j * 16);
          g0r[j] = v.x;
          g0i[j] = v.y;
          g1r[j] = v.z;
          g1i[j] = v.w;
        }
        const float4 zv = reinterpret_cast<const float4*>(zbuf)[k];
        cr[0] = zv.x;
        ci[0] = zv.y;
        cr[1] = zv.z;
        ci[1] = zv.w;
      }
    }
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
        const float a0r = __shfl_sync(0xffffffffu, d0r, base + jp);
        const float a0i = __shfl_sync(0xffffffffu, d0i, base + jp);
        const float a1r = __shfl_sync(0xffffffffu, d1r, base + jp);
        const float a1i = __shfl_sync(0xffffffffu, d1i, base + jp);
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
    __syncwarp();
  }
}

}  // namespace dcdg
