// Standalone post-equalization variance on the tensor cores (fp32 tiles):
//     sigma^2_p = (E_x/U) tr((I + (E_x/N0) G_p)^-1),  G_p = H_p^H H_p
// (post_eq_variance, src/detect.cpp:112-130; gram at :21-28), for the tile
// shapes whose CD kernel has no fused variance (ul_reg_f32<..., SIG> covers
// B_c = 32 with U = 8 and 16).
//
// Mapping: one warp per set of NPW = 64/U problems, U/2 lanes per problem in
// the factorisation (lane k keeps rows 2k, 2k+1 of A as column pairs).
//   * Gram: the whole warp, problem by problem, mma.sync.m16n8k8 TF32 with
//     fp32 accumulation and a 3-pass split x = hi + lo (hi = rna-TF32(x),
//     lo = rna-TF32(x - hi)): G = hi.hi + hi.lo + lo.hi, ~2^-21 relative to
//     |h|^2, with fp32 range (no scaling).  Used up to B_c = 256 (the launcher
//     keeps the FFMA Gram beyond, where the accumulation over 2 B_c real terms
//     reaches the 1e-5 parity edge).  k-order: thread t of k-step s takes complex row
//     4s + t, its re on k = t and its im on k = t + 4 (one 8-B load per user),
//     so W' = (im, -re) is a register swap and a sign flip.  Tiles are read
//     straight from global memory (each element once per problem).
//   * A = I + gam G goes to a per-problem column-pair image in shared memory;
//     the U/2 lanes read their rows and run the column-pair FFMA2 sweep
//     operator (gram_trace_inverse_cpairs): 16 or 32 pivots in ascending
//     order, the reference's pivot test (numerics.cpp:38-41,55-56).
#pragma once

#include <type_traits>

#include "dcdg_device.cuh"

namespace dcdg {

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// hi = rna-TF32(x), lo = rna-TF32(x - hi)
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - __uint_as_float(hi));
}

// D += A B, mma.sync m16n8k8, TF32 operands, fp32 accumulate
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int U>
struct PevTcSmem {
  static constexpr int kNpw = 64 / U;                      // problems per warp
  static constexpr int kImgB = U * (U / 2) * 16;            // column-pair image of one problem
  static constexpr int kRowB = 2 * (U / 2) * 16;            // pivot-row broadcast of one problem
  static constexpr int kWarpB = kNpw * (kImgB + kRowB);
};

// fp16 tiles (row-pair planar {re_2i, re_2i+1, im_2i, im_2i+1}): the stored
// binary16 values are multiplied exactly (mma.sync.m16n8k16, fp32
// accumulate), one pass per tile; thread t of k-step s takes row pair 4s + t,
// its re pair on k 2t, 2t+1 and its im pair on k 2t+8, 2t+9 (one 8-B load
// per user), W' = (im, -re) again a swap and a sign flip; sigma^2 is rounded
// to the fp16 wire format as the reference rounds its messages
// (detect.cpp:170-173).
template <int U, int MINB, typename T = float2>
__global__ void __launch_bounds__(32, MINB)
    pev_tc_kernel(const T* __restrict__ Hin, int P, int BC, float gam, float scale, float* __restrict__ sigma2,
                  unsigned long long* __restrict__ status) {
  constexpr bool F16 = std::is_same_v<T, __half2>;
  static_assert(U == 8 || U == 16 || U == 32, "U in {8, 16, 32}");
  using L = PevTcSmem<U>;
  constexpr int NPW = L::kNpw, MT = (U + 15) / 16, NT = U / 8, NQ = U / 2;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x;
  const int mg = lane >> 2, mt = lane & 3;           // mma fragment coordinates
  const int q = lane / NQ, k = lane % NQ;            // factorisation: problem q of the set, rows 2k, 2k+1
  float4* img_all = reinterpret_cast<float4*>(smem);
  float4* prow_all = reinterpret_cast<float4*>(smem + NPW * L::kImgB);
  const int nsets = (P + NPW - 1) / NPW;
  // the tiles are read once, straight from global memory: the next set is
  // prefetched into L2 one set ahead (one bulk prefetch per set)
  auto prefetch = [&](int s_) {
    if (lane == 0 && s_ < nsets) {
      const int p0 = s_ * NPW, n = min(NPW, P - p0);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                       reinterpret_cast<const unsigned char*>(Hin) + static_cast<size_t>(p0) * BC * U * sizeof(T)),
                   "r"(static_cast<uint32_t>(n * BC * U * sizeof(T)))
                   : "memory");
    }
  };
  prefetch(blockIdx.x);
  for (int set = blockIdx.x; set < nsets; set += gridDim.x) {
    prefetch(set + gridDim.x);
    // ---- Gram of each problem of the set on the tensor cores -> image of A
#pragma unroll 1
    for (int pl = 0; pl < NPW; ++pl) {
      const int pc = min(set * NPW + pl, P - 1);
      float gr[MT][NT][4] = {}, gi[MT][NT][4] = {};
      if constexpr (F16) {
        const uint2* h2 = reinterpret_cast<const uint2*>(Hin) + static_cast<size_t>(pc) * (BC / 2) * U;
        // chunks of KC k-steps: every load of a chunk in flight before its mma
        constexpr int KC = 4;
        const int nks = BC / 8;
#pragma unroll 1
        for (int ks0 = 0; ks0 < nks; ks0 += KC) {
          uint2 v[KC][MT][2];
#pragma unroll
          for (int c = 0; c < KC; ++c)
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int u = 16 * m + mg + 8 * hh;
                v[c][m][hh] = (ks0 + c < nks && u < U) ? h2[static_cast<size_t>(u) * (BC / 2) + 4 * (ks0 + c) + mt]
                                                      : make_uint2(0u, 0u);
              }
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            if (ks0 + c >= nks) break;
            uint32_t a[MT][4];
#pragma unroll
            for (int m = 0; m < MT; ++m) {
              a[m][0] = v[c][m][0].x;  // re pair of row pair 4ks + mt: k 2mt, 2mt+1
              a[m][2] = v[c][m][0].y;  // im pair: k 2mt+8, 2mt+9
              a[m][1] = v[c][m][1].x;
              a[m][3] = v[c][m][1].y;
            }
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
              for (int n = 0; n < NT; ++n) {
                const int bm = n >> 1, bo = n & 1;
                const uint32_t b0 = a[bm][bo], b1 = a[bm][2 + bo];
                mma_f16f32(gr[m][n], a[m], b0, b1);
                mma_f16f32(gi[m][n], a[m], b1, b0 ^ 0x80008000u);
              }
          }
        }
      } else {
        const float2* h = reinterpret_cast<const float2*>(Hin) + static_cast<size_t>(pc) * BC * U;
        constexpr int KC = 8;
        const int nks = BC / 4;
#pragma unroll 1
        for (int ks0 = 0; ks0 < nks; ks0 += KC) {
          float2 v[KC][MT][2];
#pragma unroll
          for (int c = 0; c < KC; ++c)
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int u = 16 * m + mg + 8 * hh;
                v[c][m][hh] = (ks0 + c < nks && u < U) ? h[static_cast<size_t>(u) * BC + 4 * (ks0 + c) + mt]
                                                      : make_float2(0.f, 0.f);
              }
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            if (ks0 + c >= nks) break;
            uint32_t ah[MT][4], al[MT][4];
#pragma unroll
            for (int m = 0; m < MT; ++m) {
              split_tf32(v[c][m][0].x, ah[m][0], al[m][0]);  // re: k = mt
              split_tf32(v[c][m][0].y, ah[m][2], al[m][2]);  // im: k = mt + 4
              split_tf32(v[c][m][1].x, ah[m][1], al[m][1]);
              split_tf32(v[c][m][1].y, ah[m][3], al[m][3]);
            }
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
              for (int n = 0; n < NT; ++n) {
                // B column users 8n + mg: registers of m-tile n/2, rows (n & 1) ? +8 : +0
                const int bm = n >> 1, bo = n & 1;
                const uint32_t bh0 = ah[bm][bo], bh1 = ah[bm][2 + bo], bl0 = al[bm][bo], bl1 = al[bm][2 + bo];
                mma_tf32(gr[m][n], ah[m], bh0, bh1);
                mma_tf32(gr[m][n], ah[m], bl0, bl1);
                mma_tf32(gr[m][n], al[m], bh0, bh1);
                // W' = (im, -re): k = mt takes im, k = mt + 4 takes -re
                mma_tf32(gi[m][n], ah[m], bh1, bh0 ^ 0x80000000u);
                mma_tf32(gi[m][n], ah[m], bl1, bl0 ^ 0x80000000u);
                mma_tf32(gi[m][n], al[m], bh1, bh0 ^ 0x80000000u);
              }
          }
        }
      }  // F16
      // C fragment: [0..1] row 16m + mg, cols 8n + 2mt, +1; [2..3] row 16m + mg + 8
      float4* img = img_all + pl * (L::kImgB / 16);
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int i = 16 * m + mg + 8 * hh;
            if (i >= U) continue;
            const int jq = 4 * n + mt, j0 = 2 * jq;
            img[apair_slot<U>(i, jq)] =
                make_float4(fmaf(gam, gr[m][n][2 * hh], i == j0 ? 1.f : 0.f),
                            fmaf(gam, gr[m][n][2 * hh + 1], i == j0 + 1 ? 1.f : 0.f), gam * gi[m][n][2 * hh],
                            gam * gi[m][n][2 * hh + 1]);
          }
    }
    __syncwarp();
    // ---- factorisation: lane k of problem q takes rows 2k, 2k+1 of A
#if DCDG_SIG_COLS
    float2 Cr[U], Ci[U];
    {
      const float4* a4 = img_all + q * (L::kImgB / 16);
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const float4 a = a4[apair_slot<U>(i, k)];
        Cr[i] = make_float2(a.x, a.y);
        Ci[i] = make_float2(a.z, a.w);
      }
    }
    bool singular = false;
    float4* prow = prow_all + q * (L::kRowB / 16);
    const float tr = gram_trace_inverse_cols<U>(Cr, Ci, k, prow, singular);
#else
    float2 R0r[NQ], R0i[NQ], R1r[NQ], R1i[NQ];
    {
      const float4* a4 = img_all + q * (L::kImgB / 16);
#pragma unroll
      for (int jq = 0; jq < NQ; ++jq) {
        const float4 a = a4[apair_slot<U>(2 * k, jq)], b = a4[apair_slot<U>(2 * k + 1, jq)];
        R0r[jq] = make_float2(a.x, a.y);
        R0i[jq] = make_float2(a.z, a.w);
        R1r[jq] = make_float2(b.x, b.y);
        R1i[jq] = make_float2(b.z, b.w);
      }
    }
    bool singular = false;
    float4* prow = prow_all + q * (L::kRowB / 16);
    const float tr = U <= DCDG_PEV_TC_BLOCK2_MAXU ? gram_trace_inverse_cpairs2<U>(R0r, R0i, R1r, R1i, k, prow, singular)
                                       : gram_trace_inverse_cpairs<U>(R0r, R0i, R1r, R1i, k, prow, singular);
#endif
    const unsigned sing = __ballot_sync(0xffffffffu, singular);
    const int p = set * NPW + q;
    if (p < P && k == 0) {
      sigma2[p] = F16 ? __half2float(__float2half_rn(scale * tr)) : scale * tr;
      if ((sing >> (NQ * q)) & static_cast<unsigned>((1ull << NQ) - 1)) record_status(status, p, ST_SINGULAR, 0);
    }
    __syncwarp();  // the image and pivot rows are reused by the next set
  }
}

}  // namespace dcdg
