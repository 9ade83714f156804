// Kernel lab (not part of the product): times candidate CD kernel variants
// against the current register-resident kernel at the north-star shape
// (B_c=32, U=16, K=3, 134,400 problems) on identical random inputs and
// reports the max per-problem relative difference to it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo \
//        -I paper_1902_08653_b200/csrc scripts/lab/lab_split.cu -o lab/lab_split
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#include "dcdg_split_kernels.cuh"

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

__global__ void fill_normal(float* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = (uint32_t)i * 2654435761u ^ seed, b = (uint32_t)(i >> 32) + 0x9e3779b9u * seed;
    a ^= a >> 16; a *= 0x7feb352du; a ^= a >> 15; a *= 0x846ca68bu; a ^= a >> 16;
    b ^= a; b ^= b >> 16; b *= 0x7feb352du; b ^= b >> 15; b *= 0x846ca68bu; b ^= b >> 16;
    const float u1 = (a >> 8) * (1.f / 16777216.f) + 1e-7f, u2 = (b >> 8) * (1.f / 16777216.f);
    p[i] = scale * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
  }
}

#ifndef LAB_U
#define LAB_U 16
#endif
#ifndef LAB_GREF
#define LAB_GREF 8
#endif
constexpr int BC = 32, U = LAB_U, K = 3;
static int g_sms = 148;

template <typename Kern>
int occ_of(Kern k, size_t smem, int threads) {
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem));
  return occ;
}

struct Result {
  const char* name;
  float ms;
  double maxrel;
  int occ;
  int regs;
};

template <typename Launch>
Result run(const char* name, Launch launch, int occ, int regs, const float2* Xref, float2* X, int P, int reps) {
  CK(cudaMemset(X, 0, (size_t)P * U * 8));
  launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float2> a((size_t)P * U), b((size_t)P * U);
  CK(cudaMemcpy(a.data(), Xref, a.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), X, b.size() * 8, cudaMemcpyDeviceToHost));
  double mx = 0;
  for (int p = 0; p < P; ++p) {
    double num = 0, den = 0;
    for (int u = 0; u < U; ++u) {
      const float2 x = a[(size_t)p * U + u], y = b[(size_t)p * U + u];
      num += (double)(x.x - y.x) * (x.x - y.x) + (double)(x.y - y.y) * (x.y - y.y);
      den += (double)x.x * x.x + (double)x.y * x.y;
    }
    const double r = std::sqrt(num / (den > 0 ? den : 1));
    if (!(r <= mx)) mx = r;
  }
  for (int i = 0; i < 3; ++i) launch();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return {name, ms / reps, mx, occ, regs};
}

template <typename Kern>
int regs_of(Kern k) {
  cudaFuncAttributes at;
  CK(cudaFuncGetAttributes(&at, k));
  return at.numRegs;
}

template <int JR, int MINB, int PF, int G = 8>
Result run_split(const char* name, const float2* H, const float2* Y, float kappa, const float2* Xref, float2* X, int P,
                 int reps) {
  constexpr int NPW = 32 / G;
  const size_t smem = dcdg::split_cols_bytes(BC, U, JR, G) + NPW * dcdg::ul_scal_bytes(U, 2);
  auto k = dcdg::ul_split_f32<BC, U, G, JR, MINB, PF>;
  const int occ = occ_of(k, smem, 32);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min(nsets, g_sms * occ);
  return run(name, [&] { k<<<blocks, 32, smem>>>(H, Y, P, K, kappa, X); }, occ, regs_of(k), Xref, X, P, reps);
}

int main(int argc, char** argv) {
  const int S = argc > 1 ? std::atoi(argv[1]) : 16800;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 20;
  const int P = S * 8;
  CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
  float2 *H, *Y, *Xref, *X;
  CK(cudaMalloc(&H, (size_t)P * BC * U * 8));
  CK(cudaMalloc(&Y, (size_t)P * BC * 8));
  CK(cudaMalloc(&Xref, (size_t)P * U * 8));
  CK(cudaMalloc(&X, (size_t)P * U * 8));
  fill_normal<<<1184, 256>>>((float*)H, (size_t)P * BC * U * 2, 1u, 0.70710678f);
  fill_normal<<<1184, 256>>>((float*)Y, (size_t)P * BC * 2, 2u, 2.8f);
  CK(cudaDeviceSynchronize());
  const float kappa = 1.6f;
  const double bytes = (double)P * (BC * U + BC + U) * 8;
  std::printf("U=%d, %d problems\n", U, P);

  // the current hot-path kernel (reference for timing and results)
  std::vector<Result> res;
  {
    constexpr int G = LAB_GREF, NPW = 32 / G, LB = 2;
    constexpr size_t smem = dcdg::CtaSmem<NPW*(BC * U * 8 + BC * 8), dcdg::ul_scal_bytes(U, LB), NPW, 1>::kBytes;
    auto k = dcdg::ul_reg_f32<BC, U, G, 1, 8, LB>;
    const int occ = occ_of(k, smem, 32);
    const int blocks = std::min((P + NPW - 1) / NPW, g_sms * occ);
    auto launch = [&] { k<<<blocks, 32, smem>>>(H, Y, P, K, kappa, Xref, dcdg::XMap{}); };
    launch();
    CK(cudaDeviceSynchronize());
    res.push_back(run("ul_reg_f32 (current)", launch, occ, regs_of(k), Xref, Xref, P, reps));
    res.back().maxrel = 0;
  }
#if LAB_U == 32
  res.push_back(run_split<16, 8, 1, 8>("split U=32 G=8 JR=16 MINB=8", H, Y, kappa, Xref, X, P, reps));
  res.push_back(run_split<12, 8, 1, 8>("split U=32 G=8 JR=12 MINB=8", H, Y, kappa, Xref, X, P, reps));
  res.push_back(run_split<8, 12, 1, 8>("split U=32 G=8 JR=8 MINB=12", H, Y, kappa, Xref, X, P, reps));
  res.push_back(run_split<16, 12, 1, 16>("split U=32 G=16 JR=16 MINB=12", H, Y, kappa, Xref, X, P, reps));
  res.push_back(run_split<16, 16, 1, 16>("split U=32 G=16 JR=16 MINB=16", H, Y, kappa, Xref, X, P, reps));
#else
  res.push_back(run_split<8, 16, 1>("split G=8 JR=8 MINB=16 PF=1", H, Y, kappa, Xref, X, P, reps));
#endif
  for (const auto& r : res)
    std::printf("%-34s %8.4f ms  %7.1f GB/s  %5.1f%% of 6546.6  occ %2d  regs %3d  maxrel %.2e\n", r.name, r.ms,
                bytes / r.ms / 1e6, 100.0 * bytes / r.ms / 1e6 / 6546.6, r.occ, r.regs, r.maxrel);
  return 0;
}
