// Kernel lab (not part of the product): downlink CD kernel variants at the
// north-star shape, timed against each other on identical random inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo \
//        -I paper_1902_08653_b200/csrc scripts/lab/lab_dl.cu -o lab/lab_dl
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "dcdg_reg_kernels.cuh"
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)
__global__ void fill_normal(float* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = (uint32_t)i * 2654435761u ^ seed, b = (uint32_t)(i >> 32) + 0x9e3779b9u * seed;
    a ^= a >> 16; a *= 0x7feb352du; a ^= a >> 15; a *= 0x846ca68bu; a ^= a >> 16;
    b ^= a; b ^= b >> 16; b *= 0x7feb352du; b ^= b >> 15; b *= 0x846ca68bu; b ^= b >> 16;
    const float u1 = (a >> 8) * (1.f / 16777216.f) + 1e-7f, u2 = (b >> 8) * (1.f / 16777216.f);
    p[i] = scale * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
  }
}
constexpr int BC = 32, U = 16, K = 3, C = 8;
static int g_sms = 148;
template <int MINB>
float run_dl(const float2* H, const float2* S, int P, float2* X, int reps, int* occ_out, int* regs_out) {
  constexpr int G = 8, NPW = 4;
  constexpr size_t smem = dcdg::CtaSmem<NPW*(BC * U * 8 + U * 8), dcdg::dl_scal_bytes(U), NPW, 1>::kBytes;
  auto k = dcdg::dl_reg_f32<BC, U, G, 1, MINB, false>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32, smem));
  cudaFuncAttributes at; CK(cudaFuncGetAttributes(&at, k));
  *occ_out = occ; *regs_out = at.numRegs;
  const int blocks = std::min((P + NPW - 1) / NPW, g_sms * occ);
  auto launch = [&] { k<<<blocks, 32, smem>>>(H, S, P, C, K, 1.41421356f, X, nullptr, nullptr); };
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}
int main(int argc, char** argv) {
  const int S = argc > 1 ? std::atoi(argv[1]) : 16800, reps = argc > 2 ? std::atoi(argv[2]) : 20;
  const int P = S * C;
  CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
  float2 *H, *Sy, *X;
  CK(cudaMalloc(&H, (size_t)P * BC * U * 8)); CK(cudaMalloc(&Sy, (size_t)S * U * 8)); CK(cudaMalloc(&X, (size_t)P * BC * 8));
  fill_normal<<<1184, 256>>>((float*)H, (size_t)P * BC * U * 2, 1u, 0.70710678f);
  fill_normal<<<1184, 256>>>((float*)Sy, (size_t)S * U * 2, 2u, 0.70710678f);
  const double bytes = (double)P * (BC * U + BC + U) * 8;
  int occ, regs; float ms;
#define RUN(M) ms = run_dl<M>(H, Sy, P, X, reps, &occ, &regs); \
  std::printf("dl_reg_f32 MINB=%2d  %8.4f ms  %5.1f%% of 6546.6  occ %2d regs %3d\n", M, ms, 100.0 * bytes / ms / 1e6 / 6546.6, occ, regs);
  RUN(8) RUN(10) RUN(12) RUN(16)
  return 0;
}
