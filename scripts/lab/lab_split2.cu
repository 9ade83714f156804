// Kernel lab (not part of the product): split-tile uplink variants at one
// (B_c, U) shape, timed on identical random inputs; maxrel is against the
// first variant.  -DLAB_BC=.. -DLAB_U=.. -DVARIANTS='V(G,JR,MINB) V(...)'
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1902_08653_b200/csrc -I scripts/lab \
//        -DLAB_BC=64 -DLAB_U=32 -DLAB_VARIANTS='"v.h"' scripts/lab/lab_split2.cu -o lab/x   (v.h: V(16,16,8) V(16,12,8) ...)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dcdg_split_kernels.cuh"

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
constexpr int BC = LAB_BC, U = LAB_U, K = 3;
static int g_sms = 148;
static std::vector<float2> g_first;

template <int G, int JR, int MINB>
void run(const float2* H, const float2* Y, float2* X, int P, int reps, double bytes) {
  constexpr int NPW = 32 / G;
  const size_t smem = dcdg::split_cols_bytes(BC, U, JR, G) + NPW * dcdg::ul_scal_bytes(U, 2);
  auto k = dcdg::ul_split_f32<BC, U, G, JR, MINB, 1>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32, smem));
  cudaFuncAttributes at;
  CK(cudaFuncGetAttributes(&at, k));
  const int blocks = std::min((P + NPW - 1) / NPW, g_sms * occ);
  auto launch = [&] { k<<<blocks, 32, smem>>>(H, Y, P, K, 1.6f, X); };
  CK(cudaMemset(X, 0, (size_t)P * U * 8));
  launch();
  CK(cudaDeviceSynchronize());
  std::vector<float2> x((size_t)P * U);
  CK(cudaMemcpy(x.data(), X, x.size() * 8, cudaMemcpyDeviceToHost));
  double mx = 0;
  if (g_first.empty()) g_first = x;
  for (int p = 0; p < P; ++p) {
    double num = 0, den = 0;
    for (int u = 0; u < U; ++u) {
      const float2 a = g_first[(size_t)p * U + u], b = x[(size_t)p * U + u];
      num += (double)(a.x - b.x) * (a.x - b.x) + (double)(a.y - b.y) * (a.y - b.y);
      den += (double)a.x * a.x + (double)a.y * a.y;
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
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  std::printf("BC=%d U=%d G=%2d JR=%2d MINB=%2d  %8.4f ms  %5.1f%% of 6546.6  occ %2d regs %3d smem %6zu maxrel %.2e\n", BC,
              U, G, JR, MINB, ms, 100.0 * bytes / ms / 1e6 / 6546.6, occ, at.numRegs, smem, mx);
}

int main(int argc, char** argv) {
  const int P = argc > 1 ? std::atoi(argv[1]) : 65536, reps = argc > 2 ? std::atoi(argv[2]) : 20;
  CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
  float2 *H, *Y, *X;
  CK(cudaMalloc(&H, (size_t)P * BC * U * 8));
  CK(cudaMalloc(&Y, (size_t)P * BC * 8));
  CK(cudaMalloc(&X, (size_t)P * U * 8));
  fill_normal<<<1184, 256>>>((float*)H, (size_t)P * BC * U * 2, 1u, 0.70710678f);
  fill_normal<<<1184, 256>>>((float*)Y, (size_t)P * BC * 2, 2u, 2.8f);
  CK(cudaDeviceSynchronize());
  const double bytes = (double)P * (BC * U + BC + U) * 8;
#define V(G, JR, MINB) run<G, JR, MINB>(H, Y, X, P, reps, bytes);
#include LAB_VARIANTS
  return 0;
}
