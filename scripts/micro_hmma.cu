// Microbenchmark: legacy tensor-core path (mma.sync m16n8k16, f16 inputs,
// f32 accumulate; SASS HMMA) throughput and dependent latency on this GPU.
// Sizes the Gram-space fp16 kernel (dcdg_gram_kernels.cuh): each cluster
// problem's Gram + matched filter is 16 of these.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mh scripts/micro_hmma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma16816(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int ILP>
__global__ void hmma_tp(float* out, int iters) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x << 3);
  b[0] = 0x3c003c00u;
  b[1] = 0x38003800u;
  float d[ILP][4] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) mma16816(d[i], a, b);
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4096);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  auto run = [&](auto kern, int ilp, int warps_per_sm, const char* name) {
    const int threads = 128, blocks = sms * warps_per_sm / 4;
    kern<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = double(blocks) * 4 * iters * ilp;  // warp-level mma instructions
    const double tflops = mmas * 4096 / (ms * 1e-3) / 1e12;
    printf("%-10s warps/SM %2d ILP %d: %.3f ms, %.2f mma/clk/SM @1.965GHz, %.1f TFLOP/s\n", name, warps_per_sm, ilp,
           ms, mmas / (ms * 1e-3) / 1.965e9 / sms, tflops);
  };
  run(hmma_tp<1>, 1, 4, "hmma");
  run(hmma_tp<1>, 1, 16, "hmma");
  run(hmma_tp<4>, 4, 16, "hmma");
  run(hmma_tp<4>, 4, 32, "hmma");
  run(hmma_tp<8>, 8, 32, "hmma");
  // dependent latency: 1 warp per SM, ILP 1
  run(hmma_tp<1>, 1, 1, "hmma-lat");
  return 0;
}
