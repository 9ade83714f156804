// Microbenchmark: FFMA / FFMA2 / HFMA2 throughput (many independent chains,
// full occupancy) and dependent-chain latency on this GPU.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

template <int ILP>
__global__ void ffma_tp(float* out, int iters, float a, float b) {
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
template <int ILP>
__global__ void ffma2_tp(float* out, int iters, float a, float b) {
  float2 acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  const float2 aa = make_float2(a, a * 0.5f), bb = make_float2(b, b);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = __ffma2_rn(acc[i], aa, bb);
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}
template <int ILP>
__global__ void hfma2_tp(float* out, int iters, float a, float b) {
  __half2 acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = __float2half2_rn(threadIdx.x * 1e-3f + i);
  const __half2 aa = __float2half2_rn(a), bb = __float2half2_rn(b);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = __hfma2(acc[i], aa, bb);
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += __low2float(acc[i]);
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void shfl_tp(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], 1 << (i & 3));
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  float* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const double n = double(blocks) * threads * iters;
  float t;
  t = timeit([&] { ffma_tp<8><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f); });
  printf("FFMA  ILP8 : %.1f TFMA/s  (%.3f warp-inst/clk/SM at 1.9GHz)\n", n * 8 / t / 1e9, n * 8 / 32 / (t * 1e-3) / sms / 1.9e9);
  t = timeit([&] { ffma2_tp<8><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f); });
  printf("FFMA2 ILP8 : %.1f TFMA/s  (%.3f warp-inst/clk/SM)\n", n * 16 / t / 1e9, n * 8 / 32 / (t * 1e-3) / sms / 1.9e9);
  t = timeit([&] { hfma2_tp<8><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f); });
  printf("HFMA2 ILP8 : %.1f THFMA/s (%.3f warp-inst/clk/SM)\n", n * 16 / t / 1e9, n * 8 / 32 / (t * 1e-3) / sms / 1.9e9);
  t = timeit([&] { shfl_tp<<<blocks, threads>>>(out, iters); });
  printf("SHFL       : %.3f warp-inst/clk/SM\n", n * 8 / 32 / (t * 1e-3) / sms / 1.9e9);
  // latency: one warp per SM, single chain
  const int li = 1 << 16;
  t = timeit([&] { ffma_tp<1><<<sms, 32>>>(out, li, 1.0001f, 1e-7f); });
  printf("FFMA  latency ~ %.2f clk\n", (t * 1e-3) * 1.9e9 / li);
  t = timeit([&] { ffma2_tp<1><<<sms, 32>>>(out, li, 1.0001f, 1e-7f); });
  printf("FFMA2 latency ~ %.2f clk\n", (t * 1e-3) * 1.9e9 / li);
  t = timeit([&] { hfma2_tp<1><<<sms, 32>>>(out, li, 1.0001f, 1e-7f); });
  printf("HFMA2 latency ~ %.2f clk\n", (t * 1e-3) * 1.9e9 / li);
  t = timeit([&] { shfl_tp<<<sms, 32>>>(out, li / 8); });
  printf("SHFL+FADD chain ~ %.2f clk per step (8 indep chains interleaved)\n", (t * 1e-3) * 1.9e9 / li);
  return 0;
}
