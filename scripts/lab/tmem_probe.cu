// Lab: TMEM as register spill space for the CD tile (sm_100a).
// 4-warp CTA allocates 128 columns; each warp stores 32 regs per lane to its
// lane quarter with tcgen05.st.32x32b.x32, loads them back with
// tcgen05.ld.32x32b.x32 and checks them; then times a dependent chain of
// ld -> wait -> FFMA and a throughput loop of loads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_st32(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tm_ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr));
}

__global__ void __launch_bounds__(128) probe(int* err, long long* cyc, float* sink, int iters) {
  __shared__ uint32_t base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&base_s))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = base_s + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
  uint32_t v[32], w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = (blockIdx.x * 128 + threadIdx.x) * 64 + i;
  tm_st32(base, v);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  tm_ld32(base, w);
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  int bad = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) bad += (w[i] != v[i]);
  if (bad) atomicAdd(err, bad);
  // dependent chain: ld -> wait -> use -> next address
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    tm_ld32(base + (static_cast<uint32_t>(acc == 12345.f) << 5), w);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    acc += __uint_as_float(w[0] & 0x3fffffff) * 1e-30f;
  }
  long long t1 = clock64();
  // throughput: independent loads, one wait per 4
  for (int it = 0; it < iters; it += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      tm_ld32(base, w);
      acc += __uint_as_float(w[u]) * 1e-30f;
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;");
  }
  long long t2 = clock64();
  if (lane == 0 && blockIdx.x == 0) {
    cyc[warp * 2] = (t1 - t0) / iters;
    cyc[warp * 2 + 1] = (t2 - t1) / iters;
  }
  sink[blockIdx.x * 128 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base_s));
}

int main() {
  int* err;
  long long* cyc;
  float* sink;
  cudaMalloc(&err, 4);
  cudaMalloc(&cyc, 64);
  cudaMalloc(&sink, 148 * 4 * 128 * 4);
  cudaMemset(err, 0, 4);
  for (int ctas : {1, 148, 592}) {
    probe<<<ctas, 128>>>(err, cyc, sink, 1024);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1;
    long long c[8];
    cudaMemcpy(&h, err, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(c, cyc, 64, cudaMemcpyDeviceToHost);
    std::printf("ctas %d: %s, mismatches %d, dependent ld+wait %lld cyc, throughput %lld cyc/ld (warp 0)\n", ctas,
                cudaGetErrorString(e), h, c[0], c[1]);
  }
  return 0;
}
