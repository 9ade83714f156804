// Lab: where the time of one per-subcarrier decentralized_cd_detect call goes
// (B_c=32, U=16, C=8, fp32): each stage of the call timed on the host with a
// stream synchronisation after it, medians over 2000 calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "dcdg.h"

using Clock = std::chrono::steady_clock;
static double us(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double, std::micro>(b - a).count();
}
static double med(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  const int C = 8, Bc = 32, U = 16, K = 3, N = 2000;
  dcdg_ctx* ctx = nullptr;
  if (dcdg_init(0, &ctx) != DCDG_OK) return 1;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const size_t hb = size_t(C) * Bc * U * 8, yb = size_t(C) * Bc * 8, xb = size_t(C) * U * 8, xhb = U * 8;
  unsigned char *hin, *hout, *din, *dout;
  cudaMallocHost(&hin, hb + yb);
  cudaMallocHost(&hout, xb + xhb);
  cudaMalloc(&din, hb + yb);
  cudaMalloc(&dout, xb + xhb);
  std::vector<double> src(2 * (C * Bc * U + C * Bc));
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : src) v = nd(g);
  unsigned long long* sw;
  cudaMallocHost(&sw, 8);
  std::vector<double> t_pack, t_h2d, t_kern, t_fuse, t_d2h, t_all, t_fused_call;
  for (int it = 0; it < N + 50; ++it) {
    auto a = Clock::now();
    float* f = reinterpret_cast<float*>(hin);
    for (size_t i = 0; i < src.size(); ++i) f[i] = static_cast<float>(src[i]);
    auto b = Clock::now();
    cudaMemcpyAsync(din, hin, hb + yb, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    auto c = Clock::now();
    dcdg_ul_detect(ctx, din, din + hb, 1, C, C, Bc, U, K, 1.6, 1.0, DCDG_FP32, DCDG_FUSION_UNIFORM, dout, nullptr,
                   nullptr, nullptr, st);
    cudaStreamSynchronize(st);
    auto d = Clock::now();
    dcdg_fuse(ctx, dout, nullptr, 1, C, C, U, DCDG_FP32, DCDG_FUSION_UNIFORM, reinterpret_cast<float*>(dout + xb),
              nullptr, st);
    cudaStreamSynchronize(st);
    auto e = Clock::now();
    cudaMemcpyAsync(hout, dout, xb + xhb, cudaMemcpyDeviceToHost, st);
    dcdg_status_enqueue(ctx, sw, st);
    cudaStreamSynchronize(st);
    auto f2 = Clock::now();
    // the same work without intermediate synchronisations
    cudaMemcpyAsync(din, hin, hb + yb, cudaMemcpyHostToDevice, st);
    dcdg_ul_detect(ctx, din, din + hb, 1, C, C, Bc, U, K, 1.6, 1.0, DCDG_FP32, DCDG_FUSION_UNIFORM, dout, nullptr,
                   reinterpret_cast<float*>(dout + xb), nullptr, st);
    cudaMemcpyAsync(hout, dout, xb + xhb, cudaMemcpyDeviceToHost, st);
    dcdg_status_enqueue(ctx, sw, st);
    cudaStreamSynchronize(st);
    auto h = Clock::now();
    if (it >= 50) {
      t_pack.push_back(us(a, b));
      t_h2d.push_back(us(b, c));
      t_kern.push_back(us(c, d));
      t_fuse.push_back(us(d, e));
      t_d2h.push_back(us(e, f2));
      t_fused_call.push_back(us(f2, h));
    }
  }
  std::printf("{\"pack_us\": %.2f, \"h2d_sync_us\": %.2f, \"ul_detect_sync_us\": %.2f, \"fuse_sync_us\": %.2f, "
              "\"d2h_status_sync_us\": %.2f, \"one_stream_call_us\": %.2f}\n",
              med(t_pack), med(t_h2d), med(t_kern), med(t_fuse), med(t_d2h), med(t_fused_call));
  return 0;
}
