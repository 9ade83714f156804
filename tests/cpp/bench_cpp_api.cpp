// Latency / throughput of the C++ drop-in surface (include/dcd_gpu.hpp) at the
// north-star shape (B=256, U=16, C=8 -> B_c=32, K=3), the numbers a
// maintainer swapping dcd:: for dcd::gpu:: at the reference's call sites
// (src/cluster.cpp:151-152 and :253-254) would see:
//   * per call: dcd::gpu::decentralized_cd_detect / _precode on one
//     subcarrier (host fp64 in, host fp64 out: pack, one H2D, kernels, one
//     D2H, unpack), median over many calls on a warm Engine;
//   * batched round: decentralized_cd_detect_batch / _precode_batch over a
//     1200 x 14 subcarrier-symbol round, host to host;
//   * next to the reference's own decentralized_cd_detect per call (one
//     thread), when oracle/_ref/libdcdref.so (the reference compiled from its
//     sources; test infrastructure) is present.
// Prints one JSON object.  Built and run by tests/test_cpp_api.py (-m gpu,
// --quick) and by hand for profiles/.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "dcd_gpu.hpp"

using namespace dcd::gpu;
using Clock = std::chrono::steady_clock;

namespace {
std::mt19937_64 g_rng(7);
cf64 randc() {
  static std::normal_distribution<double> g(0.0, std::sqrt(0.5));
  return {g(g_rng), g(g_rng)};
}
ComplexMatrix rmat(std::size_t r, std::size_t c) {
  ComplexMatrix m(r, c);
  for (auto& z : m.flat()) z = randc();
  return m;
}
ComplexVector rvec(std::size_t n) {
  ComplexVector v(n);
  for (auto& z : v) z = randc();
  return v;
}
double us_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::micro>(Clock::now() - t0).count();
}
double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

// the reference's decentralized_cd_detect, one thread, on prebuilt host data
double reference_us_per_call(int S, const std::vector<std::vector<ClusterData>>& subs, int C, int Bc, int U) {
  void* so = dlopen("oracle/_ref/libdcdref.so", RTLD_NOW);
  if (!so) return -1.0;
  using Create = void* (*)(int, int, int, int, const double*, const double*);
  using Run = double (*)(void*, double, double, unsigned, int, int, int, int, int, int, double*);
  using Destroy = void (*)(void*);
  auto create = reinterpret_cast<Create>(dlsym(so, "dcdref_ul_batch_create"));
  auto run = reinterpret_cast<Run>(dlsym(so, "dcdref_ul_batch_run"));
  auto destroy = reinterpret_cast<Destroy>(dlsym(so, "dcdref_ul_batch_destroy"));
  if (!create || !run || !destroy) return -1.0;
  std::vector<double> h, y;
  for (int s = 0; s < S; ++s)
    for (int c = 0; c < C; ++c) {
      for (auto z : subs[s][c].h.flat()) h.insert(h.end(), {z.real(), z.imag()});
      for (auto z : subs[s][c].y) y.insert(y.end(), {z.real(), z.imag()});
    }
  void* b = create(S, C, Bc, U, h.data(), y.data());
  run(b, 1.6, 1.0, 3, 1, 0, 0, 1, 0, S, nullptr);  // warm
  const double t = run(b, 1.6, 1.0, 3, 1, 0, 0, 1, 0, S, nullptr);
  destroy(b);
  return t * 1e6 / S;
}
}  // namespace

int main(int argc, char** argv) {
  const bool quick = argc > 1 && std::strcmp(argv[1], "--quick") == 0;
  const int C = 8, Bc = 32, U = 16, BITS = 4;
  const int calls = quick ? 50 : 2000;
  const int S_round = quick ? 1200 : 1200 * 14;
  Engine& eng = default_engine();

  // ---- per-call latency (one subcarrier per call, the reference signature)
  std::vector<ClusterData> cl(C);
  for (auto& c : cl) c = {rmat(Bc, U), rvec(Bc)};
  DetectorConfig cfg;
  cfg.n0 = 1.6;  // 10 dB at U=16
  cfg.fusion = FusionMode::uniform;
  auto per_call = [&](auto&& fn) {
    for (int i = 0; i < 20; ++i) fn();
    std::vector<double> t(calls);
    for (int i = 0; i < calls; ++i) {
      const auto t0 = Clock::now();
      fn();
      t[i] = us_since(t0);
    }
    return median(t);
  };
  const double ul_us = per_call([&] { decentralized_cd_detect(cl, cfg); });
  DetectorConfig cfg_opt = cfg;
  cfg_opt.fusion = FusionMode::optimal;
  const double ul_opt_us = per_call([&] { decentralized_cd_detect(cl, cfg_opt); });
  std::vector<ComplexMatrix> blocks;
  for (auto& c : cl) blocks.push_back(c.h.hermitian());
  const ComplexVector sym = rvec(U);
  PrecoderConfig pcfg;
  pcfg.rho = 4.0;
  const double dl_us = per_call([&] { decentralized_cd_precode(blocks, sym, pcfg); });

  // ---- batched round, host to host
  std::vector<std::vector<ClusterData>> subs(S_round);
  std::vector<std::vector<ComplexMatrix>> dblocks(S_round);
  std::vector<ComplexVector> syms(S_round);
  for (int s = 0; s < S_round; ++s) {
    subs[s].resize(C);
    for (int c = 0; c < C; ++c) {
      subs[s][c] = {rmat(Bc, U), rvec(Bc)};
      dblocks[s].push_back(subs[s][c].h.hermitian());
    }
    syms[s] = rvec(U);
  }
  decentralized_cd_detect_batch(subs, cfg, eng);  // warm (grows the engine's buffers once)
  auto t0 = Clock::now();
  const int reps = quick ? 1 : 3;
  for (int r = 0; r < reps; ++r) decentralized_cd_detect_batch(subs, cfg, eng);
  const double ul_batch_us = us_since(t0) / reps;
  decentralized_cd_precode_batch(dblocks, syms, pcfg, eng);
  t0 = Clock::now();
  for (int r = 0; r < reps; ++r) decentralized_cd_precode_batch(dblocks, syms, pcfg, eng);
  const double dl_batch_us = us_since(t0) / reps;

  const double ref_us = reference_us_per_call(std::min(S_round, quick ? 200 : 2000), subs, C, Bc, U);
  std::printf(
      "{\"shape\": \"B=256 U=16 C=8 (B_c=32), K=3, 16-QAM\", "
      "\"per_call_us\": {\"decentralized_cd_detect_uniform\": %.2f, \"decentralized_cd_detect_optimal\": %.2f, "
      "\"decentralized_cd_precode\": %.2f, \"calls\": %d, \"stat\": \"median, warm thread-local Engine\"}, "
      "\"batched_round\": {\"subcarriers\": %d, \"detect_ms\": %.3f, \"detect_us_per_subcarrier\": %.3f, "
      "\"detect_Gbps\": %.4f, \"precode_ms\": %.3f, \"precode_us_per_subcarrier\": %.3f, \"precode_Gbps\": %.4f, "
      "\"note\": \"host fp64 in/out: packing, kernels on the pinned staging (zero-copy), unpacking\"}, "
      "\"reference_us_per_call_1thread\": %.2f}\n",
      ul_us, ul_opt_us, dl_us, calls, S_round, ul_batch_us / 1e3, ul_batch_us / S_round,
      S_round * U * BITS / (ul_batch_us * 1e-6) / 1e9, dl_batch_us / 1e3, dl_batch_us / S_round,
      S_round * U * BITS / (dl_batch_us * 1e-6) / 1e9, ref_us);
  return 0;
}
