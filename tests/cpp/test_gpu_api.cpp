// C++ parity suite for the dcd::gpu host API (include/dcd_gpu.hpp), written
// like the reference's own doctest suites (tests/test_detect.cpp,
// tests/test_precode.cpp in /root/reference/proj) with the GPU's tolerances:
// fp32 results within 1e-5 relative of the fp64 reference algorithms (exact
// solvers from the C oracle, test infrastructure), exception types and texts
// identical.  Built and run by tests/test_cpp_api.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dcd_gpu.hpp"
#include "../../oracle/dcd_oracle.h"

using dcd::gpu::cf64;
using dcd::gpu::ClusterData;
using dcd::gpu::ComplexMatrix;
using dcd::gpu::ComplexVector;
using dcd::gpu::DetectionResult;
using dcd::gpu::DetectorConfig;
using dcd::gpu::FusionMode;
using dcd::gpu::PrecisionFormat;
using dcd::gpu::PrecisionMode;
using dcd::gpu::PrecisionScope;
using dcd::gpu::PrecoderConfig;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                        \
  do {                                                                                     \
    ++g_checks;                                                                            \
    if (!(cond)) {                                                                         \
      ++g_fail;                                                                            \
      std::printf("  CHECK failed in '%s' line %d: %s\n", g_case.c_str(), __LINE__, #cond); \
    }                                                                                      \
  } while (0)

template <class E, class F>
bool throws_with(F&& f, const char* needle = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return !needle || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

std::vector<std::pair<std::string, std::function<void()>>>& registry() {
  static std::vector<std::pair<std::string, std::function<void()>>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define TEST_CASE(name, id) \
  static void id();         \
  static Reg reg_##id(name, id); \
  static void id()

std::mt19937_64& rng() {
  static std::mt19937_64 e(2024);  // test_detect.cpp:26-29
  return e;
}
cf64 randc() {
  static std::normal_distribution<double> g;
  return {g(rng()), g(rng())};
}
ComplexVector random_vector(std::size_t n) {
  ComplexVector v(n);
  for (auto& z : v) z = randc();
  return v;
}
ComplexMatrix random_matrix(std::size_t r, std::size_t c) {
  ComplexMatrix m(r, c);
  for (auto& z : m.flat()) z = randc() * std::sqrt(0.5);
  return m;
}
double rel_dist(const ComplexVector& a, const ComplexVector& b) {
  double d = 0, n = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    d += std::norm(a[i] - b[i]);
    n += std::norm(b[i]);
  }
  return std::sqrt(d) / std::sqrt(n);
}
ComplexVector lmmse_exact(const ComplexMatrix& h, const ComplexVector& y, double n0, double ex) {
  ComplexVector x(h.cols());
  dcdo_lmmse_exact(reinterpret_cast<const double*>(h.flat().data()), (int)h.rows(), (int)h.cols(),
                   reinterpret_cast<const double*>(y.data()), n0, ex, reinterpret_cast<double*>(x.data()));
  return x;
}
ComplexVector zf_exact(const ComplexMatrix& hdl, const ComplexVector& s) {
  ComplexVector x(hdl.cols());
  dcdo_zf_exact(reinterpret_cast<const double*>(hdl.flat().data()), (int)hdl.rows(), (int)hdl.cols(),
                reinterpret_cast<const double*>(s.data()), reinterpret_cast<double*>(x.data()));
  return x;
}
ComplexVector cd_detect_ref(const ComplexMatrix& h, const ComplexVector& y, double n0, double ex, unsigned t) {
  ComplexVector x(h.cols());
  dcdo_cd_detect(reinterpret_cast<const double*>(h.flat().data()), (int)h.rows(), (int)h.cols(),
                 reinterpret_cast<const double*>(y.data()), n0, ex, t, 0, 0, reinterpret_cast<double*>(x.data()));
  return x;
}
ComplexVector matvec(const ComplexMatrix& a, const ComplexVector& v) {
  ComplexVector y(a.rows());
  for (std::size_t j = 0; j < a.cols(); ++j)
    for (std::size_t i = 0; i < a.rows(); ++i) y[i] += a(i, j) * v[j];
  return y;
}
constexpr double kTol = 1e-5;

}  // namespace

// ---------------------------------------------------------------- uplink
TEST_CASE("coordinate descent on an identity channel converges in one sweep", t_identity) {
  const auto y = random_vector(8);
  const auto x1 = dcd::gpu::cd_detect(ComplexMatrix::identity(8), y, 0.5, 1.0, 1);
  for (std::size_t i = 0; i < 8; ++i) CHECK(std::abs(x1[i] - y[i] / 1.5) <= 1e-6 * std::abs(y[i]));
  const auto x5 = dcd::gpu::cd_detect(ComplexMatrix::identity(8), y, 0.5, 1.0, 5);
  CHECK(rel_dist(x5, x1) <= 1e-6);
}

TEST_CASE("coordinate descent matches the reference sweeps and converges to L-MMSE", t_converge) {
  for (int trial = 0; trial < 5; ++trial) {
    const auto h = random_matrix(32, 8);
    const auto y = random_vector(32);
    CHECK(rel_dist(dcd::gpu::cd_detect(h, y, 0.1, 1.0, 3), cd_detect_ref(h, y, 0.1, 1.0, 3)) <= kTol);
    CHECK(rel_dist(dcd::gpu::cd_detect(h, y, 0.1, 1.0, 200), lmmse_exact(h, y, 0.1, 1.0)) <= kTol);
  }
}

TEST_CASE("odd and large shapes use the generic kernels", t_generic) {
  for (auto [b, u] : std::vector<std::pair<int, int>>{{24, 6}, {33, 5}, {128, 16}, {256, 32}}) {
    const auto h = random_matrix(b, u);
    const auto y = random_vector(b);
    CHECK(rel_dist(dcd::gpu::cd_detect(h, y, 0.3, 1.0, 3), cd_detect_ref(h, y, 0.3, 1.0, 3)) <= kTol);
  }
}

TEST_CASE("detector input validation", t_validation) {
  const auto h = random_matrix(16, 4);
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::cd_detect(h, random_vector(15), 0.1, 1.0, 3); },
                                           "detector: observation length must match antenna count"));
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::cd_detect(h, random_vector(16), -0.1, 1.0, 3); },
                                           "detector: need N0 >= 0 and E_x > 0"));
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::cd_detect(h, random_vector(16), 0.1, 0.0, 3); }));
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::cd_detect(h, random_vector(16), 0.1, 1.0, 0); },
                                           "cd_detect: need at least one sweep"));
  struct Probe : dcd::gpu::SweepObserver {
    int calls = 0;
    void after_update(unsigned, std::size_t, std::span<const cf64>, std::span<const cf64>) override { ++calls; }
  } probe;
  // the checks run before any observer call
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::cd_detect(h, random_vector(15), 0.1, 1.0, 3, {}, &probe); },
                                           "detector: observation length must match antenna count"));
  CHECK(probe.calls == 0);
}

// ---- per-update probes through the debug trace kernels (the reference's
// DescentProbe / ZeroingProbe, tests/test_detect.cpp:149-200 and
// tests/test_precode.cpp:170-224, with fp32 tolerances)
namespace {
double objective(const ComplexMatrix& h, const ComplexVector& y, const ComplexVector& x, double kappa) {
  const auto hx = matvec(h, x);
  double j = 0.0;
  for (std::size_t i = 0; i < y.size(); ++i) j += std::norm(y[i] - hx[i]);
  for (const auto& z : x) j += kappa * std::norm(z);
  return j;
}
double vnorm(const ComplexVector& v) {
  double s = 0.0;
  for (const auto& z : v) s += std::norm(z);
  return std::sqrt(s);
}
struct DescentProbe : dcd::gpu::SweepObserver {
  const ComplexMatrix* h = nullptr;
  const ComplexVector* y = nullptr;
  double kappa = 0.0, last_j = 0.0, slack = 0.0, rtol = 0.0;
  int violations = 0, checked = 0;
  unsigned expect_t = 0;
  std::size_t expect_j = 0;
  void after_update(unsigned t, std::size_t j, std::span<const cf64> x, std::span<const cf64> residual) override {
    if (t != expect_t || j != expect_j) ++violations;  // the reference's order
    if (++expect_j == h->cols()) {
      expect_j = 0;
      ++expect_t;
    }
    ComplexVector xv(x.begin(), x.end());
    const double jv = objective(*h, *y, xv, kappa);
    if (jv > last_j + slack) ++violations;
    last_j = jv;
    ++checked;
    // the maintained residual equals y - H x
    const auto hx = matvec(*h, xv);
    double d = 0.0;
    for (std::size_t i = 0; i < residual.size(); ++i) d += std::norm((*y)[i] - hx[i] - residual[i]);
    if (residual.size() != y->size() || std::sqrt(d) > rtol) ++violations;
  }
};
struct ZeroingProbe : dcd::gpu::SweepObserver {
  const ComplexMatrix* hn = nullptr;  // normalised rows
  const ComplexVector* sb = nullptr;  // normalised targets
  const ComplexMatrix* h_raw = nullptr;
  int violations = 0, sweep_checks = 0;
  void after_update(unsigned, std::size_t coord, std::span<const cf64> x, std::span<const cf64> residual) override {
    if (!residual.empty()) ++violations;  // precode.cpp:95 passes no residual
    cf64 r{0.0, 0.0};
    for (std::size_t j = 0; j < x.size(); ++j) r += (*hn)(coord, j) * x[j];
    r -= (*sb)[coord];
    if (std::abs(r) > 1e-5 * (1.0 + std::abs((*sb)[coord]))) ++violations;
    if (coord + 1 == hn->rows()) {  // sweep boundary: x in the channel row space
      ComplexVector xv(x.begin(), x.end());
      const auto px = zf_exact(*h_raw, matvec(*h_raw, xv));
      double d = 0.0;
      for (std::size_t j = 0; j < xv.size(); ++j) d += std::norm(xv[j] - px[j]);
      if (std::sqrt(d) > 1e-5 * (1.0 + vnorm(xv))) ++violations;
      ++sweep_checks;
    }
  }
};
}  // namespace

TEST_CASE("every coordinate update descends and keeps the residual consistent (trace kernel)", t_descent) {
  for (int trial = 0; trial < 10; ++trial) {
    const std::size_t b = 16 + 16 * (trial % 2), u = 4 + (trial % 5);
    const auto h = random_matrix(b, u);
    const auto y = random_vector(b);
    DescentProbe probe;
    probe.h = &h;
    probe.y = &y;
    probe.kappa = 0.2;
    probe.last_j = vnorm(y) * vnorm(y);
    probe.slack = 1e-5 * probe.last_j;
    probe.rtol = 1e-5 * (1.0 + vnorm(y));
    const auto xt = dcd::gpu::cd_detect(h, y, 0.2, 1.0, 3, {}, &probe);
    CHECK(probe.checked == static_cast<int>(3 * u));
    CHECK(probe.violations == 0);
    // the traced run ends where the batched kernels and the reference end
    CHECK(rel_dist(xt, dcd::gpu::cd_detect(h, y, 0.2, 1.0, 3)) <= kTol);
    CHECK(rel_dist(xt, cd_detect_ref(h, y, 0.2, 1.0, 3)) <= kTol);
  }
}

TEST_CASE("each dual update zeroes its constraint and stays in the row space (trace kernel)", t_zeroing) {
  for (int trial = 0; trial < 10; ++trial) {
    const std::size_t u = 3 + trial % 5, b = 8 + 4 * (trial % 4);
    const auto h = random_matrix(u, b);
    const auto s = random_vector(u);
    ComplexMatrix hn = h;
    ComplexVector sb = s;
    for (std::size_t i = 0; i < u; ++i) {
      double nrm = 0.0;
      for (std::size_t j = 0; j < b; ++j) nrm += std::norm(hn(i, j));
      nrm = std::sqrt(nrm);
      for (std::size_t j = 0; j < b; ++j) hn(i, j) /= nrm;
      sb[i] /= nrm;
    }
    ZeroingProbe probe;
    probe.hn = &hn;
    probe.sb = &sb;
    probe.h_raw = &h;
    const auto xt = dcd::gpu::cd_precode(h, s, 3, {}, &probe);
    CHECK(probe.violations == 0);
    CHECK(probe.sweep_checks == 3);
    CHECK(rel_dist(xt, dcd::gpu::cd_precode(h, s, 3)) <= kTol);
  }
}

TEST_CASE("post-equalization variance closed forms", t_pev) {
  const ComplexMatrix z(32, 8);  // zero channel: variance equals E_x
  CHECK(std::abs(dcd::gpu::post_eq_variance(z, 0.5, 1.0) - 1.0) <= 1e-6);
  const auto h = random_matrix(32, 8);
  double ref = 0.0;
  dcdo_post_eq_variance(reinterpret_cast<const double*>(h.flat().data()), 32, 8, 0.4, 1.0, &ref);
  CHECK(std::abs(dcd::gpu::post_eq_variance(h, 0.4, 1.0) - ref) <= kTol * ref);
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::post_eq_variance(h, 0.0, 1.0); },
                                           "post_eq_variance: need N0 > 0 and E_x > 0"));
}

TEST_CASE("fusion weights", t_fw) {
  const double mixed[] = {1.0, 1.0, 2.0};
  const auto w = dcd::gpu::fusion_weights(mixed);
  CHECK(std::abs(w[0] - 0.4) <= 1e-7 && std::abs(w[1] - 0.4) <= 1e-7 && std::abs(w[2] - 0.2) <= 1e-7);
  const double bad[] = {1.0, 0.0};
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::fusion_weights(bad); },
                                           "fusion_weights: variances must be positive and finite"));
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::fusion_weights(std::span<const double>{}); },
                                           "fusion_weights: no clusters"));
}

TEST_CASE("single-cluster decentralized detection is bitwise the centralized one", t_c1) {
  for (int trial = 0; trial < 5; ++trial) {
    const auto h = random_matrix(32, 8);
    const auto y = random_vector(32);
    const auto direct = dcd::gpu::cd_detect(h, y, 0.2, 1.0, 3);
    DetectorConfig cfg;
    cfg.n0 = 0.2;
    cfg.t_max = 3;
    cfg.fusion = FusionMode::uniform;
    const std::vector<ClusterData> one = {{h, y}};
    const auto dec = dcd::gpu::decentralized_cd_detect(one, cfg);
    CHECK(dec.weights.size() == 1 && dec.weights[0] == 1.0);
    CHECK(std::memcmp(dec.xhat.data(), direct.data(), direct.size() * sizeof(cf64)) == 0);
  }
}

TEST_CASE("decentralized detection matches the reference fusion (both modes)", t_dec) {
  for (auto fusion : {FusionMode::uniform, FusionMode::optimal}) {
    const auto h = random_matrix(128, 8);
    const auto y = random_vector(128);
    std::vector<ClusterData> cl(4);
    std::vector<double> tiles, ys;
    for (int c = 0; c < 4; ++c) {
      cl[c].h = ComplexMatrix(32, 8);
      for (int j = 0; j < 8; ++j)
        for (int i = 0; i < 32; ++i) cl[c].h(i, j) = h(32 * c + i, j);
      cl[c].y.assign(y.begin() + 32 * c, y.begin() + 32 * (c + 1));
      for (auto z : cl[c].h.flat()) tiles.insert(tiles.end(), {z.real(), z.imag()});
      for (auto z : cl[c].y) ys.insert(ys.end(), {z.real(), z.imag()});
    }
    DetectorConfig cfg;
    cfg.n0 = 0.3;
    cfg.fusion = fusion;
    const auto got = dcd::gpu::decentralized_cd_detect(cl, cfg);
    const int bc[4] = {32, 32, 32, 32};
    ComplexVector want(8);
    std::vector<double> s2(4), w(4);
    dcdo_decentralized_cd_detect(4, bc, 8, tiles.data(), ys.data(), 0.3, 1.0, 3,
                                 fusion == FusionMode::uniform ? DCDO_FUSION_UNIFORM : DCDO_FUSION_OPTIMAL, 0, 0,
                                 reinterpret_cast<double*>(want.data()), nullptr, s2.data(), w.data());
    CHECK(rel_dist(got.xhat, want) <= kTol);
    for (int c = 0; c < 4; ++c) CHECK(std::abs(got.weights[c] - w[c]) <= 1e-5);
  }
}

TEST_CASE("identical clusters under uniform fusion reproduce the single cluster", t_identical) {
  const auto h = random_matrix(32, 8);
  const auto y = random_vector(32);
  DetectorConfig cfg;
  cfg.n0 = 0.15;
  cfg.t_max = 4;
  cfg.fusion = FusionMode::uniform;
  const std::vector<ClusterData> one = {{h, y}}, three = {{h, y}, {h, y}, {h, y}};
  CHECK(rel_dist(dcd::gpu::decentralized_cd_detect(three, cfg).xhat, dcd::gpu::decentralized_cd_detect(one, cfg).xhat) <=
        1e-6);
}

TEST_CASE("message rounding applies to the transmitted estimates", t_msg16) {
  const auto h = random_matrix(32, 8);
  const auto y = random_vector(32);
  DetectorConfig cfg;
  cfg.n0 = 0.2;
  cfg.precision = {PrecisionFormat::fp16, PrecisionScope::messages_only};
  const std::vector<ClusterData> one = {{h, y}};
  const auto dec = dcd::gpu::decentralized_cd_detect(one, cfg);
  for (const auto& z : dec.local[0]) {  // every payload value is a binary16 value
    double re = z.real(), im = z.imag();
    dcdo_round_precision(&re, 1, DCDO_FP16);
    dcdo_round_precision(&im, 1, DCDO_FP16);
    CHECK(re == z.real() && im == z.imag());
  }
  for (double s : dec.sigma2) {
    double r = s;
    dcdo_round_precision(&r, 1, DCDO_FP16);
    CHECK(r == s);
  }
  CHECK(rel_dist(dec.xhat, cd_detect_ref(h, y, 0.2, 1.0, 3)) <= 2e-3);
}

TEST_CASE("full-storage fp16 detection stays within 2e-2", t_full16) {
  const auto h = random_matrix(32, 16);
  const auto y = random_vector(32);
  const auto x = dcd::gpu::cd_detect(h, y, 0.5, 1.0, 3, {PrecisionFormat::fp16, PrecisionScope::full_storage});
  CHECK(rel_dist(x, cd_detect_ref(h, y, 0.5, 1.0, 3)) <= 2e-2);
  const auto h7 = random_matrix(7, 3);  // odd B_c: padded zero row
  const auto y7 = random_vector(7);
  CHECK(rel_dist(dcd::gpu::cd_detect(h7, y7, 0.5, 1.0, 3, {PrecisionFormat::fp16, PrecisionScope::full_storage}),
                 cd_detect_ref(h7, y7, 0.5, 1.0, 3)) <= 2e-2);
}

TEST_CASE("repeated and concurrent-flag calls are bitwise identical", t_det) {
  const auto h = random_matrix(128, 8);
  const auto y = random_vector(128);
  std::vector<ClusterData> cl(4);
  for (int c = 0; c < 4; ++c) {
    cl[c].h = ComplexMatrix(32, 8);
    for (int j = 0; j < 8; ++j)
      for (int i = 0; i < 32; ++i) cl[c].h(i, j) = h(32 * c + i, j);
    cl[c].y.assign(y.begin() + 32 * c, y.begin() + 32 * (c + 1));
  }
  DetectorConfig cfg;
  cfg.n0 = 0.3;
  const auto a = dcd::gpu::decentralized_cd_detect(cl, cfg, false);
  const auto b = dcd::gpu::decentralized_cd_detect(cl, cfg, true);
  CHECK(std::memcmp(a.xhat.data(), b.xhat.data(), a.xhat.size() * sizeof(cf64)) == 0);
  CHECK(a.sigma2 == b.sigma2 && a.weights == b.weights);
}

// ---------------------------------------------------------------- downlink
TEST_CASE("dual coordinate descent is exact in one sweep for the identity", t_pid) {
  const auto s = random_vector(6);
  const auto x1 = dcd::gpu::cd_precode(ComplexMatrix::identity(6), s, 1);
  for (std::size_t i = 0; i < 6; ++i) CHECK(std::abs(x1[i] - s[i]) <= 1e-6 * std::abs(s[i]));
}

TEST_CASE("dual coordinate descent converges to the exact zero-forcing beamformer", t_zf) {
  for (int trial = 0; trial < 5; ++trial) {
    const auto hdl = random_matrix(32, 8).hermitian();
    const auto s = random_vector(8);
    CHECK(rel_dist(dcd::gpu::cd_precode(hdl, s, 200), zf_exact(hdl, s)) <= 1e-4);
  }
}

TEST_CASE("precoder input validation", t_pval) {
  ComplexMatrix h(2, 8);
  for (std::size_t j = 0; j < 8; ++j) h(0, j) = randc();  // row 1 stays zero
  CHECK(throws_with<std::runtime_error>([&] { dcd::gpu::cd_precode(h, random_vector(2), 3); },
                                        "cd_precode: user 1 has an all-zero channel row"));
  const auto good = random_matrix(8, 2).hermitian();
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::cd_precode(good, random_vector(3), 3); },
                                           "precoder: symbol count must match user count"));
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::cd_precode(good, random_vector(2), 0); },
                                           "cd_precode: need at least one sweep"));
}

TEST_CASE("power_scale sets the norm exactly", t_ps) {
  ComplexVector x = {cf64{3.0, 0.0}, cf64{0.0, 4.0}};
  dcd::gpu::power_scale(x, 2.0);
  CHECK(std::abs(x[0] - cf64{1.2, 0.0}) <= 1e-6 && std::abs(x[1] - cf64{0.0, 1.6}) <= 1e-6);
  ComplexVector zero(4);
  CHECK(throws_with<std::runtime_error>([&] { dcd::gpu::power_scale(zero, 1.0); },
                                        "power_scale: zero beamformer cannot be scaled"));
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::power_scale(x, 0.0); },
                                           "power_scale: amplitude must be positive"));
  ComplexVector empty;
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::power_scale(empty, 1.0); }, "power_scale: empty beamformer"));
}

TEST_CASE("single-cluster decentralized precoding equals the centralized one", t_pc1) {
  const auto hdl = random_matrix(32, 8).hermitian();
  const auto s = random_vector(8);
  PrecoderConfig cfg;
  cfg.rho = 2.5;
  auto direct = dcd::gpu::cd_precode(hdl, s, 3);
  dcd::gpu::power_scale(direct, 2.5);
  const ComplexMatrix blocks[] = {hdl};
  const auto dec = dcd::gpu::decentralized_cd_precode(blocks, s, cfg);
  CHECK(rel_dist(dec.x, direct) <= kTol);
}

TEST_CASE("decentralized precoding splits the power budget evenly", t_split) {
  const auto s = random_vector(8);
  std::vector<ComplexMatrix> blocks;
  for (int k = 0; k < 3; ++k) blocks.push_back(random_matrix(16, 8).hermitian());
  PrecoderConfig cfg;
  cfg.rho = std::sqrt(8.0);
  const auto res = dcd::gpu::decentralized_cd_precode(blocks, s, cfg);
  const double rho_c = cfg.rho / std::sqrt(3.0);
  double total = 0;
  for (const auto& blk : res.blocks) {
    double n = 0;
    for (auto z : blk) n += std::norm(z);
    CHECK(std::abs(std::sqrt(n) - rho_c) <= 1e-5 * rho_c);
    total += n;
  }
  CHECK(std::abs(total - 8.0) <= 1e-5 * 8.0);
  CHECK(res.x.size() == 48);
}

TEST_CASE("decentralized precoding matches the reference (beamformer and gain)", t_pref) {
  const auto s = random_vector(8);
  std::vector<ComplexMatrix> blocks;
  std::vector<double> tiles;
  for (int k = 0; k < 4; ++k) {
    blocks.push_back(random_matrix(32, 8).hermitian());
    for (auto z : blocks.back().flat()) tiles.insert(tiles.end(), {z.real(), z.imag()});
  }
  PrecoderConfig cfg;
  cfg.rho = std::sqrt(8.0);
  const auto got = dcd::gpu::decentralized_cd_precode(blocks, s, cfg);
  const int bc[4] = {32, 32, 32, 32};
  ComplexVector want(128);
  double gain = 0;
  dcdo_decentralized_cd_precode(4, bc, 8, tiles.data(), reinterpret_cast<const double*>(s.data()), cfg.rho, 3, 0, 0,
                                reinterpret_cast<double*>(want.data()), &gain);
  CHECK(rel_dist(got.x, want) <= kTol);
  CHECK(std::abs(got.effective_gain - gain) <= kTol * std::abs(gain));
}

TEST_CASE("converged decentralized precoding aligns the received signal with the symbols", t_align) {
  const auto s = random_vector(4);
  std::vector<ComplexMatrix> blocks;
  for (int k = 0; k < 2; ++k) blocks.push_back(random_matrix(24, 4).hermitian());
  PrecoderConfig cfg;
  cfg.rho = 2.0;
  cfg.t_max = 200;
  const auto res = dcd::gpu::decentralized_cd_precode(blocks, s, cfg);
  CHECK(res.effective_gain > 0.0);
  ComplexVector y(4);
  for (int k = 0; k < 2; ++k) {
    const auto yk = matvec(blocks[k], res.blocks[k]);
    for (int i = 0; i < 4; ++i) y[i] += yk[i];
  }
  ComplexVector scaled = s;
  for (auto& z : scaled) z *= res.effective_gain;
  CHECK(rel_dist(y, scaled) <= 1e-4);
}

TEST_CASE("decentralized precoding names an undersized cluster", t_under) {
  std::vector<ComplexMatrix> blocks = {random_matrix(32, 8).hermitian(), random_matrix(32, 8).hermitian(),
                                       random_matrix(4, 8).hermitian()};
  CHECK(throws_with<std::invalid_argument>(
      [&] { dcd::gpu::decentralized_cd_precode(blocks, random_vector(8), PrecoderConfig{}); },
      "decentralized_cd_precode: cluster 2 has 4 antennas for 8 users; local zero-forcing needs B_c >= U"));
}

TEST_CASE("full-storage fp16 precoding keeps the cluster power", t_p16) {
  const auto s = random_vector(4);
  std::vector<ComplexMatrix> blocks;
  for (int k = 0; k < 2; ++k) blocks.push_back(random_matrix(16, 4).hermitian());
  PrecoderConfig cfg;
  cfg.rho = 2.0;
  cfg.precision = {PrecisionFormat::fp16, PrecisionScope::full_storage};
  const auto res = dcd::gpu::decentralized_cd_precode(blocks, s, cfg);
  for (const auto& blk : res.blocks) {
    double n = 0;
    for (auto z : blk) n += std::norm(z);
    CHECK(std::abs(std::sqrt(n) - std::sqrt(2.0)) <= 2e-2 * std::sqrt(2.0));
  }
}

TEST_CASE("batched device API round trip", t_batch) {
  dcd::gpu::Engine eng(0);
  const int S = 3, C = 2, Bc = 32, U = 8;
  dcd::gpu::DeviceBatch batch(eng, S, C, Bc, U, DCDG_FP32);
  std::vector<float> h(2 * S * C * U * Bc), y(2 * S * C * Bc);
  std::vector<double> hd(h.size()), yd(y.size());
  for (std::size_t i = 0; i < h.size(); ++i) hd[i] = h[i] = static_cast<float>(randc().real());
  for (std::size_t i = 0; i < y.size(); ++i) yd[i] = y[i] = static_cast<float>(randc().real());
  batch.upload_h(h.data(), h.size() * 4);
  batch.upload_y(y.data(), y.size() * 4);
  batch.detect(C, 3, 0.2, 1.0, FusionMode::uniform);
  std::vector<float> xh(2 * S * U);
  batch.download_xhat(xh.data());
  ComplexVector want(S * U);
  dcdo_ul_detect_batch(S, C, Bc, U, hd.data(), yd.data(), 0.2, 1.0, 3, DCDO_FUSION_UNIFORM, 0, 0,
                       reinterpret_cast<double*>(want.data()), nullptr, nullptr);
  ComplexVector got(S * U);
  for (int i = 0; i < S * U; ++i) got[i] = {xh[2 * i], xh[2 * i + 1]};
  CHECK(rel_dist(got, want) <= kTol);
}

TEST_CASE("exchange window (world 1) reproduces the batched detector and precoder bitwise", t_xwin) {
  dcd::gpu::Engine eng(0);
  const int S = 4, C = 2, Bc = 32, U = 8;
  dcd::gpu::DeviceBatch plain(eng, S, C, Bc, U, DCDG_FP32), via(eng, S, C, Bc, U, DCDG_FP32);
  std::vector<float> h(2 * S * C * U * Bc), y(2 * S * C * Bc), sy(2 * S * U);
  for (auto& v : h) v = static_cast<float>(randc().real());
  for (auto& v : y) v = static_cast<float>(randc().real());
  for (auto& v : sy) v = static_cast<float>(randc().real());
  for (auto* b : {&plain, &via}) {
    b->upload_h(h.data(), h.size() * 4);
    b->upload_y(y.data(), y.size() * 4);
    b->upload_s(sy.data(), sy.size() * 4);
  }
  plain.detect(C, 3, 0.2, 1.0, FusionMode::uniform);
  plain.precode(C, 3, 2.0, true);
  dcd::gpu::ExchangeWindow w(eng, 1, 0, S, C, U, DCDG_FP32);
  w.open(0, w.handle());
  w.detect(via, 0, C, 3, 0.2, 1.0, FusionMode::uniform);
  w.precode(via, 0, 0, C, 3, 2.0);
  std::vector<float> a(2 * S * U), b(2 * S * U), xa(2 * S * C * Bc), xb(2 * S * C * Bc), ga(S), gb(S);
  plain.download_xhat(a.data());
  via.download_xhat(b.data());
  plain.download_x_dl(xa.data());
  via.download_x_dl(xb.data());
  plain.download_gain(ga.data());
  via.download_gain(gb.data());
  CHECK(std::memcmp(a.data(), b.data(), a.size() * 4) == 0);
  CHECK(std::memcmp(xa.data(), xb.data(), xa.size() * 4) == 0);
  CHECK(std::memcmp(ga.data(), gb.data(), ga.size() * 4) == 0);
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::ExchangeWindow bad(eng, 3, 0, S, C, U, DCDG_FP32); },
                                           "S must divide over the ranks"));
}

// ---------------------------------------------------------------- batched round API
namespace {
std::vector<ClusterData> random_clusters(int C, int Bc, int U) {
  std::vector<ClusterData> cl(C);
  for (auto& c : cl) {
    c.h = random_matrix(Bc, U);
    c.y = random_vector(Bc);
  }
  return cl;
}
bool same_bits(const ComplexVector& a, const ComplexVector& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(cf64)) == 0;
}
}  // namespace

TEST_CASE("batched detection is bitwise the per-subcarrier calls (both fusions)", t_ul_batch) {
  const int S = 6, C = 8, Bc = 32, U = 16;
  std::vector<std::vector<ClusterData>> subs;
  for (int s = 0; s < S; ++s) subs.push_back(random_clusters(C, Bc, U));
  for (FusionMode f : {FusionMode::uniform, FusionMode::optimal}) {
    DetectorConfig cfg;
    cfg.n0 = 1.6;
    cfg.fusion = f;
    const auto all = dcd::gpu::decentralized_cd_detect_batch(subs, cfg);
    CHECK(all.size() == static_cast<std::size_t>(S));
    for (int s = 0; s < S; ++s) {
      const auto one = dcd::gpu::decentralized_cd_detect(subs[s], cfg);
      CHECK(same_bits(all[s].xhat, one.xhat));
      for (int c = 0; c < C; ++c) CHECK(same_bits(all[s].local[c], one.local[c]));
      CHECK(all[s].weights == one.weights);
      CHECK(all[s].sigma2 == one.sigma2);
    }
  }
  // the reference's checks per subcarrier, in its order
  subs[3][2].y.pop_back();
  DetectorConfig bad;
  bad.n0 = 1.6;
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::decentralized_cd_detect_batch(subs, bad); },
                                           "detector: observation length must match antenna count"));
  // N0 = 0 with optimal fusion: subcarrier 0's post_eq_variance throws first (detect.cpp:116-117)
  CHECK(throws_with<std::invalid_argument>([&] { dcd::gpu::decentralized_cd_detect_batch(subs, DetectorConfig{}); },
                                           "post_eq_variance: need N0 > 0 and E_x > 0"));
}

TEST_CASE("batched detection with uneven clusters falls back per subcarrier", t_ul_batch_uneven) {
  std::vector<std::vector<ClusterData>> subs;
  for (int s = 0; s < 3; ++s) {
    auto cl = random_clusters(2, 24, 6);
    cl.push_back({random_matrix(20, 6), random_vector(20)});
    subs.push_back(std::move(cl));
  }
  DetectorConfig cfg;
  cfg.n0 = 0.4;
  cfg.fusion = FusionMode::uniform;
  const auto all = dcd::gpu::decentralized_cd_detect_batch(subs, cfg);
  for (int s = 0; s < 3; ++s) CHECK(same_bits(all[s].xhat, dcd::gpu::decentralized_cd_detect(subs[s], cfg).xhat));
}

TEST_CASE("batched precoding is bitwise the per-subcarrier calls", t_dl_batch) {
  const int S = 5, C = 8, Bc = 32, U = 16;
  std::vector<std::vector<ComplexMatrix>> blocks(S);
  std::vector<ComplexVector> syms;
  for (int s = 0; s < S; ++s) {
    for (int c = 0; c < C; ++c) blocks[s].push_back(random_matrix(Bc, U).hermitian());
    syms.push_back(random_vector(U));
  }
  PrecoderConfig cfg;
  cfg.rho = 4.0;
  const auto all = dcd::gpu::decentralized_cd_precode_batch(blocks, syms, cfg);
  for (int s = 0; s < S; ++s) {
    const auto one = dcd::gpu::decentralized_cd_precode(blocks[s], syms[s], cfg);
    CHECK(same_bits(all[s].x, one.x));
    CHECK(all[s].effective_gain == one.effective_gain);
  }
}

TEST_CASE("fp16 messages-only precoding: clusters get the rounded broadcast, the gain the centre's s", t_dl_msg16) {
  const auto s = random_vector(8);
  std::vector<ComplexMatrix> blocks;
  std::vector<double> tiles;
  for (int k = 0; k < 4; ++k) {
    blocks.push_back(random_matrix(32, 8).hermitian());
    for (auto z : blocks.back().flat()) tiles.insert(tiles.end(), {z.real(), z.imag()});
  }
  PrecoderConfig cfg;
  cfg.rho = std::sqrt(8.0);
  cfg.precision = {PrecisionFormat::fp16, PrecisionScope::messages_only};
  const auto got = dcd::gpu::decentralized_cd_precode(blocks, s, cfg);
  const int bc[4] = {32, 32, 32, 32};
  ComplexVector want(128);
  double gain = 0;
  dcdo_decentralized_cd_precode(4, bc, 8, tiles.data(), reinterpret_cast<const double*>(s.data()), cfg.rho, 3, 2, 0,
                                reinterpret_cast<double*>(want.data()), &gain);  // fmt fp16, messages_only
  CHECK(rel_dist(got.x, want) <= kTol);
  CHECK(std::abs(got.effective_gain - gain) <= kTol * std::abs(gain));
}

TEST_CASE("engines on separate host threads run concurrently and agree", t_threads) {
  const auto subs = random_clusters(8, 32, 16);
  DetectorConfig cfg;
  cfg.n0 = 1.6;
  cfg.fusion = FusionMode::uniform;
  const auto want = dcd::gpu::decentralized_cd_detect(subs, cfg);
  std::vector<DetectionResult> got(4);
  std::vector<std::thread> ts;
  for (int t = 0; t < 4; ++t)
    ts.emplace_back([&, t] {
      for (int i = 0; i < 20; ++i) got[t] = dcd::gpu::decentralized_cd_detect(subs, cfg);  // thread_local engine
    });
  for (auto& th : ts) th.join();
  for (const auto& g : got) CHECK(same_bits(g.xhat, want.xhat));
}

int main() {
  for (auto& [name, fn] : registry()) {
    g_case = name;
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  unexpected exception in '%s': %s\n", name.c_str(), e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name.c_str());
  }
  std::printf("%zu test cases, %d checks, %d failed\n", registry().size(), g_checks, g_fail);
  return g_fail ? 1 : 0;
}
