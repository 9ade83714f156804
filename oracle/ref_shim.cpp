// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (dcdsim, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libdcdref.so).
// It exists so Python tests, the golden-vector generator and bench.py's
// reference arm can call the reference's own C++ API through ctypes:
//   dcd::cd_detect                 src/detect.cpp:67-110
//   dcd::decentralized_cd_detect   src/detect.cpp:147-189
//   dcd::post_eq_variance          src/detect.cpp:112-130
//   dcd::fusion_weights            src/detect.cpp:132-145
//   dcd::mmse_bias_factors         src/detect.cpp:227-242
//   dcd::cd_precode                src/precode.cpp:52-99
//   dcd::power_scale               src/precode.cpp:101-111
//   dcd::decentralized_cd_precode  src/precode.cpp:136-169
//   dcd::make_batch                src/cluster.cpp:80-105
//   uplink observation             src/cluster.cpp:142-145
// Complex arrays are interleaved (re, im) doubles; matrices are column-major
// exactly like dcd::ComplexMatrix (include/dcd/numerics.hpp:35-40).
// Every entry point returns 0 on success, 1 for std::invalid_argument,
// 2 for std::runtime_error, 3 for anything else; dcdref_last_error() holds the
// exception text (thread-local).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dcd/cluster.hpp"
#include "dcd/detect.hpp"
#include "dcd/kernels.hpp"
#include "dcd/mimo.hpp"
#include "dcd/precision.hpp"
#include "dcd/precode.hpp"
#include "dcd/rng.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

using dcd::cf64;
using dcd::ComplexMatrix;
using dcd::ComplexVector;

ComplexMatrix mat_in(const double* p, int rows, int cols) {
  ComplexMatrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  if (rows * cols) std::memcpy(m.flat().data(), p, sizeof(cf64) * rows * cols);
  return m;
}

ComplexVector vec_in(const double* p, int n) {
  ComplexVector v(static_cast<std::size_t>(n));
  if (n) std::memcpy(v.data(), p, sizeof(cf64) * n);
  return v;
}

void vec_out(const ComplexVector& v, double* p) {
  if (p && !v.empty()) std::memcpy(p, v.data(), sizeof(cf64) * v.size());
}

dcd::PrecisionMode prec_of(int fmt, int scope) {
  dcd::PrecisionMode m;
  m.format = static_cast<dcd::PrecisionFormat>(fmt);
  m.scope = static_cast<dcd::PrecisionScope>(scope);
  return m;
}

// Batches pre-split into the reference's own per-cluster containers so that a
// timed run measures only decentralized_cd_detect / decentralized_cd_precode.
struct UlBatch {
  std::size_t s = 0, c = 0, u = 0;
  std::vector<std::vector<dcd::ClusterData>> sub;  // [s][c]
};

struct DlBatch {
  std::size_t s = 0, c = 0, u = 0;
  std::vector<std::vector<ComplexMatrix>> hdl;  // [s][c] U x B_c
  std::vector<ComplexVector> sym;               // [s] U
};

}  // namespace

extern "C" {

const char* dcdref_last_error(void) { return g_err.c_str(); }

int dcdref_set_backend(int b) {
  return guarded([&] { dcd::kernels::set_backend(b ? dcd::kernels::Backend::avx2 : dcd::kernels::Backend::scalar); });
}

int dcdref_active_backend(void) {
  return dcd::kernels::active_backend() == dcd::kernels::Backend::avx2 ? 1 : 0;
}

int dcdref_backend_available(int b) {
  return dcd::kernels::backend_available(b ? dcd::kernels::Backend::avx2 : dcd::kernels::Backend::scalar) ? 1 : 0;
}

// ---- precision -------------------------------------------------------------
int dcdref_round_precision(double* p, int n, int fmt) {
  return guarded([&] {
    dcd::round_precision(std::span<double>(p, static_cast<std::size_t>(n)),
                         static_cast<dcd::PrecisionFormat>(fmt));
  });
}

uint16_t dcdref_f64_to_f16_bits(double x) { return dcd::kernels::detail::f64_to_f16_bits(x); }
double dcdref_f16_bits_to_f64(uint16_t h) { return dcd::kernels::detail::f16_bits_to_f64(h); }

// ---- vector kernels --------------------------------------------------------
void dcdref_cdotc(const double* a, const double* b, int n, double* out) {
  const cf64 r = dcd::kernels::cdotc(reinterpret_cast<const cf64*>(a), reinterpret_cast<const cf64*>(b), n);
  out[0] = r.real();
  out[1] = r.imag();
}
void dcdref_caxpy(double ar, double ai, const double* x, double* y, int n) {
  dcd::kernels::caxpy(cf64{ar, ai}, reinterpret_cast<const cf64*>(x), reinterpret_cast<cf64*>(y), n);
}
double dcdref_norm2sq(const double* a, int n) {
  return dcd::kernels::norm2sq(reinterpret_cast<const cf64*>(a), n);
}

// ---- uplink ----------------------------------------------------------------
int dcdref_cd_detect(const double* h, int b, int u, const double* y, double n0, double ex,
                     unsigned t_max, int fmt, int scope, double* x_out) {
  return guarded([&] {
    vec_out(dcd::cd_detect(mat_in(h, b, u), vec_in(y, b), n0, ex, t_max, prec_of(fmt, scope)), x_out);
  });
}

int dcdref_lmmse_exact(const double* h, int b, int u, const double* y, double n0, double ex,
                       double* x_out) {
  return guarded([&] { vec_out(dcd::lmmse_exact(mat_in(h, b, u), vec_in(y, b), n0, ex), x_out); });
}

int dcdref_post_eq_variance(const double* h, int b, int u, double n0, double ex, double* out) {
  return guarded([&] { *out = dcd::post_eq_variance(mat_in(h, b, u), n0, ex); });
}

int dcdref_fusion_weights(const double* s2, int c, double* w) {
  return guarded([&] {
    const auto r = dcd::fusion_weights(std::span<const double>(s2, static_cast<std::size_t>(c)));
    std::memcpy(w, r.data(), sizeof(double) * r.size());
  });
}

int dcdref_mmse_bias_factors(const double* h, int b, int u, double n0, double ex, double* beta) {
  return guarded([&] {
    const auto r = dcd::mmse_bias_factors(mat_in(h, b, u), n0, ex);
    std::memcpy(beta, r.data(), sizeof(double) * r.size());
  });
}

// Clusters are passed back to back: tile c is bc[c] x u column-major, y block c
// has bc[c] entries.
int dcdref_decentralized_cd_detect(int nc, const int* bc, int u, const double* h_tiles,
                                   const double* y, double n0, double ex, unsigned t_max,
                                   int fusion, int fmt, int scope, int concurrent,
                                   double* xhat, double* local, double* sigma2, double* weights) {
  return guarded([&] {
    std::vector<dcd::ClusterData> cl(static_cast<std::size_t>(nc));
    std::size_t ho = 0, yo = 0;
    for (int c = 0; c < nc; ++c) {
      cl[c].h = mat_in(h_tiles + 2 * ho, bc[c], u);
      cl[c].y = vec_in(y + 2 * yo, bc[c]);
      ho += static_cast<std::size_t>(bc[c]) * u;
      yo += static_cast<std::size_t>(bc[c]);
    }
    dcd::DetectorConfig cfg;
    cfg.n0 = n0;
    cfg.ex = ex;
    cfg.t_max = t_max;
    cfg.fusion = fusion ? dcd::FusionMode::uniform : dcd::FusionMode::optimal;
    cfg.precision = prec_of(fmt, scope);
    const auto r = dcd::decentralized_cd_detect(cl, cfg, concurrent != 0);
    vec_out(r.xhat, xhat);
    if (local)
      for (int c = 0; c < nc; ++c) vec_out(r.local[c], local + 2 * static_cast<std::size_t>(c) * u);
    if (sigma2)
      for (std::size_t c = 0; c < r.sigma2.size(); ++c) sigma2[c] = r.sigma2[c];
    if (weights)
      for (std::size_t c = 0; c < r.weights.size(); ++c) weights[c] = r.weights[c];
  });
}

// ---- downlink --------------------------------------------------------------
int dcdref_cd_precode(const double* h_dl, int u, int b, const double* s, unsigned t_max, int fmt,
                      int scope, double* x_out) {
  return guarded([&] {
    vec_out(dcd::cd_precode(mat_in(h_dl, u, b), vec_in(s, u), t_max, prec_of(fmt, scope)), x_out);
  });
}

int dcdref_zf_exact(const double* h_dl, int u, int b, const double* s, double* x_out) {
  return guarded([&] { vec_out(dcd::zf_exact(mat_in(h_dl, u, b), vec_in(s, u)), x_out); });
}

int dcdref_power_scale(double* x, int n, double rho) {
  return guarded([&] {
    ComplexVector v = vec_in(x, n);
    dcd::power_scale(v, rho);
    vec_out(v, x);
  });
}

// Downlink tiles back to back: tile c is u x bc[c] column-major (H_dl,c).
int dcdref_decentralized_cd_precode(int nc, const int* bc, int u, const double* hdl_tiles,
                                    const double* s, double rho, unsigned t_max, int fmt,
                                    int scope, int concurrent, double* x, double* gain) {
  return guarded([&] {
    std::vector<ComplexMatrix> blocks(static_cast<std::size_t>(nc));
    std::size_t ho = 0;
    for (int c = 0; c < nc; ++c) {
      blocks[c] = mat_in(hdl_tiles + 2 * ho, u, bc[c]);
      ho += static_cast<std::size_t>(bc[c]) * u;
    }
    dcd::PrecoderConfig cfg;
    cfg.rho = rho;
    cfg.t_max = t_max;
    cfg.precision = prec_of(fmt, scope);
    const auto r = dcd::decentralized_cd_precode(blocks, vec_in(s, u), cfg, concurrent != 0);
    vec_out(r.x, x);
    if (gain) *gain = r.effective_gain;
  });
}

// MF baselines: tiles back to back as in dcdref_decentralized_cd_* above.
int dcdref_mf_detect(int nc, const int* bc, int u, const double* h_tiles, const double* ys, double* x_out) {
  return guarded([&] {
    std::vector<dcd::ClusterData> cl(static_cast<std::size_t>(nc));
    std::size_t ho = 0, yo = 0;
    for (int c = 0; c < nc; ++c) {
      cl[c].h = mat_in(h_tiles + 2 * ho, bc[c], u);
      cl[c].y = vec_in(ys + 2 * yo, bc[c]);
      ho += static_cast<std::size_t>(bc[c]) * u;
      yo += static_cast<std::size_t>(bc[c]);
    }
    vec_out(dcd::mf_detect(cl, dcd::PrecisionMode{}), x_out);
  });
}

int dcdref_mf_precode(int nc, const int* bc, int u, const double* hdl_tiles, const double* s, double rho,
                      double* x) {
  return guarded([&] {
    std::vector<ComplexMatrix> blocks(static_cast<std::size_t>(nc));
    std::size_t ho = 0;
    for (int c = 0; c < nc; ++c) {
      blocks[c] = mat_in(hdl_tiles + 2 * ho, u, bc[c]);
      ho += static_cast<std::size_t>(bc[c]) * u;
    }
    vec_out(dcd::mf_precode(blocks, vec_in(s, u), rho, dcd::PrecisionMode{}).x, x);
  });
}

// ---- system model / RNG ----------------------------------------------------
uint64_t dcdref_derive_seed(uint64_t master, uint64_t purpose, uint64_t index) {
  return dcd::derive_seed(master, static_cast<dcd::RngPurpose>(purpose), index);
}

// Draws `n` values of kind (0 uniform01, 1 gaussian, 2 bit) from stream seed.
void dcdref_rng_draw(uint64_t seed, int kind, int n, double* out) {
  dcd::RngStream st(seed);
  for (int i = 0; i < n; ++i)
    out[i] = kind == 0 ? st.uniform01() : kind == 1 ? st.gaussian() : static_cast<double>(st.bit());
}

int dcdref_qam_points(unsigned order, double ex, double* pts) {
  return guarded([&] {
    const auto c = dcd::Constellation::qam(order, ex);
    std::memcpy(pts, c.points().data(), sizeof(cf64) * c.order());
  });
}

int dcdref_slice(unsigned order, double ex, const double* y, int n, unsigned* labels) {
  return guarded([&] {
    const auto c = dcd::Constellation::qam(order, ex);
    for (int i = 0; i < n; ++i) labels[i] = c.slice(cf64{y[2 * i], y[2 * i + 1]});
  });
}

// make_batch (src/cluster.cpp:80-105) for a uniform layout of nc clusters of
// bc antennas. H_out: [count] B x U column-major; bits_out: [count][U*bps].
int dcdref_make_batch(int nc, int bc, int u, unsigned qam, int count, uint64_t seed,
                      uint64_t first_trial, double* h_out, uint8_t* bits_out) {
  return guarded([&] {
    const auto cons = dcd::Constellation::qam(qam, 1.0);
    const auto layout = dcd::ClusterLayout::uniform(static_cast<std::size_t>(nc) * bc, nc);
    const auto batch = dcd::make_batch(layout, u, cons, count, seed, first_trial);
    const std::size_t hb = static_cast<std::size_t>(nc) * bc * u;
    const std::size_t nb = static_cast<std::size_t>(u) * cons.bits_per_symbol();
    for (int s = 0; s < count; ++s) {
      std::memcpy(h_out + 2 * hb * s, batch.h[s].flat().data(), sizeof(cf64) * hb);
      std::memcpy(bits_out + nb * s, batch.bits[s].data(), nb);
    }
  });
}

// Uplink observation exactly as run_uplink_round builds it
// (src/cluster.cpp:152-155): y = awgn(H * modulate(bits), n0, (seed, noise, trial)).
int dcdref_uplink_observe(const double* h, int b, int u, const uint8_t* bits, unsigned qam,
                          double n0, uint64_t seed, uint64_t trial, double* y_out,
                          double* x_true_out) {
  return guarded([&] {
    const auto cons = dcd::Constellation::qam(qam, 1.0);
    const std::vector<uint8_t> bv(bits, bits + static_cast<std::size_t>(u) * cons.bits_per_symbol());
    const ComplexVector x = dcd::modulate(bv, cons);
    dcd::RngStream noise(seed, dcd::RngPurpose::noise, trial);
    vec_out(dcd::awgn(dcd::matvec(mat_in(h, b, u), x), n0, noise), y_out);
    vec_out(x, x_true_out);
  });
}

double dcdref_snr_to_n0(double snr_db, int users, double ex) { return dcd::snr_to_n0(snr_db, users, ex); }

// ---- batched CPU baseline --------------------------------------------------
// The reference's own `concurrent` argument of decentralized_cd_detect /
// decentralized_cd_precode (one std::thread per cluster per call,
// detect.cpp:32-52) for the batch runners below; off by default.
static bool g_concurrent = false;
int dcdref_set_concurrent(int on) {
  g_concurrent = on != 0;
  return 0;
}

// h_tiles: [S][C] tiles of B_c x U (column-major); y: [S][C][B_c].
void* dcdref_ul_batch_create(int s, int nc, int bc, int u, const double* h_tiles, const double* y) {
  auto* b = new UlBatch;
  b->s = s;
  b->c = nc;
  b->u = u;
  b->sub.resize(s);
  const std::size_t tile = static_cast<std::size_t>(bc) * u;
  for (int i = 0; i < s; ++i) {
    b->sub[i].resize(nc);
    for (int c = 0; c < nc; ++c) {
      const std::size_t p = static_cast<std::size_t>(i) * nc + c;
      b->sub[i][c].h = mat_in(h_tiles + 2 * tile * p, bc, u);
      b->sub[i][c].y = vec_in(y + 2 * static_cast<std::size_t>(bc) * p, bc);
    }
  }
  return b;
}

void dcdref_ul_batch_destroy(void* p) { delete static_cast<UlBatch*>(p); }

// Runs decentralized_cd_detect over subcarriers [first, first+count) split in
// contiguous slices over `threads` std::threads. Returns wall seconds, or a
// negative value on error. xhat (optional): [count][U].
double dcdref_ul_batch_run(void* p, double n0, double ex, unsigned t_max, int fusion, int fmt,
                           int scope, int threads, int first, int count, double* xhat) {
  auto* b = static_cast<UlBatch*>(p);
  dcd::DetectorConfig cfg;
  cfg.n0 = n0;
  cfg.ex = ex;
  cfg.t_max = t_max;
  cfg.fusion = fusion ? dcd::FusionMode::uniform : dcd::FusionMode::optimal;
  cfg.precision = prec_of(fmt, scope);
  if (threads < 1) threads = 1;
  std::vector<std::exception_ptr> errs(threads);
  const auto t0 = std::chrono::steady_clock::now();
  auto work = [&](int t) {
    const int lo = first + static_cast<int>(static_cast<long long>(count) * t / threads);
    const int hi = first + static_cast<int>(static_cast<long long>(count) * (t + 1) / threads);
    try {
      for (int i = lo; i < hi; ++i) {
        const auto r = dcd::decentralized_cd_detect(b->sub[i], cfg, g_concurrent);
        if (xhat) vec_out(r.xhat, xhat + 2 * static_cast<std::size_t>(i - first) * b->u);
      }
    } catch (...) {
      errs[t] = std::current_exception();
    }
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (auto& e : errs)
    if (e) {
      guarded([&] { std::rethrow_exception(e); });
      return -1.0;
    }
  return dt;
}

// Downlink batch: uplink-layout tiles [S][C] (B_c x U); the reference's own
// reciprocity step (ComplexMatrix::hermitian, src/cluster.cpp:246-248) builds
// the U x B_c downlink blocks once, outside the timed region.
void* dcdref_dl_batch_create(int s, int nc, int bc, int u, const double* h_tiles, const double* sym) {
  auto* b = new DlBatch;
  b->s = s;
  b->c = nc;
  b->u = u;
  b->hdl.resize(s);
  b->sym.resize(s);
  const std::size_t tile = static_cast<std::size_t>(bc) * u;
  for (int i = 0; i < s; ++i) {
    b->hdl[i].resize(nc);
    for (int c = 0; c < nc; ++c) {
      const std::size_t p = static_cast<std::size_t>(i) * nc + c;
      b->hdl[i][c] = mat_in(h_tiles + 2 * tile * p, bc, u).hermitian();
    }
    b->sym[i] = vec_in(sym + 2 * static_cast<std::size_t>(u) * i, u);
  }
  return b;
}

void dcdref_dl_batch_destroy(void* p) { delete static_cast<DlBatch*>(p); }

// x: [count][C*B_c] stacked beamformers; gain: [count].
double dcdref_dl_batch_run(void* p, double rho, unsigned t_max, int fmt, int scope, int threads,
                           int first, int count, double* x, double* gain) {
  auto* b = static_cast<DlBatch*>(p);
  dcd::PrecoderConfig cfg;
  cfg.rho = rho;
  cfg.t_max = t_max;
  cfg.precision = prec_of(fmt, scope);
  if (threads < 1) threads = 1;
  std::vector<std::exception_ptr> errs(threads);
  const auto t0 = std::chrono::steady_clock::now();
  auto work = [&](int t) {
    const int lo = first + static_cast<int>(static_cast<long long>(count) * t / threads);
    const int hi = first + static_cast<int>(static_cast<long long>(count) * (t + 1) / threads);
    try {
      for (int i = lo; i < hi; ++i) {
        const auto r = dcd::decentralized_cd_precode(b->hdl[i], b->sym[i], cfg, g_concurrent);
        if (x) vec_out(r.x, x + 2 * static_cast<std::size_t>(i - first) * r.x.size());
        if (gain) gain[i - first] = r.effective_gain;
      }
    } catch (...) {
      errs[t] = std::current_exception();
    }
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (auto& e : errs)
    if (e) {
      guarded([&] { std::rethrow_exception(e); });
      return -1.0;
    }
  return dt;
}

}  // extern "C"
