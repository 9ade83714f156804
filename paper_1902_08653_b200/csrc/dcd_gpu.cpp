// C++ host API (include/dcd_gpu.hpp) over the dcdg C ABI.  Mirrors the
// reference's detect.hpp / precode.hpp entry points: the same argument checks
// in the same order with the same exception types and texts, then one
// batched device call per decentralized operation.  Host code here only moves
// and re-lays-out data (fp64 <-> fp32/fp16 packing, H_dl <-> uplink tiles);
// all arithmetic of the path runs in the CUDA kernels.
#include <algorithm>
#include "dcd_gpu.hpp"

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

namespace dcd::gpu {

// ---------------------------------------------------------------------------
// ComplexMatrix
// ---------------------------------------------------------------------------
ComplexMatrix ComplexMatrix::identity(std::size_t n) {
  ComplexMatrix m(n, n);
  for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}

ComplexMatrix ComplexMatrix::hermitian() const {
  ComplexMatrix t(cols_, rows_);
  for (std::size_t j = 0; j < cols_; ++j)
    for (std::size_t i = 0; i < rows_; ++i) t(j, i) = std::conj((*this)(i, j));
  return t;
}

namespace {

[[noreturn]] void throw_status(int st, const std::string& msg) {
  if (st == DCDG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// fp64 complex -> device storage bytes (float2 or binary16 pairs, RNE)
std::size_t esize(int fmt) { return fmt == DCDG_FP16 ? 4 : 8; }

void pack(const cf64* v, std::size_t n, int fmt, unsigned char* out) {
  if (fmt == DCDG_FP16) {
    auto* h = reinterpret_cast<__half*>(out);
    for (std::size_t i = 0; i < n; ++i) {
      h[2 * i] = __double2half(v[i].real());
      h[2 * i + 1] = __double2half(v[i].imag());
    }
  } else {
    auto* f = reinterpret_cast<float*>(out);
    for (std::size_t i = 0; i < n; ++i) {
      f[2 * i] = static_cast<float>(v[i].real());
      f[2 * i + 1] = static_cast<float>(v[i].imag());
    }
  }
}

// Rows of a tile / receive vector on the device: fp16 tiles are row-pair
// planar (include/dcdg.h), so an odd antenna count is padded with one zero
// row (a zero row leaves every CD iterate unchanged).
std::size_t dev_rows(std::size_t b, int fmt) { return fmt == DCDG_FP16 ? (b + 1) & ~std::size_t(1) : b; }

// Column-major b x u block (or a b-vector when u == 1) into the device tile
// layout: fp32 interleaved; fp16 row-pair planar {re_2i, re_2i+1, im_2i, im_2i+1}.
void pack_tile(const cf64* v, std::size_t b, std::size_t u, int fmt, unsigned char* out) {
  if (fmt != DCDG_FP16) {
    pack(v, b * u, fmt, out);
    return;
  }
  const std::size_t bp = dev_rows(b, fmt);
  auto* h = reinterpret_cast<__half*>(out);
  for (std::size_t j = 0; j < u; ++j)
    for (std::size_t i = 0; i < bp; i += 2) {
      const cf64 a = v[j * b + i];
      const cf64 c = i + 1 < b ? v[j * b + i + 1] : cf64{0.0, 0.0};
      __half* o = h + 2 * (j * bp + i);
      o[0] = __double2half(a.real());
      o[1] = __double2half(c.real());
      o[2] = __double2half(a.imag());
      o[3] = __double2half(c.imag());
    }
}

void unpack(const unsigned char* in, std::size_t n, int fmt, cf64* out) {
  if (fmt == DCDG_FP16) {
    const auto* h = reinterpret_cast<const __half*>(in);
    for (std::size_t i = 0; i < n; ++i)
      out[i] = cf64{static_cast<double>(__half2float(h[2 * i])), static_cast<double>(__half2float(h[2 * i + 1]))};
  } else {
    const auto* f = reinterpret_cast<const float*>(in);
    for (std::size_t i = 0; i < n; ++i) out[i] = cf64{f[2 * i], f[2 * i + 1]};
  }
}

struct DevMem {
  void* p = nullptr;
  explicit DevMem(std::size_t bytes) {
    if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("dcd::gpu: device allocation failed");
  }
  ~DevMem() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

void h2d(void* dst, const void* src, std::size_t bytes, void* st) {
  if (!bytes) return;
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(st)) != cudaSuccess)
    throw std::runtime_error("dcd::gpu: host-to-device copy failed");
}

void d2h(void* dst, const void* src, std::size_t bytes, void* st) {
  if (!bytes) return;
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(st)) != cudaSuccess)
    throw std::runtime_error("dcd::gpu: device-to-host copy failed");
}

// How a reference PrecisionMode maps onto the device:
//   fp64 / fp32          -> fp32 kernels
//   fp16 messages_only   -> fp32 kernels + binary16 rounding of the wire payloads
//   fp16 full_storage    -> half2 sweep kernels (fp16 storage and arithmetic;
//                           the Engine selects DCDG_ALG_SWEEP)
struct DevPrecision {
  int fmt;
  bool round_messages;
};

DevPrecision map_precision(const PrecisionMode& p) {
  if (p.format == PrecisionFormat::fp16)
    return p.scope == PrecisionScope::full_storage ? DevPrecision{DCDG_FP16, false} : DevPrecision{DCDG_FP32, true};
  return {DCDG_FP32, false};
}

constexpr std::size_t kAlign = 256;
std::size_t align_up(std::size_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }

// detect.cpp:12-19
void check_system(const ComplexMatrix& h, std::size_t ylen, double n0, double ex) {
  if (h.rows() == 0 || h.cols() == 0) throw std::invalid_argument("detector: empty channel matrix");
  if (ylen != h.rows()) throw std::invalid_argument("detector: observation length must match antenna count");
  if (n0 < 0.0 || !(ex > 0.0)) throw std::invalid_argument("detector: need N0 >= 0 and E_x > 0");
}

// precode.cpp:11-16
void check_downlink(const ComplexMatrix& h_dl, const ComplexVector& s) {
  if (h_dl.rows() == 0 || h_dl.cols() == 0) throw std::invalid_argument("precoder: empty channel matrix");
  if (s.size() != h_dl.rows()) throw std::invalid_argument("precoder: symbol count must match user count");
}

void reject_observer(SweepObserver* o) {
  if (o)
    throw std::invalid_argument(
        "dcd::gpu: per-update SweepObserver hooks cannot run on the GPU (use the reference or oracle for probes)");
}

// Reciprocity: uplink tile (B_c x U, column-major) of a U x B_c downlink block.
void uplink_tile_of(const ComplexMatrix& h_dl, cf64* out) {
  const std::size_t u = h_dl.rows(), b = h_dl.cols();
  for (std::size_t j = 0; j < u; ++j)
    for (std::size_t i = 0; i < b; ++i) out[j * b + i] = std::conj(h_dl(j, i));
}

}  // namespace

// ---------------------------------------------------------------------------
// Engine
// ---------------------------------------------------------------------------
void Engine::check(int status) {
  if (status == DCDG_OK) return;
  throw_status(status, dcdg_last_error());
}

Engine::Engine(int device) : device_(device) {
  check(dcdg_init(device, &ctx_));
  // PrecisionMode{fp16, full_storage} mirrors the reference's fp16 arithmetic
  // emulation: the half2 sweep kernel, not the fp32-arithmetic Gram kernel
  check(dcdg_set_fp16_algorithm(ctx_, DCDG_ALG_SWEEP));
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    dcdg_destroy(ctx_);
    throw std::runtime_error("dcd::gpu: stream creation failed");
  }
  stream_ = st;
}

Engine::~Engine() {
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
  dcdg_destroy(ctx_);
}

void Engine::sync() { check(dcdg_sync_status(ctx_, stream_)); }

Engine& default_engine() {
  static Engine eng(0);
  return eng;
}

namespace {
std::mutex g_default_mu;  // the reference-signature calls share default_engine()
}

// ---------------------------------------------------------------------------
// uplink
// ---------------------------------------------------------------------------
ComplexVector cd_detect(const ComplexMatrix& h, const ComplexVector& y, double n0, double ex, unsigned t_max,
                        const PrecisionMode& prec, SweepObserver* observer) {
  check_system(h, y.size(), n0, ex);
  if (t_max == 0) throw std::invalid_argument("cd_detect: need at least one sweep");
  reject_observer(observer);
  std::lock_guard<std::mutex> lk(g_default_mu);
  Engine& eng = default_engine();
  const DevPrecision dp = map_precision(prec);
  const std::size_t b = h.rows(), u = h.cols(), es = esize(dp.fmt), bd = dev_rows(b, dp.fmt);
  std::vector<unsigned char> hb(bd * u * es), yb(bd * es), xb(u * es);
  pack_tile(h.flat().data(), b, u, dp.fmt, hb.data());
  pack_tile(y.data(), b, 1, dp.fmt, yb.data());
  DevMem dh(hb.size()), dy(yb.size()), dx(xb.size());
  h2d(dh.p, hb.data(), hb.size(), eng.stream());
  h2d(dy.p, yb.data(), yb.size(), eng.stream());
  Engine::check(dcdg_ul_detect(eng.ctx(), dh.p, dy.p, 1, 1, 1, static_cast<int>(bd), static_cast<int>(u),
                               static_cast<int>(t_max), n0, ex, dp.fmt, DCDG_FUSION_UNIFORM, dx.p, nullptr, nullptr,
                               nullptr, eng.stream()));
  d2h(xb.data(), dx.p, xb.size(), eng.stream());
  eng.sync();
  ComplexVector x(u);
  unpack(xb.data(), u, dp.fmt, x.data());
  return x;
}

double post_eq_variance(const ComplexMatrix& hc, double n0, double ex) {
  if (hc.rows() == 0 || hc.cols() == 0) throw std::invalid_argument("post_eq_variance: empty channel block");
  if (!(n0 > 0.0) || !(ex > 0.0)) throw std::invalid_argument("post_eq_variance: need N0 > 0 and E_x > 0");
  std::lock_guard<std::mutex> lk(g_default_mu);
  Engine& eng = default_engine();
  const std::size_t b = hc.rows(), u = hc.cols();
  std::vector<unsigned char> hb(b * u * 8);
  pack(hc.flat().data(), b * u, DCDG_FP32, hb.data());
  DevMem dh(hb.size()), ds(sizeof(float));
  h2d(dh.p, hb.data(), hb.size(), eng.stream());
  Engine::check(dcdg_post_eq_variance(eng.ctx(), dh.p, 1, static_cast<int>(b), static_cast<int>(u), n0, ex, DCDG_FP32,
                                      ds.as<float>(), eng.stream()));
  float s2 = 0.f;
  d2h(&s2, ds.p, sizeof s2, eng.stream());
  eng.sync();
  return s2;
}

std::vector<double> fusion_weights(std::span<const double> sigma2) {
  if (sigma2.empty()) throw std::invalid_argument("fusion_weights: no clusters");
  for (double v : sigma2)
    if (!(v > 0.0) || !std::isfinite(v))
      throw std::invalid_argument("fusion_weights: variances must be positive and finite");
  std::lock_guard<std::mutex> lk(g_default_mu);
  Engine& eng = default_engine();
  const int c = static_cast<int>(sigma2.size());
  std::vector<float> s2(sigma2.begin(), sigma2.end()), w(c);
  DevMem ds(c * sizeof(float)), dw(c * sizeof(float));
  h2d(ds.p, s2.data(), c * sizeof(float), eng.stream());
  Engine::check(dcdg_fusion_weights(eng.ctx(), ds.as<float>(), 1, c, dw.as<float>(), eng.stream()));
  d2h(w.data(), dw.p, c * sizeof(float), eng.stream());
  eng.sync();
  return {w.begin(), w.end()};
}

DetectionResult decentralized_cd_detect(std::span<const ClusterData> clusters, const DetectorConfig& cfg,
                                        bool /*concurrent*/) {
  // detect.cpp:150-155
  if (clusters.empty()) throw std::invalid_argument("decentralized_cd_detect: no clusters");
  const std::size_t u = clusters[0].h.cols();
  for (const auto& c : clusters)
    if (c.h.cols() != u) throw std::invalid_argument("decentralized_cd_detect: clusters disagree on user count");
  // per-cluster checks in worker order (cd_detect then post_eq_variance)
  const bool optimal = cfg.fusion == FusionMode::optimal;
  for (const auto& c : clusters) {
    check_system(c.h, c.y.size(), cfg.n0, cfg.ex);
    if (cfg.t_max == 0) throw std::invalid_argument("cd_detect: need at least one sweep");
    if (optimal && !(cfg.n0 > 0.0)) throw std::invalid_argument("post_eq_variance: need N0 > 0 and E_x > 0");
  }
  std::lock_guard<std::mutex> lk(g_default_mu);
  Engine& eng = default_engine();
  const DevPrecision dp = map_precision(cfg.precision);
  const std::size_t nc = clusters.size(), es = esize(dp.fmt);
  bool uniform_bc = true;
  for (const auto& c : clusters) uniform_bc &= c.h.rows() == clusters[0].h.rows();

  // one device buffer each for tiles, observations and per-cluster outputs
  std::vector<std::size_t> hoff(nc), yoff(nc);
  std::size_t hbytes = 0, ybytes = 0;
  for (std::size_t c = 0; c < nc; ++c) {
    hoff[c] = hbytes;
    yoff[c] = ybytes;
    const std::size_t b = dev_rows(clusters[c].h.rows(), dp.fmt);
    hbytes += uniform_bc ? b * u * es : align_up(b * u * es);
    ybytes += uniform_bc ? b * es : align_up(b * es);
  }
  std::vector<unsigned char> hb(hbytes), yb(ybytes);
  for (std::size_t c = 0; c < nc; ++c) {
    pack_tile(clusters[c].h.flat().data(), clusters[c].h.rows(), u, dp.fmt, hb.data() + hoff[c]);
    pack_tile(clusters[c].y.data(), clusters[c].y.size(), 1, dp.fmt, yb.data() + yoff[c]);
  }
  const std::size_t xl_bytes = nc * u * es;
  DevMem dh(hbytes), dy(ybytes), dxl(xl_bytes), ds2(nc * sizeof(float)), dxh(u * 8), dw(nc * sizeof(float));
  h2d(dh.p, hb.data(), hbytes, eng.stream());
  h2d(dy.p, yb.data(), ybytes, eng.stream());
  const int fusion = optimal ? DCDG_FUSION_OPTIMAL : DCDG_FUSION_UNIFORM;
  const int ui = static_cast<int>(u), K = static_cast<int>(cfg.t_max);
  if (uniform_bc) {
    Engine::check(dcdg_ul_detect(eng.ctx(), dh.p, dy.p, 1, static_cast<int>(nc), static_cast<int>(nc),
                                 static_cast<int>(dev_rows(clusters[0].h.rows(), dp.fmt)), ui, K, cfg.n0, cfg.ex, dp.fmt, fusion, dxl.p,
                                 optimal ? ds2.as<float>() : nullptr, nullptr, nullptr, eng.stream()));
  } else {
    for (std::size_t c = 0; c < nc; ++c)
      Engine::check(dcdg_ul_detect(eng.ctx(), static_cast<unsigned char*>(dh.p) + hoff[c],
                                   static_cast<unsigned char*>(dy.p) + yoff[c], 1, 1, 1,
                                   static_cast<int>(dev_rows(clusters[c].h.rows(), dp.fmt)), ui, K, cfg.n0, cfg.ex, dp.fmt, fusion,
                                   static_cast<unsigned char*>(dxl.p) + c * u * es,
                                   optimal ? ds2.as<float>() + c : nullptr, nullptr, nullptr, eng.stream()));
  }
  // message boundary: payloads leave the cluster in the wire precision (detect.cpp:169-173)
  if (dp.round_messages) {
    Engine::check(dcdg_round_fp16(eng.ctx(), dxl.as<float>(), static_cast<int64_t>(2 * nc * u), eng.stream()));
    if (optimal) Engine::check(dcdg_round_fp16(eng.ctx(), ds2.as<float>(), static_cast<int64_t>(nc), eng.stream()));
  }
  Engine::check(dcdg_fuse(eng.ctx(), dxl.p, optimal ? ds2.as<float>() : nullptr, 1, static_cast<int>(nc),
                          static_cast<int>(nc), ui, dp.fmt, fusion, dxh.as<float>(), nullptr, eng.stream()));
  if (optimal)
    Engine::check(dcdg_fusion_weights(eng.ctx(), ds2.as<float>(), 1, static_cast<int>(nc), dw.as<float>(), eng.stream()));
  std::vector<unsigned char> xl(xl_bytes);
  std::vector<float> xh(2 * u), s2(nc), w(nc);
  d2h(xl.data(), dxl.p, xl_bytes, eng.stream());
  d2h(xh.data(), dxh.p, u * 8, eng.stream());
  if (optimal) {
    d2h(s2.data(), ds2.p, nc * sizeof(float), eng.stream());
    d2h(w.data(), dw.p, nc * sizeof(float), eng.stream());
  }
  eng.sync();

  DetectionResult res;
  res.local.resize(nc);
  for (std::size_t c = 0; c < nc; ++c) {
    res.local[c].resize(u);
    unpack(xl.data() + c * u * es, u, dp.fmt, res.local[c].data());
  }
  res.xhat.resize(u);
  for (std::size_t j = 0; j < u; ++j) res.xhat[j] = cf64{xh[2 * j], xh[2 * j + 1]};
  if (optimal) {
    res.sigma2.assign(s2.begin(), s2.end());
    res.weights.assign(w.begin(), w.end());
  } else {
    res.weights.assign(nc, 1.0 / static_cast<double>(nc));  // detect.cpp:181
  }
  return res;
}

// ---------------------------------------------------------------------------
// downlink
// ---------------------------------------------------------------------------
ComplexVector cd_precode(const ComplexMatrix& h_dl, const ComplexVector& s, unsigned t_max,
                         const PrecisionMode& prec, SweepObserver* observer) {
  check_downlink(h_dl, s);
  if (t_max == 0) throw std::invalid_argument("cd_precode: need at least one sweep");
  reject_observer(observer);
  std::lock_guard<std::mutex> lk(g_default_mu);
  Engine& eng = default_engine();
  const DevPrecision dp = map_precision(prec);
  const std::size_t u = h_dl.rows(), b = h_dl.cols(), es = esize(dp.fmt), bd = dev_rows(b, dp.fmt);
  std::vector<cf64> tile(b * u);
  uplink_tile_of(h_dl, tile.data());
  std::vector<unsigned char> hb(bd * u * es), sb(u * es), xb(bd * es);
  pack_tile(tile.data(), b, u, dp.fmt, hb.data());
  pack(s.data(), u, dp.fmt, sb.data());
  DevMem dh(hb.size()), ds(sb.size()), dx(xb.size());
  h2d(dh.p, hb.data(), hb.size(), eng.stream());
  h2d(ds.p, sb.data(), sb.size(), eng.stream());
  // rho == 0: unnormalised beamformer, exactly what cd_precode returns
  Engine::check(dcdg_dl_precode(eng.ctx(), dh.p, ds.p, 1, 1, 1, static_cast<int>(bd), static_cast<int>(u),
                                static_cast<int>(t_max), 0.0, dp.fmt, dx.p, nullptr, nullptr, eng.stream()));
  d2h(xb.data(), dx.p, xb.size(), eng.stream());
  eng.sync();
  ComplexVector x(b);
  unpack(xb.data(), b, dp.fmt, x.data());
  return x;
}

void power_scale(ComplexVector& x, double rho) {
  if (!(rho > 0.0)) throw std::invalid_argument("power_scale: amplitude must be positive");
  if (x.empty()) throw std::invalid_argument("power_scale: empty beamformer");
  std::lock_guard<std::mutex> lk(g_default_mu);
  Engine& eng = default_engine();
  std::vector<unsigned char> xb(x.size() * 8);
  pack(x.data(), x.size(), DCDG_FP32, xb.data());
  DevMem dx(xb.size());
  h2d(dx.p, xb.data(), xb.size(), eng.stream());
  Engine::check(dcdg_power_scale(eng.ctx(), dx.p, 1, static_cast<int>(x.size()), rho, DCDG_FP32, eng.stream()));
  d2h(xb.data(), dx.p, xb.size(), eng.stream());
  eng.sync();
  unpack(xb.data(), x.size(), DCDG_FP32, x.data());
}

PrecodeResult decentralized_cd_precode(std::span<const ComplexMatrix> h_dl_blocks, const ComplexVector& s,
                                       const PrecoderConfig& cfg, bool /*concurrent*/) {
  // precode.cpp:138-152
  if (h_dl_blocks.empty()) throw std::invalid_argument("decentralized_cd_precode: no clusters");
  const std::size_t u = s.size();
  for (std::size_t c = 0; c < h_dl_blocks.size(); ++c) {
    if (h_dl_blocks[c].rows() != u)
      throw std::invalid_argument("decentralized_cd_precode: cluster " + std::to_string(c) +
                                  " disagrees on user count");
    if (h_dl_blocks[c].cols() < u)
      throw std::invalid_argument("decentralized_cd_precode: cluster " + std::to_string(c) + " has " +
                                  std::to_string(h_dl_blocks[c].cols()) + " antennas for " + std::to_string(u) +
                                  " users; local zero-forcing needs B_c >= U");
  }
  if (cfg.t_max == 0) throw std::invalid_argument("cd_precode: need at least one sweep");
  if (!(cfg.rho > 0.0)) throw std::invalid_argument("power_scale: amplitude must be positive");
  std::lock_guard<std::mutex> lk(g_default_mu);
  Engine& eng = default_engine();
  const DevPrecision dp = map_precision(cfg.precision);
  const std::size_t nc = h_dl_blocks.size(), es = esize(dp.fmt);
  bool uniform_bc = true;
  for (const auto& h : h_dl_blocks) uniform_bc &= h.cols() == h_dl_blocks[0].cols();
  std::vector<std::size_t> hoff(nc), xoff(nc);
  std::size_t hbytes = 0, xbytes = 0, btot = 0;
  for (std::size_t c = 0; c < nc; ++c) {
    const std::size_t b = dev_rows(h_dl_blocks[c].cols(), dp.fmt);
    hoff[c] = hbytes;
    xoff[c] = xbytes;
    hbytes += uniform_bc ? b * u * es : align_up(b * u * es);
    xbytes += uniform_bc ? b * es : align_up(b * es);
    btot += h_dl_blocks[c].cols();
  }
  std::vector<unsigned char> hb(hbytes), sb(u * es), xb(xbytes);
  for (std::size_t c = 0; c < nc; ++c) {
    std::vector<cf64> tile(h_dl_blocks[c].cols() * u);
    uplink_tile_of(h_dl_blocks[c], tile.data());
    pack_tile(tile.data(), h_dl_blocks[c].cols(), u, dp.fmt, hb.data() + hoff[c]);
  }
  pack(s.data(), u, dp.fmt, sb.data());
  DevMem dh(hbytes), ds(sb.size()), dx(xbytes), dgp(nc * sizeof(float)), dg(sizeof(float));
  h2d(dh.p, hb.data(), hbytes, eng.stream());
  h2d(ds.p, sb.data(), sb.size(), eng.stream());
  // broadcast boundary: every cluster receives s in the wire precision (precode.cpp:157-160)
  if (dp.round_messages)
    Engine::check(dcdg_round_fp16(eng.ctx(), ds.as<float>(), static_cast<int64_t>(2 * u), eng.stream()));
  const int ui = static_cast<int>(u), K = static_cast<int>(cfg.t_max), nci = static_cast<int>(nc);
  if (uniform_bc) {
    Engine::check(dcdg_dl_precode(eng.ctx(), dh.p, ds.p, 1, nci, nci,
                                  static_cast<int>(dev_rows(h_dl_blocks[0].cols(), dp.fmt)), ui, K,
                                  cfg.rho, dp.fmt, dx.p, dgp.as<float>(), nullptr, eng.stream()));
  } else {
    // each cluster is its own launch; rho/sqrt(C) is applied with C = nc
    const double rho_1 = cfg.rho / std::sqrt(static_cast<double>(nc));
    for (std::size_t c = 0; c < nc; ++c)
      Engine::check(dcdg_dl_precode(eng.ctx(), static_cast<unsigned char*>(dh.p) + hoff[c], ds.p, 1, 1, 1,
                                    static_cast<int>(dev_rows(h_dl_blocks[c].cols(), dp.fmt)), ui, K, rho_1, dp.fmt,
                                    static_cast<unsigned char*>(dx.p) + xoff[c], dgp.as<float>() + c, nullptr,
                                    eng.stream()));
  }
  Engine::check(dcdg_gain_reduce(eng.ctx(), dgp.as<float>(), ds.p, 1, nci, ui, dp.fmt, dg.as<float>(), eng.stream()));
  float gain = 0.f;
  d2h(xb.data(), dx.p, xbytes, eng.stream());
  d2h(&gain, dg.p, sizeof gain, eng.stream());
  eng.sync();

  PrecodeResult res;
  res.blocks.resize(nc);
  res.x.reserve(btot);
  for (std::size_t c = 0; c < nc; ++c) {
    res.blocks[c].resize(h_dl_blocks[c].cols());
    unpack(xb.data() + xoff[c], res.blocks[c].size(), dp.fmt, res.blocks[c].data());
    res.x.insert(res.x.end(), res.blocks[c].begin(), res.blocks[c].end());
  }
  res.effective_gain = gain;
  return res;
}

// ---------------------------------------------------------------------------
// DeviceBatch
// ---------------------------------------------------------------------------
namespace {
void* dalloc(std::size_t bytes) {
  void* p = nullptr;
  if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("dcd::gpu: device allocation failed");
  return p;
}
}  // namespace

DeviceBatch::DeviceBatch(Engine& eng, int S_, int C_, int Bc_, int U_, int fmt_)
    : S(S_), C(C_), Bc(Bc_), U(U_), fmt(fmt_), eng_(eng) {
  const std::size_t P = static_cast<std::size_t>(S) * C, es = esize(fmt);
  H = dalloc(P * Bc * U * es);
  y = dalloc(P * Bc * es);
  s = dalloc(static_cast<std::size_t>(S) * U * es);
  x_local = dalloc(P * U * es);
  x_dl = dalloc(P * Bc * es);
  xhat = static_cast<float*>(dalloc(static_cast<std::size_t>(S) * U * 8));
  sigma2 = static_cast<float*>(dalloc(P * sizeof(float)));
  gain = static_cast<float*>(dalloc(static_cast<std::size_t>(S) * sizeof(float)));
  gain_part = static_cast<float*>(dalloc(P * sizeof(float)));
}

DeviceBatch::~DeviceBatch() {
  for (void* p : {H, y, s, x_local, x_dl, static_cast<void*>(xhat), static_cast<void*>(sigma2),
                  static_cast<void*>(gain), static_cast<void*>(gain_part)})
    if (p) cudaFree(p);
}

void DeviceBatch::upload_h(const void* host, std::size_t bytes) { h2d(H, host, bytes, eng_.stream()); }
void DeviceBatch::upload_y(const void* host, std::size_t bytes) { h2d(y, host, bytes, eng_.stream()); }
void DeviceBatch::upload_s(const void* host, std::size_t bytes) { h2d(s, host, bytes, eng_.stream()); }

void DeviceBatch::detect(int C_total, int K, double n0, double ex, FusionMode fusion) {
  Engine::check(dcdg_ul_detect(eng_.ctx(), H, y, S, C, C_total, Bc, U, K, n0, ex, fmt,
                               fusion == FusionMode::optimal ? DCDG_FUSION_OPTIMAL : DCDG_FUSION_UNIFORM, x_local,
                               sigma2, xhat, nullptr, eng_.stream()));
}

void DeviceBatch::precode(int C_total, int K, double rho, bool with_gain) {
  Engine::check(dcdg_dl_precode(eng_.ctx(), H, s, S, C, C_total, Bc, U, K, rho, fmt, x_dl,
                                with_gain ? gain_part : nullptr, with_gain && C == C_total ? gain : nullptr,
                                eng_.stream()));
}

void DeviceBatch::download_xhat(void* host) const {
  d2h(host, xhat, static_cast<std::size_t>(S) * U * 8, eng_.stream());
  eng_.sync();
}
void DeviceBatch::download_x_local(void* host) const {
  d2h(host, x_local, static_cast<std::size_t>(S) * C * U * esize(fmt), eng_.stream());
  eng_.sync();
}
void DeviceBatch::download_x_dl(void* host) const {
  d2h(host, x_dl, static_cast<std::size_t>(S) * C * Bc * esize(fmt), eng_.stream());
  eng_.sync();
}
void DeviceBatch::download_gain(float* host) const {
  d2h(host, gain, static_cast<std::size_t>(S) * sizeof(float), eng_.stream());
  eng_.sync();
}
void DeviceBatch::download_sigma2(float* host) const {
  d2h(host, sigma2, static_cast<std::size_t>(S) * C * sizeof(float), eng_.stream());
  eng_.sync();
}

// ---------------------------------------------------------------------------
// ExchangeWindow
// ---------------------------------------------------------------------------
ExchangeWindow::ExchangeWindow(Engine& eng, int world_, int rank_, int S, int C_total, int U, int fmt)
    : world(world_), rank(rank_), eng_(eng) {
  if (world_ <= 0 || S % world_) throw std::invalid_argument("dcd::gpu::ExchangeWindow: S must divide over the ranks");
  const std::int64_t es = static_cast<std::int64_t>(esize(fmt)), s_own = S / world_;
  const std::int64_t ul = ((s_own * C_total * U * es + 255) / 256) * 256 + s_own * C_total * 4;
  const std::int64_t dl = ((static_cast<std::int64_t>(S) * U * es + 255) / 256) * 256 + std::int64_t{S} * C_total * 4;
  Engine::check(dcdg_xwin_create(eng.ctx(), world_, rank_, std::max(ul, dl), &w_));
}

ExchangeWindow::~ExchangeWindow() {
  if (w_) dcdg_xwin_destroy(w_);
}

std::vector<std::uint8_t> ExchangeWindow::handle() const {
  std::vector<std::uint8_t> h(DCDG_XWIN_HANDLE_BYTES);
  Engine::check(dcdg_xwin_handle(w_, h.data()));
  return h;
}

void ExchangeWindow::open(int peer, const std::vector<std::uint8_t>& h) {
  if (h.size() != DCDG_XWIN_HANDLE_BYTES)
    throw std::invalid_argument("dcd::gpu::ExchangeWindow: handle has the wrong size");
  Engine::check(dcdg_xwin_open(w_, peer, h.data()));
}

void ExchangeWindow::detect(DeviceBatch& b, int c0, int C_total, int K, double n0, double ex, FusionMode fusion) {
  Engine::check(dcdg_ul_detect_xchg(eng_.ctx(), w_, b.H, b.y, b.S, b.C, c0, C_total, b.Bc, b.U, K, n0, ex, b.fmt,
                                    fusion == FusionMode::optimal ? DCDG_FUSION_OPTIMAL : DCDG_FUSION_UNIFORM, b.xhat,
                                    eng_.stream()));
}

void ExchangeWindow::precode(DeviceBatch& b, int root, int c0, int C_total, int K, double rho) {
  Engine::check(dcdg_dl_precode_xchg(eng_.ctx(), w_, root, b.H, b.s, b.S, b.C, c0, C_total, b.Bc, b.U, K, rho, b.fmt,
                                     b.x_dl, b.gain, eng_.stream()));
}

}  // namespace dcd::gpu
