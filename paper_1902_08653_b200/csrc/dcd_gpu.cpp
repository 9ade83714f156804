// C++ host API (include/dcd_gpu.hpp) over the dcdg C ABI.  Mirrors the
// reference's detect.hpp / precode.hpp entry points: the same argument checks
// in the same order with the same exception types and texts, then one
// batched device call per decentralized operation.  Host code here only moves
// and re-lays-out data (fp64 <-> fp32/fp16 packing, H_dl <-> uplink tiles);
// all arithmetic of the path runs in the CUDA kernels.
#include "dcd_gpu.hpp"

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>

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

// One call's buffers, laid out identically in the engine's pinned staging and
// device scratch: inputs [0, in_end) go over in one H2D copy, outputs
// [in_end, end) come back in one D2H copy.
struct Layout {
  std::size_t end = 0, in_end = 0;
  std::size_t take(std::size_t bytes) {
    const std::size_t off = end;
    end = align_up(end + bytes);
    return off;
  }
  void close_inputs() { in_end = end; }
};

// DCDG_CPP_ZERO_COPY (default): the kernels read the packed inputs and write
// the results straight in the pinned staging (UVA-mapped host memory; the
// bulk copies and loads cross PCIe as they run), so a call is its kernels and
// one synchronisation, no separate H2D/D2H copies (per-call latency 42 -> see
// DESIGN.md §1).  0: device scratch with one H2D and one D2H copy per call.
#ifndef DCDG_CPP_ZERO_COPY
#define DCDG_CPP_ZERO_COPY 1
#endif
struct Call {
  Engine& eng;
  unsigned char* host;
  unsigned char* dev;
  Call(Engine& e, const Layout& l)
      : eng(e),
        host(static_cast<unsigned char*>(e.host_staging(l.end))),
        dev(DCDG_CPP_ZERO_COPY ? host : static_cast<unsigned char*>(e.device_scratch(l.end))) {}
  template <class T = unsigned char>
  T* h(std::size_t off) const { return reinterpret_cast<T*>(host + off); }
  template <class T = unsigned char>
  T* d(std::size_t off) const { return reinterpret_cast<T*>(dev + off); }
  void upload(const Layout& l) const {
    if (dev != host) h2d(dev, host, l.in_end, eng.stream());
  }
  void download(const Layout& l) const {
    if (dev != host) d2h(host + l.in_end, dev + l.in_end, l.end - l.in_end, eng.stream());
  }
};

// Host-side packing / unpacking of a batched call over the subcarriers: on
// several threads for large batches (the fp64 <-> fp32 conversion of a
// 16 800-subcarrier round is ~1.2 GB of host memory traffic).
template <class F>
void for_subcarriers(std::size_t S, F&& fn) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t nt = std::min<std::size_t>(hw, S / 256);
  if (nt <= 1) {
    fn(std::size_t{0}, S);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(nt);
  for (std::size_t t = 0; t < nt; ++t) pool.emplace_back([&, t] { fn(S * t / nt, S * (t + 1) / nt); });
  for (auto& th : pool) th.join();
}

// Graph-cache key of one call (Engine::run): the bytes of every value that
// shapes its stream work (sizes, scalars, buffer addresses).
struct Key {
  std::string s;
  template <class T>
  Key& operator<<(const T& v) {
    s.append(reinterpret_cast<const char*>(&v), sizeof v);
    return *this;
  }
};

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

// fp32 complex device trace entries -> cf64
void trace_vec(const float* f, std::size_t n, ComplexVector& out) {
  out.resize(n);
  for (std::size_t i = 0; i < n; ++i) out[i] = cf64{f[2 * i], f[2 * i + 1]};
}

// Reciprocity: uplink tile (B_c x U, column-major) of a U x B_c downlink block.
void uplink_tile_of(const ComplexMatrix& h_dl, cf64* out) {
  const std::size_t u = h_dl.rows(), b = h_dl.cols();
  for (std::size_t j = 0; j < u; ++j)
    for (std::size_t i = 0; i < b; ++i) out[j * b + i] = std::conj(h_dl(j, i));
}

// ---- the reference's per-call checks, in its order -------------------------
// detect.cpp:150-155 then each worker's cd_detect / post_eq_variance checks
std::size_t check_detect_call(std::span<const ClusterData> clusters, const DetectorConfig& cfg) {
  if (clusters.empty()) throw std::invalid_argument("decentralized_cd_detect: no clusters");
  const std::size_t u = clusters[0].h.cols();
  for (const auto& c : clusters)
    if (c.h.cols() != u) throw std::invalid_argument("decentralized_cd_detect: clusters disagree on user count");
  const bool optimal = cfg.fusion == FusionMode::optimal;
  for (const auto& c : clusters) {
    check_system(c.h, c.y.size(), cfg.n0, cfg.ex);
    if (cfg.t_max == 0) throw std::invalid_argument("cd_detect: need at least one sweep");
    if (optimal && !(cfg.n0 > 0.0)) throw std::invalid_argument("post_eq_variance: need N0 > 0 and E_x > 0");
  }
  return u;
}

// precode.cpp:138-152, then cd_precode / power_scale
void check_precode_call(std::span<const ComplexMatrix> h_dl_blocks, const ComplexVector& s, const PrecoderConfig& cfg) {
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
}

bool uniform_rows(std::span<const ClusterData> cl) {
  for (const auto& c : cl)
    if (c.h.rows() != cl[0].h.rows()) return false;
  return true;
}
bool uniform_cols(std::span<const ComplexMatrix> bl) {
  for (const auto& b : bl)
    if (b.cols() != bl[0].cols()) return false;
  return true;
}

// ---- uplink: S subcarriers with identical cluster shapes in one launch -----
// (uniform B_c, the layout of include/dcdg.h), or one subcarrier with
// per-cluster launches (non-uniform B_c).
using ClusterSpan = std::span<const ClusterData>;
using BlockSpan = std::span<const ComplexMatrix>;

std::vector<DetectionResult> detect_impl(std::span<const ClusterSpan> subs, std::size_t u,
                                         const DetectorConfig& cfg, Engine& eng) {
  const DevPrecision dp = map_precision(cfg.precision);
  const bool optimal = cfg.fusion == FusionMode::optimal;
  const std::size_t S = subs.size(), nc = subs[0].size(), es = esize(dp.fmt);
  const bool uniform = S > 1 || uniform_rows(subs[0]);  // S > 1: shapes checked equal by the caller
  // per-cluster byte offsets inside one subcarrier's tile / vector block
  std::vector<std::size_t> hoff(nc), yoff(nc);
  std::size_t hsub = 0, ysub = 0;
  for (std::size_t c = 0; c < nc; ++c) {
    hoff[c] = hsub;
    yoff[c] = ysub;
    const std::size_t b = dev_rows(subs[0][c].h.rows(), dp.fmt);
    hsub += uniform ? b * u * es : align_up(b * u * es);
    ysub += uniform ? b * es : align_up(b * es);
  }
  Layout L;
  const std::size_t oH = L.take(S * hsub), oY = L.take(S * ysub);
  L.close_inputs();
  const std::size_t oXL = L.take(S * nc * u * es), oS2 = L.take(optimal ? S * nc * sizeof(float) : 0),
                    oXH = L.take(S * u * 8), oW = L.take(optimal ? S * nc * sizeof(float) : 0);
  Call k(eng, L);
  for_subcarriers(S, [&](std::size_t s0, std::size_t s1) {
    for (std::size_t s = s0; s < s1; ++s)
      for (std::size_t c = 0; c < nc; ++c) {
        const auto& cl = subs[s][c];
        pack_tile(cl.h.flat().data(), cl.h.rows(), u, dp.fmt, k.h(oH + s * hsub + hoff[c]));
        pack_tile(cl.y.data(), cl.y.size(), 1, dp.fmt, k.h(oY + s * ysub + yoff[c]));
      }
  });
  const int fusion = optimal ? DCDG_FUSION_OPTIMAL : DCDG_FUSION_UNIFORM;
  const int ui = static_cast<int>(u), K = static_cast<int>(cfg.t_max), nci = static_cast<int>(nc);
  const int Si = static_cast<int>(S);
  float* s2 = optimal ? k.d<float>(oS2) : nullptr;
  Key key;
  key << 'U' << S << nc << u << K << cfg.n0 << cfg.ex << dp.fmt << dp.round_messages << fusion << uniform << k.host
      << k.dev << L.end;
  for (std::size_t c = 0; c < nc; ++c) key << subs[0][c].h.rows();
  eng.run(key.s, [&] {
  k.upload(L);
  if (uniform) {
    Engine::check(dcdg_ul_detect(eng.ctx(), k.d(oH), k.d(oY), Si, nci, nci,
                                 static_cast<int>(dev_rows(subs[0][0].h.rows(), dp.fmt)), ui, K, cfg.n0, cfg.ex,
                                 dp.fmt, fusion, k.d(oXL), s2, nullptr, nullptr, eng.stream()));
  } else {
    for (std::size_t c = 0; c < nc; ++c)
      Engine::check(dcdg_ul_detect(eng.ctx(), k.d(oH + hoff[c]), k.d(oY + yoff[c]), 1, 1, 1,
                                   static_cast<int>(dev_rows(subs[0][c].h.rows(), dp.fmt)), ui, K, cfg.n0, cfg.ex,
                                   dp.fmt, fusion, k.d(oXL + c * u * es), optimal ? s2 + c : nullptr, nullptr,
                                   nullptr, eng.stream()));
  }
  // message boundary: payloads leave the cluster in the wire precision (detect.cpp:169-173)
  if (dp.round_messages) {
    Engine::check(dcdg_round_fp16(eng.ctx(), k.d<float>(oXL), static_cast<int64_t>(2 * S * nc * u), eng.stream()));
    if (optimal) Engine::check(dcdg_round_fp16(eng.ctx(), s2, static_cast<int64_t>(S * nc), eng.stream()));
  }
  Engine::check(dcdg_fuse(eng.ctx(), k.d(oXL), s2, Si, nci, nci, ui, dp.fmt, fusion, k.d<float>(oXH), nullptr,
                          eng.stream()));
  if (optimal) Engine::check(dcdg_fusion_weights(eng.ctx(), s2, Si, nci, k.d<float>(oW), eng.stream()));
  k.download(L);
  });

  std::vector<DetectionResult> out(S);
  for_subcarriers(S, [&](std::size_t s0, std::size_t s1) {
  for (std::size_t s = s0; s < s1; ++s) {
    DetectionResult& res = out[s];
    res.local.resize(nc);
    for (std::size_t c = 0; c < nc; ++c) {
      res.local[c].resize(u);
      unpack(k.h(oXL + (s * nc + c) * u * es), u, dp.fmt, res.local[c].data());
    }
    const float* xh = k.h<float>(oXH) + 2 * s * u;
    res.xhat.resize(u);
    for (std::size_t j = 0; j < u; ++j) res.xhat[j] = cf64{xh[2 * j], xh[2 * j + 1]};
    if (optimal) {
      const float* sv = k.h<float>(oS2) + s * nc;
      const float* wv = k.h<float>(oW) + s * nc;
      res.sigma2.assign(sv, sv + nc);
      res.weights.assign(wv, wv + nc);
    } else {
      res.weights.assign(nc, 1.0 / static_cast<double>(nc));  // detect.cpp:181
    }
  }
  });
  return out;
}

// ---- downlink ---------------------------------------------------------------
std::vector<PrecodeResult> precode_impl(std::span<const BlockSpan> blocks,
                                        std::span<const ComplexVector> syms, const PrecoderConfig& cfg,
                                        Engine& eng) {
  const DevPrecision dp = map_precision(cfg.precision);
  const std::size_t S = blocks.size(), nc = blocks[0].size(), u = syms[0].size(), es = esize(dp.fmt);
  const bool uniform = S > 1 || uniform_cols(blocks[0]);
  std::vector<std::size_t> hoff(nc), xoff(nc);
  std::size_t hsub = 0, xsub = 0, btot = 0;
  for (std::size_t c = 0; c < nc; ++c) {
    const std::size_t b = dev_rows(blocks[0][c].cols(), dp.fmt);
    hoff[c] = hsub;
    xoff[c] = xsub;
    hsub += uniform ? b * u * es : align_up(b * u * es);
    xsub += uniform ? b * es : align_up(b * es);
    btot += blocks[0][c].cols();
  }
  Layout L;
  const std::size_t oH = L.take(S * hsub), oS = L.take(S * u * es);
  // fp16 messages_only: the clusters precode the rounded broadcast, the gain
  // uses the centre's own s (assemble_blocks, precode.cpp:157-168)
  const std::size_t oSw = L.take(dp.round_messages ? S * u * es : 0);
  L.close_inputs();
  const std::size_t oX = L.take(S * xsub), oGP = L.take(S * nc * sizeof(float)), oG = L.take(S * sizeof(float));
  Call k(eng, L);
  for_subcarriers(S, [&](std::size_t s0, std::size_t s1) {
    std::vector<cf64> tile;
    for (std::size_t s = s0; s < s1; ++s) {
      for (std::size_t c = 0; c < nc; ++c) {
        tile.resize(blocks[s][c].cols() * u);
        uplink_tile_of(blocks[s][c], tile.data());
        pack_tile(tile.data(), blocks[s][c].cols(), u, dp.fmt, k.h(oH + s * hsub + hoff[c]));
      }
      pack(syms[s].data(), u, dp.fmt, k.h(oS + s * u * es));
      if (dp.round_messages) pack(syms[s].data(), u, dp.fmt, k.h(oSw + s * u * es));
    }
  });
  Key key;
  key << 'D' << S << nc << u << cfg.t_max << cfg.rho << dp.fmt << dp.round_messages << uniform << k.host << k.dev
      << L.end;
  for (std::size_t c = 0; c < nc; ++c) key << blocks[0][c].cols();
  eng.run(key.s, [&] {
  k.upload(L);
  const void* s_in = k.d(oS);
  if (dp.round_messages) {  // broadcast boundary (precode.cpp:157-160)
    Engine::check(dcdg_round_fp16(eng.ctx(), k.d<float>(oSw), static_cast<int64_t>(2 * S * u), eng.stream()));
    s_in = k.d(oSw);
  }
  const int ui = static_cast<int>(u), K = static_cast<int>(cfg.t_max), nci = static_cast<int>(nc);
  const int Si = static_cast<int>(S);
  float* gp = k.d<float>(oGP);
  if (uniform) {
    Engine::check(dcdg_dl_precode(eng.ctx(), k.d(oH), s_in, Si, nci, nci,
                                  static_cast<int>(dev_rows(blocks[0][0].cols(), dp.fmt)), ui, K, cfg.rho, dp.fmt,
                                  k.d(oX), dp.round_messages ? nullptr : gp, nullptr, eng.stream()));
    if (dp.round_messages)
      Engine::check(dcdg_gain_part(eng.ctx(), k.d(oH), k.d(oX), k.d(oS), Si, nci,
                                   static_cast<int>(dev_rows(blocks[0][0].cols(), dp.fmt)), ui, dp.fmt, gp,
                                   eng.stream()));
  } else {
    // each cluster is its own launch; rho/sqrt(C) is applied with C = nc
    const double rho_1 = cfg.rho / std::sqrt(static_cast<double>(nc));
    for (std::size_t c = 0; c < nc; ++c) {
      const int bc = static_cast<int>(dev_rows(blocks[0][c].cols(), dp.fmt));
      Engine::check(dcdg_dl_precode(eng.ctx(), k.d(oH + hoff[c]), s_in, 1, 1, 1, bc, ui, K, rho_1, dp.fmt,
                                    k.d(oX + xoff[c]), dp.round_messages ? nullptr : gp + c, nullptr, eng.stream()));
      if (dp.round_messages)
        Engine::check(dcdg_gain_part(eng.ctx(), k.d(oH + hoff[c]), k.d(oX + xoff[c]), k.d(oS), 1, 1, bc, ui, dp.fmt,
                                     gp + c, eng.stream()));
    }
  }
  Engine::check(dcdg_gain_reduce(eng.ctx(), gp, k.d(oS), Si, nci, ui, dp.fmt, k.d<float>(oG), eng.stream()));
  k.download(L);
  });

  std::vector<PrecodeResult> out(S);
  for_subcarriers(S, [&](std::size_t s0, std::size_t s1) {
    for (std::size_t s = s0; s < s1; ++s) {
      PrecodeResult& res = out[s];
      res.blocks.resize(nc);
      res.x.reserve(btot);
      for (std::size_t c = 0; c < nc; ++c) {
        res.blocks[c].resize(blocks[s][c].cols());
        unpack(k.h(oX + s * xsub + xoff[c]), res.blocks[c].size(), dp.fmt, res.blocks[c].data());
        res.x.insert(res.x.end(), res.blocks[c].begin(), res.blocks[c].end());
      }
      res.effective_gain = k.h<float>(oG)[s];
    }
  });
  return out;
}

}  // namespace

// ---------------------------------------------------------------------------
// Engine
// ---------------------------------------------------------------------------
void Engine::check(int status) {
  if (status == DCDG_OK) return;
  throw_status(status, dcdg_last_error());
}

// Captured calls of one Engine: key -> instantiated graph (keys seen once run
// eagerly, which also warms the kernels' one-time attribute setup).
struct Engine::Graphs {
  std::unordered_map<std::string, cudaGraphExec_t> exec;
  std::unordered_set<std::string> seen;
  void clear() {
    for (auto& kv : exec) cudaGraphExecDestroy(kv.second);
    exec.clear();
    seen.clear();
  }
  ~Graphs() { clear(); }
};

Engine::Engine(int device)
    : graphs_(std::make_unique<Graphs>()), device_(device), mu_(std::make_unique<std::mutex>()) {
  check(dcdg_init(device, &ctx_));
  if (cudaMallocHost(reinterpret_cast<void**>(&status_host_), sizeof(unsigned long long)) != cudaSuccess) {
    dcdg_destroy(ctx_);
    throw std::runtime_error("dcd::gpu: pinned host allocation failed");
  }
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
  if (stream_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
  graphs_->clear();
  if (status_host_) cudaFreeHost(status_host_);
  if (dscratch_) cudaFree(dscratch_);
  if (hstage_) cudaFreeHost(hstage_);
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
  dcdg_destroy(ctx_);
}

void Engine::sync() { check(dcdg_sync_status(ctx_, stream_)); }

void Engine::run(const std::string& key, const std::function<void()>& enqueue) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  auto finish = [&] {
    if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("dcd::gpu: stream synchronize failed");
    check(dcdg_status_decode(ctx_, *status_host_));
  };
  auto it = graphs_->exec.find(key);
  if (it == graphs_->exec.end()) {
    if (graphs_->seen.insert(key).second) {  // first use: eager
      enqueue();
      check(dcdg_status_enqueue(ctx_, status_host_, stream_));
      finish();
      return;
    }
    if (graphs_->exec.size() >= 64) graphs_->clear();  // bounded: a long-running caller with many shapes
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      throw std::runtime_error("dcd::gpu: stream capture failed");
    try {
      enqueue();
      check(dcdg_status_enqueue(ctx_, status_host_, stream_));
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraphExec_t ex = nullptr;
    const bool ok = cudaStreamEndCapture(st, &g) == cudaSuccess && g &&
                    cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) throw std::runtime_error("dcd::gpu: graph instantiation failed");
    it = graphs_->exec.emplace(key, ex).first;
  }
  if (cudaGraphLaunch(it->second, st) != cudaSuccess) throw std::runtime_error("dcd::gpu: graph launch failed");
  finish();
}

namespace {
std::size_t grow_to(std::size_t have, std::size_t need) {
  std::size_t n = std::max<std::size_t>(have, 1 << 16);
  while (n < need) n += n / 2;
  return n;
}
}  // namespace

void* Engine::device_scratch(std::size_t bytes) {
  if (bytes <= dscratch_bytes_) return dscratch_;
  const std::size_t n = grow_to(dscratch_bytes_, bytes);
  graphs_->clear();  // captured calls hold the old addresses
  cudaSetDevice(device_);
  if (dscratch_) {
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));  // the old buffer may still be in use
    cudaFree(dscratch_);
    dscratch_ = nullptr;
    dscratch_bytes_ = 0;
  }
  if (cudaMalloc(&dscratch_, n) != cudaSuccess) {
    dscratch_ = nullptr;
    throw std::runtime_error("dcd::gpu: device allocation failed");
  }
  dscratch_bytes_ = n;
  return dscratch_;
}

void* Engine::host_staging(std::size_t bytes) {
  if (bytes <= hstage_bytes_) return hstage_;
  const std::size_t n = grow_to(hstage_bytes_, bytes);
  graphs_->clear();  // captured calls hold the old addresses
  if (hstage_) {
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
    cudaFreeHost(hstage_);
    hstage_ = nullptr;
    hstage_bytes_ = 0;
  }
  if (cudaMallocHost(&hstage_, n) != cudaSuccess) {
    hstage_ = nullptr;
    throw std::runtime_error("dcd::gpu: pinned host allocation failed");
  }
  hstage_bytes_ = n;
  return hstage_;
}

Engine& default_engine() {
  thread_local Engine eng(0);
  return eng;
}

// ---------------------------------------------------------------------------
// uplink
// ---------------------------------------------------------------------------
ComplexVector cd_detect(const ComplexMatrix& h, const ComplexVector& y, double n0, double ex, unsigned t_max,
                        const PrecisionMode& prec, SweepObserver* observer) {
  return cd_detect(h, y, n0, ex, t_max, prec, observer, default_engine());
}

ComplexVector cd_detect(const ComplexMatrix& h, const ComplexVector& y, double n0, double ex, unsigned t_max,
                        const PrecisionMode& prec, SweepObserver* observer, Engine& eng) {
  check_system(h, y.size(), n0, ex);
  if (t_max == 0) throw std::invalid_argument("cd_detect: need at least one sweep");
  std::lock_guard<std::mutex> lk(eng.mutex());
  const DevPrecision dp = map_precision(prec);
  const std::size_t b = h.rows(), u = h.cols(), es = esize(dp.fmt), bd = dev_rows(b, dp.fmt);
  if (observer) {
    // per-update hooks (detect.cpp:106): the debug trace kernel dumps x and r
    // after every update; the hooks replay them in order on this thread, and
    // the result is the traced run's final iterate
    const std::size_t n = static_cast<std::size_t>(t_max) * u;
    Layout L;
    const std::size_t oH = L.take(bd * u * es), oY = L.take(bd * es);
    L.close_inputs();
    const std::size_t oXT = L.take(n * u * 8), oRT = L.take(n * bd * 8);
    Call k(eng, L);
    pack_tile(h.flat().data(), b, u, dp.fmt, k.h(oH));
    pack_tile(y.data(), b, 1, dp.fmt, k.h(oY));
    k.upload(L);
    Engine::check(dcdg_ul_trace(eng.ctx(), k.d(oH), k.d(oY), static_cast<int>(bd), static_cast<int>(u),
                                static_cast<int>(t_max), n0, ex, dp.fmt, k.d<float>(oXT), k.d<float>(oRT),
                                eng.stream()));
    k.download(L);
    eng.sync();
    ComplexVector x, r;
    for (std::size_t e = 0; e < n; ++e) {
      trace_vec(k.h<float>(oXT) + 2 * e * u, u, x);
      trace_vec(k.h<float>(oRT) + 2 * e * bd, b, r);
      observer->after_update(static_cast<unsigned>(e / u), e % u, x, r);
    }
    return x;
  }
  Layout L;
  const std::size_t oH = L.take(bd * u * es), oY = L.take(bd * es);
  L.close_inputs();
  const std::size_t oX = L.take(u * es);
  Call k(eng, L);
  pack_tile(h.flat().data(), b, u, dp.fmt, k.h(oH));
  pack_tile(y.data(), b, 1, dp.fmt, k.h(oY));
  Key key;
  key << 'u' << b << u << t_max << n0 << ex << dp.fmt << k.host << k.dev << L.end;
  eng.run(key.s, [&] {
    k.upload(L);
    Engine::check(dcdg_ul_detect(eng.ctx(), k.d(oH), k.d(oY), 1, 1, 1, static_cast<int>(bd), static_cast<int>(u),
                                 static_cast<int>(t_max), n0, ex, dp.fmt, DCDG_FUSION_UNIFORM, k.d(oX), nullptr,
                                 nullptr, nullptr, eng.stream()));
    k.download(L);
  });
  ComplexVector x(u);
  unpack(k.h(oX), u, dp.fmt, x.data());
  return x;
}

double post_eq_variance(const ComplexMatrix& hc, double n0, double ex) {
  return post_eq_variance(hc, n0, ex, default_engine());
}

double post_eq_variance(const ComplexMatrix& hc, double n0, double ex, Engine& eng) {
  if (hc.rows() == 0 || hc.cols() == 0) throw std::invalid_argument("post_eq_variance: empty channel block");
  if (!(n0 > 0.0) || !(ex > 0.0)) throw std::invalid_argument("post_eq_variance: need N0 > 0 and E_x > 0");
  std::lock_guard<std::mutex> lk(eng.mutex());
  const std::size_t b = hc.rows(), u = hc.cols();
  Layout L;
  const std::size_t oH = L.take(b * u * 8);
  L.close_inputs();
  const std::size_t oS = L.take(sizeof(float));
  Call k(eng, L);
  pack(hc.flat().data(), b * u, DCDG_FP32, k.h(oH));
  k.upload(L);
  Engine::check(dcdg_post_eq_variance(eng.ctx(), k.d(oH), 1, static_cast<int>(b), static_cast<int>(u), n0, ex,
                                      DCDG_FP32, k.d<float>(oS), eng.stream()));
  k.download(L);
  eng.sync();
  return *k.h<float>(oS);
}

std::vector<double> fusion_weights(std::span<const double> sigma2) { return fusion_weights(sigma2, default_engine()); }

std::vector<double> fusion_weights(std::span<const double> sigma2, Engine& eng) {
  if (sigma2.empty()) throw std::invalid_argument("fusion_weights: no clusters");
  for (double v : sigma2)
    if (!(v > 0.0) || !std::isfinite(v))
      throw std::invalid_argument("fusion_weights: variances must be positive and finite");
  std::lock_guard<std::mutex> lk(eng.mutex());
  const int c = static_cast<int>(sigma2.size());
  Layout L;
  const std::size_t oS = L.take(c * sizeof(float));
  L.close_inputs();
  const std::size_t oW = L.take(c * sizeof(float));
  Call k(eng, L);
  std::copy(sigma2.begin(), sigma2.end(), k.h<float>(oS));
  k.upload(L);
  Engine::check(dcdg_fusion_weights(eng.ctx(), k.d<float>(oS), 1, c, k.d<float>(oW), eng.stream()));
  k.download(L);
  eng.sync();
  return {k.h<float>(oW), k.h<float>(oW) + c};
}

DetectionResult decentralized_cd_detect(std::span<const ClusterData> clusters, const DetectorConfig& cfg,
                                        bool concurrent) {
  return decentralized_cd_detect(clusters, cfg, concurrent, default_engine());
}

DetectionResult decentralized_cd_detect(std::span<const ClusterData> clusters, const DetectorConfig& cfg,
                                        bool /*concurrent: all clusters run in one launch*/, Engine& eng) {
  const std::size_t u = check_detect_call(clusters, cfg);
  std::lock_guard<std::mutex> lk(eng.mutex());
  const ClusterSpan one[1] = {clusters};
  return std::move(detect_impl(one, u, cfg, eng)[0]);
}

std::vector<DetectionResult> decentralized_cd_detect_batch(std::span<const std::vector<ClusterData>> subcarriers,
                                                           const DetectorConfig& cfg, Engine& eng) {
  if (subcarriers.empty()) return {};
  std::size_t u = 0;
  for (const auto& sc : subcarriers) u = check_detect_call(sc, cfg);
  // one launch when every subcarrier has the first one's cluster shapes and
  // those are uniform; otherwise subcarrier by subcarrier
  const auto& first = subcarriers[0];
  bool same = uniform_rows(first);
  for (const auto& sc : subcarriers) {
    if (!same) break;
    same = sc.size() == first.size() && sc[0].h.cols() == first[0].h.cols();
    for (std::size_t c = 0; same && c < sc.size(); ++c) same = sc[c].h.rows() == first[c].h.rows();
  }
  const std::vector<ClusterSpan> subs(subcarriers.begin(), subcarriers.end());
  std::lock_guard<std::mutex> lk(eng.mutex());
  if (same) return detect_impl(subs, u, cfg, eng);
  std::vector<DetectionResult> out;
  out.reserve(subs.size());
  for (std::size_t s = 0; s < subs.size(); ++s)
    out.push_back(std::move(detect_impl(std::span<const ClusterSpan>(subs).subspan(s, 1), subs[s][0].h.cols(), cfg,
                                        eng)[0]));
  return out;
}

// ---------------------------------------------------------------------------
// downlink
// ---------------------------------------------------------------------------
ComplexVector cd_precode(const ComplexMatrix& h_dl, const ComplexVector& s, unsigned t_max,
                         const PrecisionMode& prec, SweepObserver* observer) {
  return cd_precode(h_dl, s, t_max, prec, observer, default_engine());
}

ComplexVector cd_precode(const ComplexMatrix& h_dl, const ComplexVector& s, unsigned t_max,
                         const PrecisionMode& prec, SweepObserver* observer, Engine& eng) {
  check_downlink(h_dl, s);
  if (t_max == 0) throw std::invalid_argument("cd_precode: need at least one sweep");
  std::lock_guard<std::mutex> lk(eng.mutex());
  const DevPrecision dp = map_precision(prec);
  const std::size_t u = h_dl.rows(), b = h_dl.cols(), es = esize(dp.fmt), bd = dev_rows(b, dp.fmt);
  if (observer) {
    // per-update hooks (precode.cpp:95): x after every update, empty residual
    const std::size_t n = static_cast<std::size_t>(t_max) * u;
    Layout L;
    const std::size_t oH = L.take(bd * u * es), oS = L.take(u * es);
    L.close_inputs();
    const std::size_t oXT = L.take(n * bd * 8);
    Call k(eng, L);
    std::vector<cf64> tile(b * u);
    uplink_tile_of(h_dl, tile.data());
    pack_tile(tile.data(), b, u, dp.fmt, k.h(oH));
    pack(s.data(), u, dp.fmt, k.h(oS));
    k.upload(L);
    Engine::check(dcdg_dl_trace(eng.ctx(), k.d(oH), k.d(oS), static_cast<int>(bd), static_cast<int>(u),
                                static_cast<int>(t_max), dp.fmt, k.d<float>(oXT), eng.stream()));
    k.download(L);
    eng.sync();
    ComplexVector x;
    for (std::size_t e = 0; e < n; ++e) {
      trace_vec(k.h<float>(oXT) + 2 * e * bd, b, x);
      observer->after_update(static_cast<unsigned>(e / u), e % u, x, {});
    }
    return x;
  }
  Layout L;
  const std::size_t oH = L.take(bd * u * es), oS = L.take(u * es);
  L.close_inputs();
  const std::size_t oX = L.take(bd * es);
  Call k(eng, L);
  std::vector<cf64> tile(b * u);
  uplink_tile_of(h_dl, tile.data());
  pack_tile(tile.data(), b, u, dp.fmt, k.h(oH));
  pack(s.data(), u, dp.fmt, k.h(oS));
  Key key;
  key << 'd' << b << u << t_max << dp.fmt << k.host << k.dev << L.end;
  eng.run(key.s, [&] {
    k.upload(L);
    // rho == 0: unnormalised beamformer, exactly what cd_precode returns
    Engine::check(dcdg_dl_precode(eng.ctx(), k.d(oH), k.d(oS), 1, 1, 1, static_cast<int>(bd), static_cast<int>(u),
                                  static_cast<int>(t_max), 0.0, dp.fmt, k.d(oX), nullptr, nullptr, eng.stream()));
    k.download(L);
  });
  ComplexVector x(b);
  unpack(k.h(oX), b, dp.fmt, x.data());
  return x;
}

void power_scale(ComplexVector& x, double rho) { power_scale(x, rho, default_engine()); }

void power_scale(ComplexVector& x, double rho, Engine& eng) {
  if (!(rho > 0.0)) throw std::invalid_argument("power_scale: amplitude must be positive");
  if (x.empty()) throw std::invalid_argument("power_scale: empty beamformer");
  std::lock_guard<std::mutex> lk(eng.mutex());
  Layout L;
  const std::size_t oX = L.take(x.size() * 8);
  L.close_inputs();
  Call k(eng, L);
  pack(x.data(), x.size(), DCDG_FP32, k.h(oX));
  k.upload(L);
  Engine::check(dcdg_power_scale(eng.ctx(), k.d(oX), 1, static_cast<int>(x.size()), rho, DCDG_FP32, eng.stream()));
  d2h(k.h(oX), k.d(oX), x.size() * 8, eng.stream());  // in place: the result comes back over the input
  eng.sync();
  unpack(k.h(oX), x.size(), DCDG_FP32, x.data());
}

PrecodeResult decentralized_cd_precode(std::span<const ComplexMatrix> h_dl_blocks, const ComplexVector& s,
                                       const PrecoderConfig& cfg, bool concurrent) {
  return decentralized_cd_precode(h_dl_blocks, s, cfg, concurrent, default_engine());
}

PrecodeResult decentralized_cd_precode(std::span<const ComplexMatrix> h_dl_blocks, const ComplexVector& s,
                                       const PrecoderConfig& cfg, bool /*concurrent*/, Engine& eng) {
  check_precode_call(h_dl_blocks, s, cfg);
  std::lock_guard<std::mutex> lk(eng.mutex());
  const BlockSpan one[1] = {h_dl_blocks};
  return std::move(precode_impl(one, std::span<const ComplexVector>(&s, 1), cfg, eng)[0]);
}

std::vector<PrecodeResult> decentralized_cd_precode_batch(std::span<const std::vector<ComplexMatrix>> h_dl_blocks,
                                                          std::span<const ComplexVector> s, const PrecoderConfig& cfg,
                                                          Engine& eng) {
  if (h_dl_blocks.size() != s.size())
    throw std::invalid_argument("decentralized_cd_precode_batch: one symbol vector per subcarrier");
  if (h_dl_blocks.empty()) return {};
  for (std::size_t i = 0; i < s.size(); ++i) check_precode_call(h_dl_blocks[i], s[i], cfg);
  const auto& first = h_dl_blocks[0];
  bool same = uniform_cols(first);
  for (std::size_t i = 0; same && i < s.size(); ++i) {
    same = h_dl_blocks[i].size() == first.size() && s[i].size() == s[0].size();
    for (std::size_t c = 0; same && c < first.size(); ++c) same = h_dl_blocks[i][c].cols() == first[c].cols();
  }
  const std::vector<BlockSpan> blocks(h_dl_blocks.begin(), h_dl_blocks.end());
  std::lock_guard<std::mutex> lk(eng.mutex());
  if (same) return precode_impl(blocks, s, cfg, eng);
  std::vector<PrecodeResult> out;
  out.reserve(s.size());
  for (std::size_t i = 0; i < s.size(); ++i)
    out.push_back(std::move(precode_impl(std::span<const BlockSpan>(blocks).subspan(i, 1), s.subspan(i, 1), cfg,
                                         eng)[0]));
  return out;
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
