/**
 * @file dcd_gpu.hpp
 * @brief C++ host API of the B200 decentralized CD baseband — the drop-in
 *        surface for the reference's dcd/detect.hpp and dcd/precode.hpp.
 *
 * Same names, argument meaning and exception behaviour as the reference
 * (paths relative to /root/reference/proj):
 *   dcd::gpu::cd_detect                 <- dcd::cd_detect                include/dcd/detect.hpp:60-63
 *   dcd::gpu::post_eq_variance          <- dcd::post_eq_variance         include/dcd/detect.hpp:67
 *   dcd::gpu::fusion_weights            <- dcd::fusion_weights           include/dcd/detect.hpp:70
 *   dcd::gpu::decentralized_cd_detect   <- dcd::decentralized_cd_detect  include/dcd/detect.hpp:84-86
 *   dcd::gpu::cd_precode                <- dcd::cd_precode               include/dcd/precode.hpp:58-60
 *   dcd::gpu::power_scale               <- dcd::power_scale              include/dcd/precode.hpp:63
 *   dcd::gpu::decentralized_cd_precode  <- dcd::decentralized_cd_precode include/dcd/precode.hpp:72-75
 * plus the batched device API (UplinkBatch / DownlinkBatch) the reference's
 * per-subcarrier loops (src/cluster.cpp:138,239) become.
 *
 * Arithmetic: the GPU computes natively in fp32 (PrecisionFormat fp64 and
 * fp32) or in half2 (fp16, both scopes); it does not emulate binary64.
 * Results agree with the reference within 1e-5 (fp32) / 2e-2 (fp16) relative.
 *
 * Errors: std::invalid_argument / std::runtime_error with the reference's
 * messages.  There is no CPU fallback: without a CUDA device every call
 * throws std::runtime_error.  A non-null SweepObserver is rejected with
 * std::invalid_argument (per-update host hooks cannot run on the GPU).
 */
#pragma once

#include <complex>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <functional>
#include <mutex>
#include <string>
#include <span>
#include <vector>

#include "dcdg.h"

namespace dcd::gpu {

using cf64 = std::complex<double>;
using ComplexVector = std::vector<cf64>;

/// Column-major complex matrix with the reference's interface
/// (include/dcd/numerics.hpp:23-53).
class ComplexMatrix {
 public:
  ComplexMatrix() = default;
  ComplexMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols) {}
  static ComplexMatrix identity(std::size_t n);

  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  bool empty() const { return data_.empty(); }
  cf64& operator()(std::size_t i, std::size_t j) { return data_[j * rows_ + i]; }
  const cf64& operator()(std::size_t i, std::size_t j) const { return data_[j * rows_ + i]; }
  std::span<cf64> col(std::size_t j) { return {data_.data() + j * rows_, rows_}; }
  std::span<const cf64> col(std::size_t j) const { return {data_.data() + j * rows_, rows_}; }
  std::span<cf64> flat() { return data_; }
  std::span<const cf64> flat() const { return data_; }
  ComplexMatrix hermitian() const;
  bool same_shape(const ComplexMatrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<cf64> data_;
};

enum class PrecisionFormat : std::uint8_t { fp64, fp32, fp16 };          // precision.hpp:26
enum class PrecisionScope : std::uint8_t { messages_only, full_storage };  // precision.hpp:27

struct PrecisionMode {
  PrecisionFormat format = PrecisionFormat::fp64;
  PrecisionScope scope = PrecisionScope::messages_only;
  bool rounds() const { return format != PrecisionFormat::fp64; }
  bool rounds_storage() const { return rounds() && scope == PrecisionScope::full_storage; }
};

enum class FusionMode : std::uint8_t { optimal, uniform };  // detect.hpp:24

/// Declared for signature compatibility only (detect.hpp:28-36).
class SweepObserver {
 public:
  virtual ~SweepObserver() = default;
  virtual void after_update(unsigned sweep, std::size_t coord, std::span<const cf64> x,
                            std::span<const cf64> residual) = 0;
};

struct DetectorConfig {  // detect.hpp:38-44
  double n0 = 0.0;
  double ex = 1.0;
  unsigned t_max = 3;
  FusionMode fusion = FusionMode::optimal;
  PrecisionMode precision{};
};

struct ClusterData {  // detect.hpp:47-50
  ComplexMatrix h;
  ComplexVector y;
};

struct DetectionResult {  // detect.hpp:72-77
  ComplexVector xhat;
  std::vector<ComplexVector> local;
  std::vector<double> sigma2;
  std::vector<double> weights;
};

struct PrecoderConfig {  // precode.hpp:27-31
  double rho = 1.0;
  unsigned t_max = 3;
  PrecisionMode precision{};
};

struct PrecodeResult {  // precode.hpp:33-37
  ComplexVector x;
  std::vector<ComplexVector> blocks;
  double effective_gain = 0.0;
};

/// One CUDA device context (dcdg_ctx), its own stream, and the buffers every
/// call reuses: grow-only device scratch and pinned host staging (no
/// allocation, free or device-wide synchronisation per call once warm).
/// Calls on one Engine serialise on its mutex; Engines run concurrently.
class Engine {
 public:
  explicit Engine(int device = 0);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  dcdg_ctx* ctx() const { return ctx_; }
  void* stream() const { return stream_; }
  int device() const { return device_; }
  /// Throws the reference exception type for a non-OK dcdg status.
  static void check(int status);
  /// Waits for the stream and rethrows any recorded numerical error.
  void sync();
  /// Device scratch of at least `bytes` (grow-only; valid until the next call
  /// that needs more).  Callers hold mutex().
  void* device_scratch(std::size_t bytes);
  /// Pinned host staging of at least `bytes` (grow-only).  Callers hold mutex().
  void* host_staging(std::size_t bytes);
  std::mutex& mutex() { return *mu_; }
  /// Runs one call's stream work (`enqueue`: its H2D copy, kernels and D2H
  /// copy on stream()), waits for it and rethrows any recorded numerical
  /// error.  Calls with the same `key` (shapes, scalars, buffer addresses)
  /// replay a CUDA graph captured on the key's second use, so a warm call is
  /// one graph launch and one synchronisation.  Callers hold mutex().
  void run(const std::string& key, const std::function<void()>& enqueue);

 private:
  struct Graphs;
  std::unique_ptr<Graphs> graphs_;
  unsigned long long* status_host_ = nullptr;  // pinned status word of run()
  dcdg_ctx* ctx_ = nullptr;
  void* stream_ = nullptr;
  int device_ = 0;
  void* dscratch_ = nullptr;
  std::size_t dscratch_bytes_ = 0;
  void* hstage_ = nullptr;
  std::size_t hstage_bytes_ = 0;
  std::unique_ptr<std::mutex> mu_;
};

/// The calling thread's engine on device 0 (thread_local): the
/// reference-signature functions below use it, so concurrent host threads
/// never serialise on a shared engine.
Engine& default_engine();

// ---- reference-signature API (one subcarrier per call) --------------------
// `concurrent` is accepted for signature compatibility: every cluster of the
// call already runs in one batched launch.  Each function also has an
// overload taking the Engine explicitly (last argument).
ComplexVector cd_detect(const ComplexMatrix& h, const ComplexVector& y, double n0, double ex,
                        unsigned t_max, const PrecisionMode& prec = {},
                        SweepObserver* observer = nullptr);
ComplexVector cd_detect(const ComplexMatrix& h, const ComplexVector& y, double n0, double ex,
                        unsigned t_max, const PrecisionMode& prec, SweepObserver* observer,
                        Engine& eng);
double post_eq_variance(const ComplexMatrix& hc, double n0, double ex);
double post_eq_variance(const ComplexMatrix& hc, double n0, double ex, Engine& eng);
std::vector<double> fusion_weights(std::span<const double> sigma2);
std::vector<double> fusion_weights(std::span<const double> sigma2, Engine& eng);
DetectionResult decentralized_cd_detect(std::span<const ClusterData> clusters,
                                        const DetectorConfig& cfg, bool concurrent = false);
DetectionResult decentralized_cd_detect(std::span<const ClusterData> clusters,
                                        const DetectorConfig& cfg, bool concurrent, Engine& eng);
ComplexVector cd_precode(const ComplexMatrix& h_dl, const ComplexVector& s, unsigned t_max,
                         const PrecisionMode& prec = {}, SweepObserver* observer = nullptr);
ComplexVector cd_precode(const ComplexMatrix& h_dl, const ComplexVector& s, unsigned t_max,
                         const PrecisionMode& prec, SweepObserver* observer, Engine& eng);
void power_scale(ComplexVector& x, double rho);
void power_scale(ComplexVector& x, double rho, Engine& eng);
PrecodeResult decentralized_cd_precode(std::span<const ComplexMatrix> h_dl_blocks,
                                       const ComplexVector& s, const PrecoderConfig& cfg,
                                       bool concurrent = false);
PrecodeResult decentralized_cd_precode(std::span<const ComplexMatrix> h_dl_blocks,
                                       const ComplexVector& s, const PrecoderConfig& cfg,
                                       bool concurrent, Engine& eng);

// ---- batched round API (what the reference's per-subcarrier round loops,
// src/cluster.cpp:138-152 and :239-254, become) ------------------------------
/// decentralized_cd_detect for every subcarrier in ONE device call: the same
/// checks (in the reference's order, per subcarrier) and the same results as
/// calling decentralized_cd_detect per subcarrier.  Subcarriers whose clusters
/// all have the same antenna count (the round's partition_rows case) share one
/// launch; otherwise each subcarrier is its own launch sequence.
std::vector<DetectionResult> decentralized_cd_detect_batch(
    std::span<const std::vector<ClusterData>> subcarriers, const DetectorConfig& cfg,
    Engine& eng = default_engine());
/// decentralized_cd_precode for every subcarrier (blocks[s], symbols[s]) in ONE
/// device call, with the reference's per-subcarrier checks and results.
std::vector<PrecodeResult> decentralized_cd_precode_batch(
    std::span<const std::vector<ComplexMatrix>> h_dl_blocks, std::span<const ComplexVector> s,
    const PrecoderConfig& cfg, Engine& eng = default_engine());

// ---- batched device API (the hot path) --------------------------------------
/// Device-resident batch of S subcarriers x C local clusters in the dcdg.h
/// layout.  Owns its device buffers.
class DeviceBatch {
 public:
  DeviceBatch(Engine& eng, int S, int C, int Bc, int U, int fmt);
  ~DeviceBatch();
  DeviceBatch(const DeviceBatch&) = delete;
  DeviceBatch& operator=(const DeviceBatch&) = delete;

  /// Host -> device upload of channel tiles [S][C][U][Bc] and receive samples
  /// [S][C][Bc] (uplink) or symbols [S][U] (downlink), already in `fmt`.
  void upload_h(const void* host, std::size_t bytes);
  void upload_y(const void* host, std::size_t bytes);
  void upload_s(const void* host, std::size_t bytes);

  /// Uplink: fills x_local [S][C][U] (fmt) and xhat [S][U] (fp32 complex).
  void detect(int C_total, int K, double n0, double ex, FusionMode fusion);
  /// Downlink: fills x [S][C][Bc] (fmt) and gain [S] (fp32).
  void precode(int C_total, int K, double rho, bool with_gain);

  void download_xhat(void* host) const;
  void download_x_local(void* host) const;
  void download_x_dl(void* host) const;
  void download_gain(float* host) const;
  void download_sigma2(float* host) const;

  int S, C, Bc, U, fmt;
  void *H = nullptr, *y = nullptr, *s = nullptr, *x_local = nullptr, *x_dl = nullptr;
  float *xhat = nullptr, *sigma2 = nullptr, *gain = nullptr, *gain_part = nullptr;

 private:
  Engine& eng_;
};

/// This rank's window of the fused cross-GPU exchange (dcdg_xwin_*, one
/// process per GPU): DeviceBatch::detect / precode with the fusion stores and
/// the symbol broadcast done by the kernels in peer memory.
/// Every rank sends handle() to the others over the host's own transport and
/// opens theirs; then all ranks issue the same sequence of calls.
class ExchangeWindow {
 public:
  ExchangeWindow(Engine& eng, int world, int rank, int S, int C_total, int U, int fmt);
  ~ExchangeWindow();
  ExchangeWindow(const ExchangeWindow&) = delete;
  ExchangeWindow& operator=(const ExchangeWindow&) = delete;

  std::vector<std::uint8_t> handle() const;
  void open(int peer, const std::vector<std::uint8_t>& handle);

  /// Uplink of the batch's C clusters [c0, c0 + C): batch.xhat receives the
  /// fused estimates of the subcarriers this rank owns, [S/world][U].
  void detect(DeviceBatch& batch, int c0, int C_total, int K, double n0, double ex, FusionMode fusion);
  /// Downlink: the root's batch.s is pushed to every rank; batch.x_dl gets this
  /// rank's beamformers and batch.gain the effective gain (every rank).
  void precode(DeviceBatch& batch, int root, int c0, int C_total, int K, double rho);

  int world, rank;

 private:
  Engine& eng_;
  dcdg_xwin* w_ = nullptr;
};

}  // namespace dcd::gpu
