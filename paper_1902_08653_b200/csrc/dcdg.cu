// C-ABI implementation (include/dcdg.h): argument validation with the
// reference's exception texts, kernel dispatch by problem shape, launch
// geometry (persistent grids sized to SM count x occupancy), and the
// numerical-status word.  No CPU fallback exists: without a CUDA device every
// entry point fails with DCDG_ECUDA.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <utility>

#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "dcdg.h"
#include "dcdg_aux_kernels.cuh"
#include "dcdg_gram_kernels.cuh"
#include "dcdg_mw_kernels.cuh"
#include "dcdg_pev_kernels.cuh"
#include "dcdg_sweep_kernels.cuh"
#include "dcdg_reg_kernels.cuh"
#ifndef DCDG_UL_PP2
#define DCDG_UL_PP2 0
#endif
#if DCDG_UL_PP2
#include "dcdg_pp2_kernels.cuh"
#endif
#include "dcdg_split_kernels.cuh"
#include "dcdg_tmem_kernels.cuh"
// target uplink tile in TMEM (see launch_ul_tm below)
#ifndef DCDG_UL_TMEM
#define DCDG_UL_TMEM 3
#endif
#ifndef DCDG_UL_TMEM_MINB
#define DCDG_UL_TMEM_MINB (DCDG_UL_TMEM == 3 ? 3 : 2)
#endif

struct dcdg_ctx {
  int device = 0;
  int sms = 0;
  unsigned long long* d_status = nullptr;
  uint64_t launches = 0;
  void* scratch = nullptr;  // x_local / sigma2 / gain_part scratch
  size_t scratch_bytes = 0;
  int fp16_alg = DCDG_ALG_GRAM;  // dcdg_set_fp16_algorithm
};

// Exchange window of one rank (dcdg_ul_detect_xchg): [flags][parity 0][parity 1]
// in device memory exported by CUDA IPC; the peers' windows are mapped into
// this process (NVLink P2P between GPUs, plain device memory on one GPU).
struct dcdg_xwin {
  dcdg_ctx* ctx = nullptr;
  int world = 1, rank = 0;
  long long buf_bytes = 0;  // one parity buffer
  unsigned char* base = nullptr;
  unsigned char* peer[dcdg::kXchgMaxRanks] = {};
  bool opened[dcdg::kXchgMaxRanks] = {};
  unsigned int* counter = nullptr;
  // One epoch sequence for BOTH directions: parity = epoch & 1 alternates over
  // the window's calls in issue order, so an uplink and a downlink call never
  // reuse a parity buffer before every peer's wait of the call in between
  // (which implies all consumers of the older call are done) — DESIGN §6.1.
  // The counter lives in device memory and each call's first kernel advances
  // it, so a call captured into a CUDA graph replays with fresh epochs.
  unsigned long long* d_epoch = nullptr;
  long long timeout_ns = 20000000000LL;  // 20 s: a missing peer becomes ST_XCHG_TIMEOUT, not a hang
};

namespace {

// NVTX range per ABI call (the batch stages in Nsight timelines; header-only
// NVTX3, a no-op unless a tool injects itself).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

thread_local std::string g_err;
thread_local long long g_err_problem = -1;

int fail(int code, const std::string& msg) {
  g_err = msg;
  g_err_problem = -1;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(DCDG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr, where)                 \
  do {                                        \
    cudaError_t e_ = (expr);                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int ensure_scratch(dcdg_ctx* ctx, size_t bytes) {
  if (ctx->scratch_bytes >= bytes) return DCDG_OK;
  if (ctx->scratch) cudaFree(ctx->scratch);
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  CUDA_TRY(cudaMalloc(&ctx->scratch, bytes), "scratch allocation");
  ctx->scratch_bytes = bytes;
  return DCDG_OK;
}

inline size_t esize(int fmt) { return fmt == DCDG_FP16 ? 4 : 8; }

#ifndef DCDG_PDL
#define DCDG_PDL 1
#endif
// Launch a stage kernel that consumes its stream predecessor's output (fusion
// after detection, gain after precoding) as a programmatic dependent: it is
// scheduled while the CD kernel's last CTAs drain and waits in
// griddep_wait(), which hides the launch gap between the two.
template <typename... KArgs, typename... Args>
cudaError_t launch_dependent(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = DCDG_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// launchers for the register-resident kernels
// ---------------------------------------------------------------------------
#ifndef DCDG_CTA_WARPS
#define DCDG_CTA_WARPS 1
#endif
// Warps per CTA of the register-resident kernels.  Each warp owns its own
// staging slot and mbarrier, so CTAs need no block-level synchronisation;
// one-warp CTAs let occupancy follow the register budget exactly.
constexpr int kWarps = DCDG_CTA_WARPS;

// Resident CTAs per SM of a kernel on the context's device.  Function
// attributes (the dynamic shared-memory opt-in) and occupancy are per device,
// so both are cached per (device, kernel, smem, threads), never process-wide.
int occupancy_cached(dcdg_ctx* ctx, const void* kern, size_t smem, int threads) {
  using Key = std::tuple<int, const void*, size_t, int>;
  static std::mutex mu;
  static std::map<Key, int> cache;
  const Key key{ctx->device, kern, smem, threads};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  cache.emplace(key, occ);
  return occ;
}
template <typename Kern>
int occupancy_of(dcdg_ctx* ctx, Kern kern, size_t smem, int threads = 32 * kWarps) {
  return occupancy_cached(ctx, reinterpret_cast<const void*>(kern), smem, threads);
}

using UlLaunch = cudaError_t (*)(dcdg_ctx*, const void*, const void*, int, int, float, void*, const dcdg::XMap*,
                                 cudaStream_t);
using DlLaunch = cudaError_t (*)(dcdg_ctx*, const void*, const void*, int, int, int, float, void*, float*,
                                 cudaStream_t);

#ifndef DCDG_LB_UL
#define DCDG_LB_UL 2
#endif
// coordinate block for full-warp groups (G = 32: 5-round reductions, the
// per-block dependency chain dominates; measured +8% at U = 32 on B200)
#ifndef DCDG_LB_UL_WIDE
#define DCDG_LB_UL_WIDE 4
#endif
#ifndef DCDG_LB_UL_MW
#define DCDG_LB_UL_MW DCDG_LB_UL_WIDE
#endif
// xm != nullptr: the fused-exchange instantiation (estimates stored into the
// owners' exchange windows, last CTA signals; dcdg_ul_detect_xchg).
template <int BC, int U, int G, int MINB>
cudaError_t launch_ul_f32(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                          const dcdg::XMap* xm, cudaStream_t st) {
  constexpr int NPW = 32 / G;
  constexpr int LBW = G >= 32 ? DCDG_LB_UL_WIDE : DCDG_LB_UL;
  constexpr int LB = (U % LBW == 0) ? LBW : 2;
  constexpr size_t smem =
      dcdg::CtaSmem<NPW*(BC * U * 8 + BC * 8), dcdg::ul_scal_bytes(U, LB), NPW, kWarps>::kBytes;
  auto kern = dcdg::ul_reg_f32<BC, U, G, kWarps, MINB, LB, false>;
  auto kx = dcdg::ul_reg_f32<BC, U, G, kWarps, MINB, LB, true>;
  const int occ = occupancy_of(ctx, kern, smem);
  const int occx = occupancy_of(ctx, kx, smem);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + kWarps - 1) / kWarps, ctx->sms * (xm ? occx : occ));
  (xm ? kx : kern)<<<blocks, 32 * kWarps, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P,
                                                       K, kappa, static_cast<float2*>(X), xm ? *xm : dcdg::XMap{},
                                                       nullptr, 0.f, 0.f, nullptr);
  return cudaGetLastError();
}

// Lab (off): two problems per 16-lane group (dcdg_pp2_kernels.cuh) for the
// uniform-fusion uplink at the north-star tile, measured slower than
// ul_reg_f32 (profiles/lab/README.md); the exchange instantiation keeps
// ul_reg_f32.
#if DCDG_UL_PP2
template <int BC, int U, int G, int MINB>
cudaError_t launch_ul_pp2(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                          const dcdg::XMap* xm, cudaStream_t st) {
  if (xm) return launch_ul_f32<BC, U, G, MINB>(ctx, H, Y, P, K, kappa, X, xm, st);
  constexpr int NPW = 4;
  constexpr size_t smem = dcdg::CtaSmem<NPW*(BC * U * 8 + BC * 8), dcdg::ul_scal_bytes(U, 2), NPW, kWarps>::kBytes;
  auto kern = dcdg::ul_pp2_f32<BC, U, kWarps, MINB>;
  const int occ = occupancy_of(ctx, kern, smem);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + kWarps - 1) / kWarps, ctx->sms * occ);
  kern<<<blocks, 32 * kWarps, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P, K, kappa,
                                          static_cast<float2*>(X));
  return cudaGetLastError();
}
#endif

// Optimal fusion at the north-star tile (B_c = 32, U = 16, fp32): the CD
// kernel with post_eq_variance fused (ul_reg_f32<..., SIG = true>): one pass
// over H for the estimates and sigma^2.
#ifndef DCDG_UL_SIG_MINB
#define DCDG_UL_SIG_MINB 8
#endif
#ifndef DCDG_UL_SIG
#define DCDG_UL_SIG 1
#endif
bool ul_sig_shape(int bc, int u, int fmt) {
  return DCDG_UL_SIG && fmt == DCDG_FP32 && bc == 32 && (u == 16 || u == 8);
}

template <int BC, int U, int G>
cudaError_t launch_ul_f32_sig_k(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                                float* s2, float gam, float scale, cudaStream_t st) {
  constexpr int NPW = 32 / G, LB = 2;
  constexpr size_t smem = dcdg::CtaSmem<NPW*(BC * U * 8 + BC * 8), dcdg::ul_scal_bytes(U, LB), NPW, kWarps>::kBytes;
  auto kern = dcdg::ul_reg_f32<BC, U, G, kWarps, DCDG_UL_SIG_MINB, LB, false, true>;
  const int occ = occupancy_of(ctx, kern, smem);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + kWarps - 1) / kWarps, ctx->sms * occ);
  kern<<<blocks, 32 * kWarps, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P, K, kappa,
                                          static_cast<float2*>(X), dcdg::XMap{}, s2, gam, scale, ctx->d_status);
  return cudaGetLastError();
}

// B_c = 32 with U = 16 (the north-star tile, 8 lanes per problem) or U = 8
// (the paper's / configs[0] tile, 4 lanes per problem)
// lab (off): the fused-variance batch on the TMEM half-tile kernel, 168
// registers and 12 warps/SM: 0.3771 vs 0.3754 ms (no gain, profiles/lab/README.md)
#ifndef DCDG_UL_TMEM_SIG
#define DCDG_UL_TMEM_SIG 0
#endif
cudaError_t launch_ul_f32_sig(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                              float* s2, float gam, float scale, int U, cudaStream_t st) {
#if DCDG_UL_TMEM == 3 && DCDG_UL_TMEM_SIG
  if (U == 16) {  // the TMEM half-tile kernel with the fused variance (dcdg_tmem_kernels.cuh)
    constexpr int NPW = 4;
    constexpr size_t smem =
        dcdg::CtaSmem<NPW*(32 * 16 * 8 + 32 * 8), dcdg::ul_scal_bytes(16, 2), NPW, dcdg::kTmhWarps>::kBytes;
    auto kern = dcdg::ul_tmh_f32<DCDG_UL_TMEM_MINB, true>;
    (void)occupancy_of(ctx, kern, smem, 32 * dcdg::kTmhWarps);  // sets the shared-memory attribute
    const int nsets = (P + NPW - 1) / NPW;
    const int blocks = std::min((nsets + dcdg::kTmhWarps - 1) / dcdg::kTmhWarps, ctx->sms * DCDG_UL_TMEM_MINB);
    kern<<<blocks, 32 * dcdg::kTmhWarps, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P,
                                                      K, kappa, static_cast<float2*>(X), s2, gam, scale,
                                                      ctx->d_status, dcdg::XMap{});
    return cudaGetLastError();
  }
#endif
  return U == 8 ? launch_ul_f32_sig_k<32, 8, 4>(ctx, H, Y, P, K, kappa, X, s2, gam, scale, st)
                : launch_ul_f32_sig_k<32, 16, 8>(ctx, H, Y, P, K, kappa, X, s2, gam, scale, st);
}

// The north-star tile (B_c = 32, U = 16, fp32, uniform fusion) with half of
// each channel tile in TMEM (dcdg_tmem_kernels.cuh).  3 (default): ul_tmh_f32,
// 8 lanes per problem and the TMA staging slot as ul_reg_f32, odd coordinate
// blocks' columns in TMEM, 138 registers -> 3 warps per scheduler (12 per SM,
// 4-warp CTAs): 0.151 -> 0.141 ms per 134 400 problems (profiles/lab/README.md).
// 1, 2: lab variants with 4 lanes per problem (slower); 0: ul_reg_f32.
// (DCDG_UL_TMEM, DCDG_UL_TMEM_MINB: defined after the includes)
// Also the 64x16 tile (G = 16): 0.52 -> 0.55 of HBM in the configs[4] sweep;
// the 16x16 tile (G = 4, 8 problems per warp) measured 0.558 -> 0.547 and
// keeps ul_reg_f32 unless DCDG_UL_TMH_MORE = 2 (profiles/lab/README.md).
#ifndef DCDG_UL_TMH_MORE
#define DCDG_UL_TMH_MORE 1
#endif
bool ul_tm_shape(int bc, int u, int fmt) {
  return DCDG_UL_TMEM && fmt == DCDG_FP32 && u == 16 &&
         (bc == 32 || (DCDG_UL_TMEM == 3 && ((DCDG_UL_TMH_MORE >= 1 && bc == 64) ||
                                            (DCDG_UL_TMH_MORE >= 2 && bc == 16))));
}
int ul_tmh_g(int bc) { return bc == 64 ? 16 : bc == 16 ? 4 : 8; }

#if DCDG_UL_TMEM == 3
template <int BC, int G, bool XCHG = false>
cudaError_t launch_ul_tmh(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                          cudaStream_t st, const dcdg::XMap* xm = nullptr) {
  constexpr int NPW = 32 / G;
  constexpr size_t smem =
      dcdg::CtaSmem<NPW*(BC * 16 * 8 + BC * 8), dcdg::ul_scal_bytes(16, 2), NPW, dcdg::kTmhWarps>::kBytes;
  auto kern = dcdg::ul_tmh_f32<DCDG_UL_TMEM_MINB, false, BC, 16, G, XCHG>;
  // the occupancy query reports 1 CTA for this kernel although ncu's launch
  // limits (shared memory, registers) both allow 3: size the grid from MINB
  (void)occupancy_of(ctx, kern, smem, 32 * dcdg::kTmhWarps);  // sets the shared-memory attribute
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + dcdg::kTmhWarps - 1) / dcdg::kTmhWarps, ctx->sms * DCDG_UL_TMEM_MINB);
  kern<<<blocks, 32 * dcdg::kTmhWarps, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P, K,
                                                    kappa, static_cast<float2*>(X), nullptr, 0.f, 0.f, nullptr,
                                                    xm ? *xm : dcdg::XMap{});
  return cudaGetLastError();
}
// the spec-table entry of the target tile: the exchange instantiation (xm set,
// dcdg_ul_detect_xchg) on the TMEM kernel too
#ifndef DCDG_UL_TMH_XCHG
#define DCDG_UL_TMH_XCHG 1
#endif
template <int BC, int U, int G, int MINB>
cudaError_t launch_ul_f32_tmx(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                              const dcdg::XMap* xm, cudaStream_t st) {
  if (xm && DCDG_UL_TMH_XCHG) return launch_ul_tmh<BC, G, true>(ctx, H, Y, P, K, kappa, X, st, xm);
  return launch_ul_f32<BC, U, G, MINB>(ctx, H, Y, P, K, kappa, X, xm, st);
}
#endif

cudaError_t launch_ul_tm(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                         cudaStream_t st, int bc) {
#if DCDG_UL_TMEM  // lab kernels (profiles/lab/README.md): only compiled when switched on
  constexpr int NPW = 8;
  constexpr size_t smem = dcdg::kTmWarps * NPW * dcdg::ul_scal_bytes(16, 2);
#if DCDG_UL_TMEM == 3  // 4 rows per lane, odd blocks in TMEM, 3 warps per scheduler
  (void)NPW;
  if (P > 0) {
    return bc == 64 ? launch_ul_tmh<64, 16>(ctx, H, Y, P, K, kappa, X, st)
           : bc == 16 ? launch_ul_tmh<16, 4>(ctx, H, Y, P, K, kappa, X, st)
                      : launch_ul_tmh<32, 8>(ctx, H, Y, P, K, kappa, X, st);
  }
  return cudaSuccess;
#endif
#if DCDG_UL_TMEM == 2  // staged in two TMA phases per set (dcdg_tmem_kernels.cuh)
  constexpr size_t smem2 = dcdg::kTmWarps * (dcdg::kTm2SlotB + NPW * dcdg::ul_scal_bytes(16, 2)) + dcdg::kTmWarps * 16;
  auto kern2 = dcdg::ul_tm2_f32<DCDG_UL_TMEM_MINB>;
  const int occ2 = occupancy_of(ctx, kern2, smem2, 32 * dcdg::kTmWarps);
  const int nsets2 = (P + NPW - 1) / NPW;
  const int blocks2 = std::min((nsets2 + dcdg::kTmWarps - 1) / dcdg::kTmWarps, ctx->sms * occ2);
  kern2<<<blocks2, 32 * dcdg::kTmWarps, smem2, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P,
                                                      K, kappa, static_cast<float2*>(X));
  return cudaGetLastError();
#endif
  auto kern = dcdg::ul_tm_f32<DCDG_UL_TMEM_MINB>;
  const int occ = occupancy_of(ctx, kern, smem, 32 * dcdg::kTmWarps);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + dcdg::kTmWarps - 1) / dcdg::kTmWarps, ctx->sms * occ);
  kern<<<blocks, 32 * dcdg::kTmWarps, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P, K,
                                                   kappa, static_cast<float2*>(X));
  return cudaGetLastError();
#else
  (void)ctx, (void)H, (void)Y, (void)P, (void)K, (void)kappa, (void)X, (void)st, (void)bc;
  return cudaErrorNotSupported;
#endif
}

template <int BC, int U, int G, int MINB>
cudaError_t launch_ul_f16(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                          const dcdg::XMap* xm, cudaStream_t st) {
  constexpr int NPW = 32 / G;
  constexpr size_t smem =
      dcdg::CtaSmem<NPW*(BC * U * 4 + BC * 4), dcdg::ul_scal_bytes(U), NPW, kWarps>::kBytes;
  auto kern = dcdg::ul_reg_f16<BC, U, G, kWarps, MINB, false>;
  auto kx = dcdg::ul_reg_f16<BC, U, G, kWarps, MINB, true>;
  const int occ = occupancy_of(ctx, kern, smem);
  const int occx = occupancy_of(ctx, kx, smem);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + kWarps - 1) / kWarps, ctx->sms * (xm ? occx : occ));
  (xm ? kx : kern)<<<blocks, 32 * kWarps, smem, st>>>(static_cast<const __half2*>(H), static_cast<const __half2*>(Y),
                                                       P, K, kappa, static_cast<__half2*>(X),
                                                       xm ? *xm : dcdg::XMap{});
  return cudaGetLastError();
}

// lab: the effective-gain instantiation of the downlink kernel may run with
// fewer resident warps per SM (more registers for v = H_c s)
#ifndef DCDG_DL_GAIN_MINB_DELTA
#define DCDG_DL_GAIN_MINB_DELTA 0
#endif
template <int BC, int U, int G, int MINB, bool GAIN>
cudaError_t launch_dl_f32_k(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                            float* gp, cudaStream_t st) {
  constexpr int NPW = 32 / G;
  constexpr size_t smem =
      dcdg::CtaSmem<NPW*(BC * U * 8 + U * 8), dcdg::dl_scal_bytes(U), NPW, kWarps>::kBytes;
  auto kern = dcdg::dl_reg_f32<BC, U, G, kWarps, (GAIN ? MINB - DCDG_DL_GAIN_MINB_DELTA : MINB), GAIN>;
  const int occ = occupancy_of(ctx, kern, smem);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + kWarps - 1) / kWarps, ctx->sms * occ);
  kern<<<blocks, 32 * kWarps, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(S), P, C, K, rho_c,
                                          static_cast<float2*>(X), gp, ctx->d_status);
  return cudaGetLastError();
}

template <int BC, int U, int G, int MINB>
cudaError_t launch_dl_f32(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                          float* gp, cudaStream_t st) {
  return gp ? launch_dl_f32_k<BC, U, G, MINB, true>(ctx, H, S, P, C, K, rho_c, X, gp, st)
            : launch_dl_f32_k<BC, U, G, MINB, false>(ctx, H, S, P, C, K, rho_c, X, gp, st);
}

template <int BC, int U, int G, int MINB, bool GAIN>
cudaError_t launch_dl_f16_k(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                            float* gp, cudaStream_t st) {
  constexpr int NPW = 32 / G;
  constexpr size_t smem =
      dcdg::CtaSmem<NPW*(BC * U * 4 + U * 4), dcdg::dl_scal_bytes(U), NPW, kWarps>::kBytes;
  auto kern = dcdg::dl_reg_f16<BC, U, G, kWarps, MINB, GAIN>;
  const int occ = occupancy_of(ctx, kern, smem);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min((nsets + kWarps - 1) / kWarps, ctx->sms * occ);
  kern<<<blocks, 32 * kWarps, smem, st>>>(static_cast<const __half2*>(H), static_cast<const __half2*>(S), P, C, K,
                                          rho_c, static_cast<__half2*>(X), gp, ctx->d_status);
  return cudaGetLastError();
}

template <int BC, int U, int G, int MINB>
cudaError_t launch_dl_f16(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                          float* gp, cudaStream_t st) {
  return gp ? launch_dl_f16_k<BC, U, G, MINB, true>(ctx, H, S, P, C, K, rho_c, X, gp, st)
            : launch_dl_f16_k<BC, U, G, MINB, false>(ctx, H, S, P, C, K, rho_c, X, gp, st);
}

// Multi-warp kernels (one CTA of NW warps per problem, dcdg_mw_kernels.cuh)
template <int BC, int U, int NW, int MINB>
cudaError_t launch_ul_mw(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                         const dcdg::XMap* /*no exchange epilogue: dcdg_ul_detect_xchg uses xchg_put_kernel*/,
                         cudaStream_t st) {
  constexpr int LB = DCDG_LB_UL_MW;
  constexpr size_t smem = dcdg::MwSmem<dcdg::ul_mw_slot_bytes(BC, U, NW), dcdg::ul_scal_bytes(U, LB), NW,
                                       dcdg::mw_setup_floats(U, LB), 2 * LB>::kBytes;
  auto kern = dcdg::ul_mw_f32<BC, U, NW, MINB, LB>;
  const int occ = occupancy_of(ctx, kern, smem, 32 * NW);
  const int blocks = std::min(P, ctx->sms * occ);
  kern<<<blocks, 32 * NW, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P, K, kappa,
                                      static_cast<float2*>(X));
  return cudaGetLastError();
}

template <int BC, int U, int NW, int MINB, bool GAIN>
cudaError_t launch_dl_mw_k(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                           float* gp, cudaStream_t st) {
  constexpr size_t smem = dcdg::MwSmem<dcdg::dl_mw_slot_bytes(BC, U, NW), dcdg::dl_scal_bytes(U), NW,
                                       dcdg::mw_setup_floats(U, 2), 4>::kBytes;
  auto kern = dcdg::dl_mw_f32<BC, U, NW, MINB, GAIN>;
  const int occ = occupancy_of(ctx, kern, smem, 32 * NW);
  const int blocks = std::min(P, ctx->sms * occ);
  kern<<<blocks, 32 * NW, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(S), P, C, K, rho_c,
                                      static_cast<float2*>(X), gp, ctx->d_status);
  return cudaGetLastError();
}

template <int BC, int U, int NW, int MINB>
cudaError_t launch_dl_mw(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                         float* gp, cudaStream_t st) {
  return gp ? launch_dl_mw_k<BC, U, NW, MINB, true>(ctx, H, S, P, C, K, rho_c, X, gp, st)
            : launch_dl_mw_k<BC, U, NW, MINB, false>(ctx, H, S, P, C, K, rho_c, X, gp, st);
}

// Kernel of one direction: kind 0 register-resident (a = lanes per problem),
// 1 multi-warp (a = warps per problem), 2 split tile (a = lanes, b = register
// columns; dcdg_split_kernels.cuh).
// Split-tile kernels (dcdg_split_kernels.cuh): one-warp CTAs, grid = SMs x occupancy.
// DCDG_SPLIT_PF: sets of L2 prefetch lead.
#ifndef DCDG_SPLIT_PF
#define DCDG_SPLIT_PF 1
#endif
template <int BC, int U, int G, int JR, int MINB>
cudaError_t launch_ul_split(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X,
                            const dcdg::XMap* /*exchange via xchg_put_kernel*/, cudaStream_t st) {
  constexpr int NPW = 32 / G;
  constexpr size_t smem = dcdg::split_cols_bytes(BC, U, JR, G) + NPW * dcdg::ul_scal_bytes(U, 2);
  auto kern = dcdg::ul_split_f32<BC, U, G, JR, MINB, DCDG_SPLIT_PF>;
  const int occ = occupancy_of(ctx, kern, smem, 32);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min(nsets, ctx->sms * occ);
  kern<<<blocks, 32, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(Y), P, K, kappa,
                                 static_cast<float2*>(X));
  return cudaGetLastError();
}

template <int BC, int U, int G, int JR, int MINB, bool GAIN>
cudaError_t launch_dl_split_k(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                              float* gp, cudaStream_t st) {
  constexpr int NPW = 32 / G;
  constexpr size_t smem = dcdg::split_cols_bytes(BC, U, JR, G) + NPW * dcdg::dl_scal_bytes(U);
  auto kern = dcdg::dl_split_f32<BC, U, G, JR, MINB, GAIN, DCDG_SPLIT_PF>;
  const int occ = occupancy_of(ctx, kern, smem, 32);
  const int nsets = (P + NPW - 1) / NPW;
  const int blocks = std::min(nsets, ctx->sms * occ);
  kern<<<blocks, 32, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(S), P, C, K, rho_c,
                                 static_cast<float2*>(X), gp, ctx->d_status);
  return cudaGetLastError();
}

template <int BC, int U, int G, int JR, int MINB>
cudaError_t launch_dl_split(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X,
                            float* gp, cudaStream_t st) {
  return gp ? launch_dl_split_k<BC, U, G, JR, MINB, true>(ctx, H, S, P, C, K, rho_c, X, gp, st)
            : launch_dl_split_k<BC, U, G, JR, MINB, false>(ctx, H, S, P, C, K, rho_c, X, gp, st);
}

struct KDesc {
  int kind, a, b;
};
constexpr int kReg = 0, kMw = 1, kSplit = 2, kPp2 = 3;

struct Spec {
  int bc, u, fmt;
  UlLaunch ul;
  KDesc ulk;
  DlLaunch dl;
  KDesc dlk;
};

// Register-resident specialisations: B_c*U/G complex per lane = 128 regs of
// channel for fp32 (64-128 for fp16).  Everything else runs the generic path.
// Minimum resident warps per SM requested from ptxas per kernel family
// (register cap = 65536 / (32 * warps)); tuned on B200 with scripts/kbench.py.
#ifndef DCDG_MIN_WARPS_UL_F32
#define DCDG_MIN_WARPS_UL_F32 8
#endif
#ifndef DCDG_MIN_WARPS_DL_F32
#define DCDG_MIN_WARPS_DL_F32 10
#endif
#ifndef DCDG_MIN_WARPS_UL_F16
#define DCDG_MIN_WARPS_UL_F16 8
#endif
#ifndef DCDG_MIN_WARPS_DL_F16
#define DCDG_MIN_WARPS_DL_F16 8
#endif
#ifndef DCDG_MIN_WARPS_SPLIT
#define DCDG_MIN_WARPS_SPLIT 8
#endif
// lanes per problem of the fp16 north-star kernel (B_c=32, U=16)
#ifndef DCDG_F16_G_TARGET
#define DCDG_F16_G_TARGET 4
#endif
// lanes per problem of the paper's 32x8 tile (configs[0])
#ifndef DCDG_G_32x8
#define DCDG_G_32x8 4
#endif
// lanes per problem of the 16x16 downlink tile (B=128, C=8)
#ifndef DCDG_G_16x16_DL
#define DCDG_G_16x16_DL 4
#endif
// lanes per problem of the 16x16 uplink tile
#ifndef DCDG_G_16x16_UL
#define DCDG_G_16x16_UL 4
#endif
constexpr int minb(int warps) { return warps / kWarps > 0 ? warps / kWarps : 1; }
constexpr int minb_mw(int warps, int nw) { return warps / nw > 0 ? warps / nw : 1; }

#define UL_REG(BC, U, G) launch_ul_f32<BC, U, G, minb(DCDG_MIN_WARPS_UL_F32)>, KDesc{kReg, G, 0}
#define DL_REG(BC, U, G) launch_dl_f32<BC, U, G, minb(DCDG_MIN_WARPS_DL_F32)>, KDesc{kReg, G, 0}
#define UL_MW(BC, U, NW) launch_ul_mw<BC, U, NW, minb_mw(DCDG_MIN_WARPS_UL_F32, NW)>, KDesc{kMw, NW, 0}
#define DL_MW(BC, U, NW) launch_dl_mw<BC, U, NW, minb_mw(DCDG_MIN_WARPS_UL_F32, NW)>, KDesc{kMw, NW, 0}
#define UL_SPLIT(BC, U, G, JR) launch_ul_split<BC, U, G, JR, DCDG_MIN_WARPS_SPLIT>, KDesc{kSplit, G, JR}
#define DL_SPLIT(BC, U, G, JR) launch_dl_split<BC, U, G, JR, DCDG_MIN_WARPS_SPLIT>, KDesc{kSplit, G, JR}
#define UL_F16(BC, U, G) launch_ul_f16<BC, U, G, minb(DCDG_MIN_WARPS_UL_F16)>, KDesc{kReg, G, 0}
#define DL_F16(BC, U, G) launch_dl_f16<BC, U, G, minb(DCDG_MIN_WARPS_DL_F16)>, KDesc{kReg, G, 0}

// Measured on B200 (profiles/r01_configs4_sweep.json, scripts/lab/lab_split2.cu):
// the split tile wins wherever the register kernel needs G >= 16 lanes or
// several warps per problem; at B_c = 32, U = 16 the register kernel stays.
const Spec kSpecs[] = {
#if DCDG_UL_PP2
    {32, 16, DCDG_FP32, launch_ul_pp2<32, 16, 8, minb(DCDG_MIN_WARPS_UL_F32)>, KDesc{kPp2, 16, 0}, DL_REG(32, 16, 8)},
#else
#if DCDG_UL_TMEM == 3
    {32, 16, DCDG_FP32, launch_ul_f32_tmx<32, 16, 8, minb(DCDG_MIN_WARPS_UL_F32)>, KDesc{kReg, 8, 0},
     DL_REG(32, 16, 8)},  // north-star target: B=256, C=8, U=16 (uniform path: ul_tm_shape)
#else
    {32, 16, DCDG_FP32, UL_REG(32, 16, 8), DL_REG(32, 16, 8)},  // north-star target: B=256, C=8, U=16
#endif
#endif
    {32, 8, DCDG_FP32, UL_REG(32, 8, DCDG_G_32x8), DL_REG(32, 8, DCDG_G_32x8)},  // paper / config 1: B_c=32, U=8
    {16, 16, DCDG_FP32, UL_REG(16, 16, DCDG_G_16x16_UL), DL_REG(16, 16, DCDG_G_16x16_DL)},  // B=128, C=8
    {64, 16, DCDG_FP32, UL_REG(64, 16, 16), DL_REG(64, 16, 16)},  // B=256, C=4 / B=512, C=8
    {64, 8, DCDG_FP32, UL_REG(64, 8, 8), DL_REG(64, 8, 8)},
    {128, 16, DCDG_FP32, UL_SPLIT(128, 16, 16, 8), DL_REG(128, 16, 32)},  // B=128,C=1 / 256,2 / 512,4
    {16, 32, DCDG_FP32, UL_REG(16, 32, 8), DL_REG(16, 32, 8)},    // configs[4]: U=32
    {32, 32, DCDG_FP32, UL_SPLIT(32, 32, 8, 16), DL_SPLIT(32, 32, 8, 16)},
    {64, 32, DCDG_FP32, UL_SPLIT(64, 32, 16, 16), DL_SPLIT(64, 32, 16, 16)},
    {128, 32, DCDG_FP32, UL_SPLIT(128, 32, 32, 16), DL_SPLIT(128, 32, 32, 16)},
    {256, 16, DCDG_FP32, UL_SPLIT(256, 16, 32, 8), DL_SPLIT(256, 16, 32, 8)},
    {512, 16, DCDG_FP32, UL_SPLIT(512, 16, 32, 4), DL_MW(512, 16, 4)},
    {256, 32, DCDG_FP32, UL_SPLIT(256, 32, 32, 8), DL_SPLIT(256, 32, 32, 8)},
    {512, 32, DCDG_FP32, UL_SPLIT(512, 32, 32, 4), DL_MW(512, 32, 8)},
    {1024, 16, DCDG_FP32, UL_MW(1024, 16, 8), DL_MW(1024, 16, 8)},  // one CTA of 8 warps per problem
    {32, 16, DCDG_FP16, UL_F16(32, 16, DCDG_F16_G_TARGET), DL_F16(32, 16, DCDG_F16_G_TARGET)},  // half2 target
    {32, 8, DCDG_FP16, UL_F16(32, 8, 4), DL_F16(32, 8, 4)},
    {16, 16, DCDG_FP16, UL_F16(16, 16, 4), DL_F16(16, 16, 4)},
    {64, 16, DCDG_FP16, UL_F16(64, 16, 8), DL_F16(64, 16, 8)},
};

// ---------------------------------------------------------------------------
// Gram-space fp16 uplink (dcdg_gram_kernels.cuh): B_c = 32, U = 16.
// ---------------------------------------------------------------------------
#ifndef DCDG_GRAM_MINB
#define DCDG_GRAM_MINB 16
#endif
#ifndef DCDG_GRAM_SIG_MINB  // the variance-fused instance (optimal fusion)
#define DCDG_GRAM_SIG_MINB 12  // 168 registers (30 spilled loop invariants), 0.283 vs 0.289 ms at 16 warps (profiles/lab/README.md)
#endif
constexpr int kGramNpw = 4;

bool gram_shape(int bc, int u, int fmt) { return fmt == DCDG_FP16 && bc == 32 && u == 16; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// sigma2 != NULL: optimal fusion, post_eq_variance fused into the same kernel
// (gam = E_x/N0, scale = E_x/U) from the Gram it already holds
int launch_ul_gram(dcdg_ctx* ctx, const void* H, const void* Y, int P, int K, float kappa, void* X, cudaStream_t st,
                   float* sigma2 = nullptr, float gam = 0.f, float scale = 0.f) {
  constexpr int U = 16, NPW = kGramNpw;
  using L = dcdg::GramSmem<U, NPW>;
  auto encode = tensor_map_encoder();
  if (!encode) return fail(DCDG_ECUDA, "dcdg_ul_detect: cuTensorMapEncodeTiled unavailable");
  // the tiles as rows of 128 B (one fp16 column of 32 antennas), P*U rows
  CUtensorMap map;
  const cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(P) * U};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(NPW * U)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(H), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DCDG_ECUDA, "dcdg_ul_detect: tensor map encode failed (" + std::to_string(r) + ")");
  const int nsets = (P + NPW - 1) / NPW;
  if (sigma2) {
    auto kern = dcdg::ul_gram_f16<U, NPW, DCDG_GRAM_SIG_MINB, true>;
    const int occ = occupancy_of(ctx, kern, L::kAlloc, 32);
    const int blocks = std::min(nsets, ctx->sms * occ);
    kern<<<blocks, 32, L::kAlloc, st>>>(map, static_cast<const __half2*>(Y), P, K, kappa, static_cast<__half2*>(X),
                                        sigma2, gam, scale, ctx->d_status);
  } else {
    auto kern = dcdg::ul_gram_f16<U, NPW, DCDG_GRAM_MINB, false>;
    const int occ = occupancy_of(ctx, kern, L::kAlloc, 32);
    const int blocks = std::min(nsets, ctx->sms * occ);
    kern<<<blocks, 32, L::kAlloc, st>>>(map, static_cast<const __half2*>(Y), P, K, kappa, static_cast<__half2*>(X),
                                        nullptr, 0.f, 0.f, nullptr);
  }
  CUDA_TRY(cudaGetLastError(), "ul_gram launch");
  return DCDG_OK;
}

int launch_dl_gram(dcdg_ctx* ctx, const void* H, const void* S, int P, int C, int K, float rho_c, void* X, float* gp,
                   cudaStream_t st) {
  constexpr int U = 16, NPW = kGramNpw;
  using L = dcdg::GramSmem<U, NPW>;
  auto encode = tensor_map_encoder();
  if (!encode) return fail(DCDG_ECUDA, "dcdg_dl_precode: cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;  // as launch_ul_gram: P*U rows of 128 B
  const cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(P) * U};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(NPW * U)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(H), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DCDG_ECUDA, "dcdg_dl_precode: tensor map encode failed (" + std::to_string(r) + ")");
  const int nsets = (P + NPW - 1) / NPW;
#define DL_GRAM(GAIN)                                                                                              \
  {                                                                                                                \
    auto kern = dcdg::dl_gram_f16<U, NPW, DCDG_GRAM_MINB, GAIN>;                                                   \
    const int occ = occupancy_of(ctx, kern, L::kAlloc, 32);                                                      \
    const int blocks = std::min(nsets, ctx->sms * occ);                                                           \
    kern<<<blocks, 32, L::kAlloc, st>>>(map, static_cast<const __half2*>(H), static_cast<const __half2*>(S), P, C, K, \
                                        rho_c, static_cast<__half2*>(X), gp, ctx->d_status);                       \
  }
  if (gp)
    DL_GRAM(true)
  else
    DL_GRAM(false)
#undef DL_GRAM
  CUDA_TRY(cudaGetLastError(), "dl_gram launch");
  return DCDG_OK;
}

const Spec* find_spec(int bc, int u, int fmt) {
  for (const auto& s : kSpecs)
    if (s.bc == bc && s.u == u && s.fmt == fmt) return &s;
  return nullptr;
}

int check_ctx(dcdg_ctx* ctx) {
  if (!ctx) return fail(DCDG_EINVAL, "dcdg: null context");
  return DCDG_OK;
}

int check_fmt(int fmt) {
  if (fmt != DCDG_FP32 && fmt != DCDG_FP16) return fail(DCDG_EINVAL, "dcdg: unknown storage format");
  return DCDG_OK;
}

int launch_fuse(dcdg_ctx* ctx, const void* xl, const float* s2, int S, int C, int C_total, int U, int fmt,
                bool optimal, float* xhat, float* wsum, cudaStream_t st) {
  const long long n = static_cast<long long>(S) * U;
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>((n + threads - 1) / threads);
  if (fmt == DCDG_FP16)
    CUDA_TRY(launch_dependent(dcdg::fuse_kernel<__half2>, blocks, threads, 0, st, static_cast<const __half2*>(xl), s2, S,
                              C, C_total, U, optimal, reinterpret_cast<float2*>(xhat), wsum, ctx->d_status),
             "fuse launch");
  else
    CUDA_TRY(launch_dependent(dcdg::fuse_kernel<float2>, blocks, threads, 0, st, static_cast<const float2*>(xl), s2, S,
                              C, C_total, U, optimal, reinterpret_cast<float2*>(xhat), wsum, ctx->d_status),
             "fuse launch");
  ++ctx->launches;
  return DCDG_OK;
}

// Gram/Cholesky kernels: post_eq_variance (mode kPev, one tile per problem) and
// the full-H MMSE bias factors (mode kBias, the NT cluster tiles of a subcarrier).
template <int MODE>
int launch_gram_chol(dcdg_ctx* ctx, const void* H, int P, int NT, int Bc, int U, float a0, float a1, float scale,
                     int fmt, float* out, cudaStream_t st) {
  const size_t smem = 4 * static_cast<size_t>(dcdg::pev_smem_per_warp(U));
  const int blocks = (P + 3) / 4;
#define GC_LAUNCH(T, UT, BT)                                                                                \
  {                                                                                                         \
    auto k = dcdg::gram_chol<T, UT, BT, MODE>;                                                              \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));           \
    k<<<blocks, 128, smem, st>>>(static_cast<const T*>(H), P, NT, Bc, U, a0, a1, scale,                     \
                                 MODE == dcdg::kPev && fmt == DCDG_FP16, out, ctx->d_status, nullptr, nullptr); \
  }
#define GC_DISPATCH(T)                            \
  if (U == 16 && Bc == 32) GC_LAUNCH(T, 16, 32)   \
  else if (U == 8 && Bc == 32) GC_LAUNCH(T, 8, 32) \
  else switch (U) {                               \
    case 8: GC_LAUNCH(T, 8, 0) break;             \
    case 16: GC_LAUNCH(T, 16, 0) break;           \
    case 32: GC_LAUNCH(T, 32, 0) break;           \
    default: GC_LAUNCH(T, 0, 0) break;            \
  }
  if (fmt == DCDG_FP16)
    GC_DISPATCH(__half2)
  else
    GC_DISPATCH(float2)
#undef GC_DISPATCH
#undef GC_LAUNCH
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "gram/cholesky launch");
  return DCDG_OK;
}

// Exact solvers (fp32 tiles): one warp per subcarrier over its C stacked tiles.
template <int MODE>
int launch_solve(dcdg_ctx* ctx, const void* H, const void* V, int S, int C, int Bc, int U, float a0, float scale,
                 float2* xo, cudaStream_t st) {
  const size_t smem = 4 * static_cast<size_t>(dcdg::pev_smem_per_warp(U));
  const int blocks = (S + 3) / 4;
#define SV_LAUNCH(UT)                                                                                        \
  {                                                                                                          \
    auto k = dcdg::gram_chol<float2, UT, 0, MODE>;                                                           \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));            \
    k<<<blocks, 128, smem, st>>>(static_cast<const float2*>(H), S, C, Bc, U, a0, 1.f, scale, false, nullptr, \
                                 ctx->d_status, static_cast<const float2*>(V), xo);                          \
  }
  switch (U) {
    case 8: SV_LAUNCH(8) break;
    case 16: SV_LAUNCH(16) break;
    case 32: SV_LAUNCH(32) break;
    default: SV_LAUNCH(0) break;
  }
#undef SV_LAUNCH
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "exact solver launch");
  return DCDG_OK;
}

// U = 16 runs two problems per warp (pev16_pair_kernel) for the common antenna
// counts; everything else the one-warp-per-problem gram_chol.
template <typename T, int BT>
int launch_pev16(dcdg_ctx* ctx, const void* H, int P, float gam, float scale, bool rnd, float* s2, cudaStream_t st) {
  constexpr size_t smem = 4 * (2 * 16 * (BT + 1) + 2 * 16 * 16) * sizeof(float2);
  auto k = dcdg::pev16_pair_kernel<T, BT>;
  occupancy_of(ctx, k, smem, 128);  // sets the shared-memory opt-in on this device (cached per device)
  k<<<(P + 7) / 8, 128, smem, st>>>(static_cast<const T*>(H), P, gam, scale, rnd, s2, ctx->d_status);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "post_eq_variance launch");
  return DCDG_OK;
}

// fp32 tiles with U in {8, 16, 32}: the tensor-core Gram + column-pair sweep
// operator kernel (dcdg_pev_kernels.cuh)
#ifndef DCDG_PEV_TC
#define DCDG_PEV_TC 1
#endif
#ifndef DCDG_PEV_TC_MINB
#define DCDG_PEV_TC_MINB 8
#endif
template <int U, typename T = float2>
int launch_pev_tc(dcdg_ctx* ctx, const void* H, int P, int Bc, float gam, float scale, float* s2, cudaStream_t st) {
  using L = dcdg::PevTcSmem<U>;
  constexpr size_t smem = L::kWarpB;
  auto k = dcdg::pev_tc_kernel<U, DCDG_PEV_TC_MINB, T>;
  const int occ = occupancy_of(ctx, k, smem, 32);
  const int nsets = (P + L::kNpw - 1) / L::kNpw;
  const int blocks = std::min(nsets, ctx->sms * occ);
  k<<<blocks, 32, smem, st>>>(static_cast<const T*>(H), P, Bc, gam, scale, s2, ctx->d_status);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "post_eq_variance launch");
  return DCDG_OK;
}

#ifndef DCDG_PEV_PAIR
#define DCDG_PEV_PAIR 1
#endif
int launch_post_eq(dcdg_ctx* ctx, const void* H, int P, int Bc, int U, double n0, double ex, int fmt, float* s2,
                   cudaStream_t st) {
  const float gam = static_cast<float>(ex / n0), scale = static_cast<float>(ex / U);
  // (B_c <= 256: beyond that the tensor cores' fp32 accumulation over 2 B_c
  // real terms leaves sigma^2 at the 1e-5 parity edge; the FFMA Gram is used)
  if (DCDG_PEV_TC && fmt == DCDG_FP32 && Bc % 4 == 0 && Bc <= 256) {
    if (U == 16) return launch_pev_tc<16>(ctx, H, P, Bc, gam, scale, s2, st);
    if (U == 32) return launch_pev_tc<32>(ctx, H, P, Bc, gam, scale, s2, st);
    if (U == 8) return launch_pev_tc<8>(ctx, H, P, Bc, gam, scale, s2, st);
  }
  // fp16 tiles: the stored binary16 values multiply exactly on the tensor cores
  if (DCDG_PEV_TC && fmt == DCDG_FP16 && Bc % 8 == 0) {
    if (U == 16) return launch_pev_tc<16, __half2>(ctx, H, P, Bc, gam, scale, s2, st);
    if (U == 32) return launch_pev_tc<32, __half2>(ctx, H, P, Bc, gam, scale, s2, st);
    if (U == 8) return launch_pev_tc<8, __half2>(ctx, H, P, Bc, gam, scale, s2, st);
  }
  if (DCDG_PEV_PAIR && U == 16) {
    const bool rnd = fmt == DCDG_FP16;
#define PEV16(BT)                                                                                  \
  if (Bc == BT)                                                                                    \
    return fmt == DCDG_FP16 ? launch_pev16<__half2, BT>(ctx, H, P, gam, scale, rnd, s2, st)        \
                            : launch_pev16<float2, BT>(ctx, H, P, gam, scale, rnd, s2, st);
    PEV16(32)
    PEV16(16)
    PEV16(64)
#undef PEV16
  }
  return launch_gram_chol<dcdg::kPev>(ctx, H, P, 1, Bc, U, 1.f, gam, scale, fmt, s2, st);
}

}  // namespace

extern "C" {

int dcdg_abi_version(void) { return DCDG_ABI_VERSION; }

int dcdg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char* dcdg_last_error(void) { return g_err.c_str(); }

int dcdg_init(int device, dcdg_ctx** out) {
  if (!out) return fail(DCDG_EINVAL, "dcdg_init: null output pointer");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(DCDG_ECUDA, "dcdg_init: no CUDA device available (there is no CPU fallback)");
  if (device < 0 || device >= n) return fail(DCDG_EINVAL, "dcdg_init: device index out of range");
  CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
  auto* ctx = new dcdg_ctx;
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  e = cudaMalloc(&ctx->d_status, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_fail(e, "dcdg_init status buffer");
  }
  cudaMemset(ctx->d_status, 0xff, sizeof(unsigned long long));
  cudaDeviceSynchronize();
  *out = ctx;
  return DCDG_OK;
}

int dcdg_destroy(dcdg_ctx* ctx) {
  if (!ctx) return DCDG_OK;
  cudaSetDevice(ctx->device);
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->scratch) cudaFree(ctx->scratch);
  delete ctx;
  return DCDG_OK;
}

uint64_t dcdg_launch_count(dcdg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int dcdg_set_fp16_algorithm(dcdg_ctx* ctx, int alg) {
  if (int rc = check_ctx(ctx)) return rc;
  if (alg != DCDG_ALG_SWEEP && alg != DCDG_ALG_GRAM) return fail(DCDG_EINVAL, "dcdg_set_fp16_algorithm: unknown algorithm");
  ctx->fp16_alg = alg;
  return DCDG_OK;
}

int dcdg_ctx_kernel_name(dcdg_ctx* ctx, int direction, int Bc, int U, int fmt, char* buf, int len) {
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->fp16_alg == DCDG_ALG_GRAM && gram_shape(Bc, U, fmt)) {
    if (buf && len > 0) {
      std::snprintf(buf, static_cast<size_t>(len), "%s_gram_f16<%d,%d,%d>", direction ? "dl" : "ul", Bc, U, kGramNpw);
    }
    return DCDG_OK;
  }
  return dcdg_kernel_name(direction, Bc, U, fmt, buf, len);
}

int dcdg_kernel_name(int direction, int Bc, int U, int fmt, char* buf, int len) {
  const Spec* s = find_spec(Bc, U, fmt);
  char tmp[96];
  const char* dir = direction ? "dl" : "ul";
  const char* f = fmt == DCDG_FP16 ? "f16" : "f32";
  const KDesc* kd = s ? (direction ? &s->dlk : &s->ulk) : nullptr;
  if (!direction && ul_tm_shape(Bc, U, fmt))
    std::snprintf(tmp, sizeof tmp, DCDG_UL_TMEM == 3 ? "ul_tmh_f32<%d,%d,%d>" : "ul_tm_f32<%d,%d,%d>", Bc, U,
                  DCDG_UL_TMEM == 3 ? ul_tmh_g(Bc) : 4);
  else if (kd && kd->kind == kPp2)
    std::snprintf(tmp, sizeof tmp, "%s_pp2_%s<%d,%d,%d>", dir, f, Bc, U, kd->a);
  else if (kd && kd->kind == kMw)
    std::snprintf(tmp, sizeof tmp, "%s_mw_%s<%d,%d,%d>", dir, f, Bc, U, kd->a);
  else if (kd && kd->kind == kSplit)
    std::snprintf(tmp, sizeof tmp, "%s_split_%s<%d,%d,%d,%d>", dir, f, Bc, U, kd->a, kd->b);
  else if (kd)
    std::snprintf(tmp, sizeof tmp, "%s_reg_%s<%d,%d,%d>", dir, f, Bc, U, kd->a);
  else
    std::snprintf(tmp, sizeof tmp, "%s_generic_%s", dir, f);
  if (buf && len > 0) {
    std::strncpy(buf, tmp, static_cast<size_t>(len - 1));
    buf[len - 1] = 0;
  }
  return DCDG_OK;
}

int dcdg_sync_status(dcdg_ctx* ctx, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  CUDA_TRY(cudaStreamSynchronize(as_stream(stream)), "stream synchronize");
  unsigned long long key = ~0ULL;
  CUDA_TRY(cudaMemcpy(&key, ctx->d_status, sizeof key, cudaMemcpyDeviceToHost), "status read");
  return dcdg_status_decode(ctx, key);
}

#ifndef DCDG_STATUS_KERNEL
#define DCDG_STATUS_KERNEL 1
#endif
int dcdg_status_enqueue(dcdg_ctx* ctx, unsigned long long* host_word, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!host_word) return fail(DCDG_EINVAL, "dcdg_status_enqueue: null host word");
#if DCDG_STATUS_KERNEL
  // a one-thread kernel stores the word into the (pinned, UVA-mapped) host
  // word: one kernel node instead of a copy node in the caller's stream/graph
  dcdg::status_mirror_kernel<<<1, 1, 0, as_stream(stream)>>>(ctx->d_status, host_word);
  CUDA_TRY(cudaGetLastError(), "status mirror launch");
#else
  CUDA_TRY(cudaMemcpyAsync(host_word, ctx->d_status, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           as_stream(stream)),
           "status copy");
#endif
  return DCDG_OK;
}

int dcdg_status_decode(dcdg_ctx* ctx, unsigned long long key) {
  if (int rc = check_ctx(ctx)) return rc;
  if (key == ~0ULL) return DCDG_OK;
  CUDA_TRY(cudaMemset(ctx->d_status, 0xff, sizeof(unsigned long long)), "status reset");
  const unsigned code = static_cast<unsigned>((key >> 16) & 0xff);
  const unsigned detail = static_cast<unsigned>(key & 0xffff);
  g_err_problem = static_cast<long long>(key >> 24);
  switch (code) {
    case dcdg::ST_ZERO_ROW:
      g_err = "cd_precode: user " + std::to_string(detail) + " has an all-zero channel row";
      return DCDG_ENUMERIC;
    case dcdg::ST_ZERO_BEAMFORMER:
      g_err = "power_scale: zero beamformer cannot be scaled";
      return DCDG_ENUMERIC;
    case dcdg::ST_SINGULAR:
      g_err = "hermitian_solve: matrix is numerically singular";
      return DCDG_ENUMERIC;
    case dcdg::ST_BAD_VARIANCE:
      g_err = "fusion_weights: variances must be positive and finite";
      return DCDG_EINVAL;
    case dcdg::ST_RANK_DEFICIENT:
      g_err = "zf_exact: channel rows are rank deficient";
      return DCDG_ENUMERIC;
    case dcdg::ST_MF_ZERO_ENERGY:
      g_err = "mf_detect: user " + std::to_string(detail) + " has zero channel energy";
      return DCDG_ENUMERIC;
    case dcdg::ST_MF_ZERO_BEAMFORMER:
      g_err = "mf_precode: cluster " + std::to_string(detail) + " produced a zero beamformer";
      return DCDG_ENUMERIC;
    case dcdg::ST_XCHG_TIMEOUT:
      g_err = "fused exchange: rank " + std::to_string(detail) + " never published this batch";
      return DCDG_ECUDA;
    default:
      g_err = "dcdg: unknown device status";
      return DCDG_ENUMERIC;
  }
}

long long dcdg_last_error_problem(void) { return g_err_problem; }

int dcdg_ul_detect(dcdg_ctx* ctx, const void* H, const void* y, int S, int C, int C_total, int Bc, int U, int K,
                   double n0, double ex, int fmt, int fusion, void* x_local, float* sigma2, float* xhat, float* wsum,
                   void* stream) {
  NvtxRange nvtx_("dcdg_ul_detect");
  if (int rc = check_fmt(fmt)) return rc;
  // argument checks in the reference's order and words (detect.cpp:12-19,71-72,150-155)
  if (C <= 0 || S < 0) return fail(DCDG_EINVAL, "decentralized_cd_detect: no clusters");
  if (C_total < C) return fail(DCDG_EINVAL, "dcdg_ul_detect: C_total must be >= C");
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "detector: empty channel matrix");
  if (n0 < 0.0 || !(ex > 0.0)) return fail(DCDG_EINVAL, "detector: need N0 >= 0 and E_x > 0");
  if (K <= 0) return fail(DCDG_EINVAL, "cd_detect: need at least one sweep");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  const bool optimal = fusion == DCDG_FUSION_OPTIMAL;
  if (fusion != DCDG_FUSION_OPTIMAL && fusion != DCDG_FUSION_UNIFORM)
    return fail(DCDG_EINVAL, "dcdg_ul_detect: unknown fusion mode");
  if (optimal && !(n0 > 0.0)) return fail(DCDG_EINVAL, "post_eq_variance: need N0 > 0 and E_x > 0");
  // the variance kernels factorise U x U Grams with one lane per row
  if (optimal && U > 32) return fail(DCDG_EINVAL, "dcdg_post_eq_variance: U > 32 not supported");
  if (!H || !y) return fail(DCDG_EINVAL, "dcdg_ul_detect: null input buffer");
  const long long P = static_cast<long long>(S) * C;
  if (P > 0x7fffffffLL) return fail(DCDG_EINVAL, "dcdg_ul_detect: batch too large (S*C must fit in int32)");
  if (int rc = check_ctx(ctx)) return rc;  // after the device-independent argument checks
  if (P == 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);
  const size_t xl_bytes = static_cast<size_t>(P) * U * esize(fmt);
  const size_t s2_bytes = optimal ? static_cast<size_t>(P) * sizeof(float) : 0;
  size_t need = 0;
  if (!x_local) need += (xl_bytes + 255) & ~size_t(255);
  if (optimal && !sigma2) need += (s2_bytes + 255) & ~size_t(255);
  if (need)
    if (int rc = ensure_scratch(ctx, need)) return rc;
  unsigned char* sp = static_cast<unsigned char*>(ctx->scratch);
  if (!x_local) {
    x_local = sp;
    sp += (xl_bytes + 255) & ~size_t(255);
  }
  if (optimal && !sigma2) sigma2 = reinterpret_cast<float*>(sp);

  const float kappa = static_cast<float>(n0 / ex);
  const Spec* spec = find_spec(Bc, U, fmt);
  const bool gram = ctx->fp16_alg == DCDG_ALG_GRAM && gram_shape(Bc, U, fmt);
  if (gram) {
    if (int rc = launch_ul_gram(ctx, H, y, static_cast<int>(P), K, kappa, x_local, st, optimal ? sigma2 : nullptr,
                                static_cast<float>(ex / n0), static_cast<float>(ex / U)))
      return rc;
  } else if (optimal && ul_sig_shape(Bc, U, fmt)) {
    CUDA_TRY(launch_ul_f32_sig(ctx, H, y, static_cast<int>(P), K, kappa, x_local, sigma2, static_cast<float>(ex / n0),
                               static_cast<float>(ex / U), U, st),
             "ul_detect (fused variance) launch");
  } else if (ul_tm_shape(Bc, U, fmt)) {
    CUDA_TRY(launch_ul_tm(ctx, H, y, static_cast<int>(P), K, kappa, x_local, st, Bc), "ul_detect (TMEM tile) launch");
  } else if (spec) {
    CUDA_TRY(spec->ul(ctx, H, y, static_cast<int>(P), K, kappa, x_local, nullptr, st), "ul_detect launch");
  } else {
    const size_t smem = 4 * (static_cast<size_t>(Bc) + 2 * U) * sizeof(float2);
    const long long blocks = (P + 3) / 4;
    if (fmt == DCDG_FP16) {
      auto k = dcdg::ul_generic<__half2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      k<<<blocks, 128, smem, st>>>(static_cast<const __half2*>(H), static_cast<const __half2*>(y), static_cast<int>(P),
                                   Bc, U, K, kappa, static_cast<__half2*>(x_local), nullptr, nullptr);
    } else {
      auto k = dcdg::ul_generic<float2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      k<<<blocks, 128, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(y), static_cast<int>(P),
                                   Bc, U, K, kappa, static_cast<float2*>(x_local), nullptr, nullptr);
    }
    CUDA_TRY(cudaGetLastError(), "ul_generic launch");
  }
  ++ctx->launches;
  if (optimal && !gram && !ul_sig_shape(Bc, U, fmt))  // the Gram / fused kernels computed sigma^2 themselves
    if (int rc = launch_post_eq(ctx, H, static_cast<int>(P), Bc, U, n0, ex, fmt, sigma2, st)) return rc;
  if (xhat)
    if (int rc = launch_fuse(ctx, x_local, sigma2, S, C, C_total, U, fmt, optimal, xhat, wsum, st)) return rc;
  return DCDG_OK;
}

int dcdg_dl_precode(dcdg_ctx* ctx, const void* H, const void* s, int S, int C, int C_total, int Bc, int U, int K,
                    double rho, int fmt, void* x_dl, float* gain_part, float* gain, void* stream) {
  NvtxRange nvtx_("dcdg_dl_precode");
  if (int rc = check_fmt(fmt)) return rc;
  // precode.cpp:11-16,57-58,138-152,101-104
  if (C <= 0 || S < 0) return fail(DCDG_EINVAL, "decentralized_cd_precode: no clusters");
  if (C_total < C) return fail(DCDG_EINVAL, "dcdg_dl_precode: C_total must be >= C");
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "precoder: empty channel matrix");
  if (Bc < U)
    return fail(DCDG_EINVAL, "decentralized_cd_precode: cluster 0 has " + std::to_string(Bc) + " antennas for " +
                                 std::to_string(U) + " users; local zero-forcing needs B_c >= U");
  if (K <= 0) return fail(DCDG_EINVAL, "cd_precode: need at least one sweep");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  if (rho < 0.0 || std::isnan(rho)) return fail(DCDG_EINVAL, "power_scale: amplitude must be positive");
  if (gain && C != C_total) return fail(DCDG_EINVAL, "dcdg_dl_precode: effective gain needs every cluster (C == C_total)");
  if (!H || !s || !x_dl) return fail(DCDG_EINVAL, "dcdg_dl_precode: null buffer");
  const long long P = static_cast<long long>(S) * C;
  if (P > 0x7fffffffLL) return fail(DCDG_EINVAL, "dcdg_dl_precode: batch too large (S*C must fit in int32)");
  if (int rc = check_ctx(ctx)) return rc;  // after the device-independent argument checks
  if (P == 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);
  if (gain && !gain_part) {
    if (int rc = ensure_scratch(ctx, static_cast<size_t>(P) * sizeof(float))) return rc;
    gain_part = static_cast<float*>(ctx->scratch);
  }
  // rho == 0: return the raw cd_precode beamformer (no power_scale)
  const float rho_c = static_cast<float>(rho / std::sqrt(static_cast<double>(C_total)));
  const Spec* spec = find_spec(Bc, U, fmt);
  if (ctx->fp16_alg == DCDG_ALG_GRAM && gram_shape(Bc, U, fmt)) {
    if (int rc = launch_dl_gram(ctx, H, s, static_cast<int>(P), C, K, rho_c, x_dl, gain_part, st)) return rc;
  } else if (spec) {
    CUDA_TRY(spec->dl(ctx, H, s, static_cast<int>(P), C, K, rho_c, x_dl, gain_part, st), "dl_precode launch");
  } else {
    const size_t smem = 4 * (static_cast<size_t>(Bc) + 2 * U) * sizeof(float2);
    const long long blocks = (P + 3) / 4;
#define DL_GENERIC(T, GAIN)                                                                                     \
  {                                                                                                             \
    auto k = dcdg::dl_generic<T, GAIN>;                                                                         \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));               \
    k<<<blocks, 128, smem, st>>>(static_cast<const T*>(H), static_cast<const T*>(s), static_cast<int>(P), C, Bc, \
                                 U, K, rho_c, static_cast<T*>(x_dl), gain_part, ctx->d_status, nullptr);       \
  }
    if (fmt == DCDG_FP16) {
      if (gain_part) DL_GENERIC(__half2, true) else DL_GENERIC(__half2, false)
    } else {
      if (gain_part) DL_GENERIC(float2, true) else DL_GENERIC(float2, false)
    }
#undef DL_GENERIC
    CUDA_TRY(cudaGetLastError(), "dl_generic launch");
  }
  ++ctx->launches;
  if (gain) return dcdg_gain_reduce(ctx, gain_part, s, S, C, U, fmt, gain, stream);
  return DCDG_OK;
}

int dcdg_ul_trace(dcdg_ctx* ctx, const void* H, const void* y, int Bc, int U, int K, double n0, double ex, int fmt,
                  float* x_trace, float* r_trace, void* stream) {
  NvtxRange nvtx_("dcdg_ul_trace");
  if (int rc = check_fmt(fmt)) return rc;
  // cd_detect's checks (detect.cpp:12-19,71-72)
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "detector: empty channel matrix");
  if (n0 < 0.0 || !(ex > 0.0)) return fail(DCDG_EINVAL, "detector: need N0 >= 0 and E_x > 0");
  if (K <= 0) return fail(DCDG_EINVAL, "cd_detect: need at least one sweep");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  if (!H || !y || !x_trace || !r_trace) return fail(DCDG_EINVAL, "dcdg_ul_trace: null buffer");
  if (int rc = check_ctx(ctx)) return rc;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);
  const size_t xl_bytes = static_cast<size_t>(U) * 8;
  if (int rc = ensure_scratch(ctx, xl_bytes)) return rc;
  const size_t smem = 4 * (static_cast<size_t>(Bc) + 2 * U) * sizeof(float2);
  const float kappa = static_cast<float>(n0 / ex);
  auto* xt = reinterpret_cast<float2*>(x_trace);
  auto* rt = reinterpret_cast<float2*>(r_trace);
  if (fmt == DCDG_FP16) {
    auto k = dcdg::ul_generic<__half2, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<1, 128, smem, st>>>(static_cast<const __half2*>(H), static_cast<const __half2*>(y), 1, Bc, U, K, kappa,
                            static_cast<__half2*>(ctx->scratch), xt, rt);
  } else {
    auto k = dcdg::ul_generic<float2, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<1, 128, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(y), 1, Bc, U, K, kappa,
                            static_cast<float2*>(ctx->scratch), xt, rt);
  }
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "ul_trace launch");
  return DCDG_OK;
}

int dcdg_dl_trace(dcdg_ctx* ctx, const void* H, const void* s, int Bc, int U, int K, int fmt, float* x_trace,
                  void* stream) {
  NvtxRange nvtx_("dcdg_dl_trace");
  if (int rc = check_fmt(fmt)) return rc;
  // cd_precode's checks (precode.cpp:11-16,57-58)
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "precoder: empty channel matrix");
  if (K <= 0) return fail(DCDG_EINVAL, "cd_precode: need at least one sweep");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  if (!H || !s || !x_trace) return fail(DCDG_EINVAL, "dcdg_dl_trace: null buffer");
  if (int rc = check_ctx(ctx)) return rc;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);
  if (int rc = ensure_scratch(ctx, static_cast<size_t>(Bc) * 8)) return rc;
  const size_t smem = 4 * (static_cast<size_t>(Bc) + 2 * U) * sizeof(float2);
  auto* xt = reinterpret_cast<float2*>(x_trace);
  if (fmt == DCDG_FP16) {
    auto k = dcdg::dl_generic<__half2, false, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<1, 128, smem, st>>>(static_cast<const __half2*>(H), static_cast<const __half2*>(s), 1, 1, Bc, U, K, 0.f,
                            static_cast<__half2*>(ctx->scratch), nullptr, ctx->d_status, xt);
  } else {
    auto k = dcdg::dl_generic<float2, false, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<1, 128, smem, st>>>(static_cast<const float2*>(H), static_cast<const float2*>(s), 1, 1, Bc, U, K, 0.f,
                            static_cast<float2*>(ctx->scratch), nullptr, ctx->d_status, xt);
  }
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "dl_trace launch");
  return DCDG_OK;
}

int dcdg_post_eq_variance(dcdg_ctx* ctx, const void* H, int P, int Bc, int U, double n0, double ex, int fmt,
                          float* sigma2, void* stream) {
  NvtxRange nvtx_("dcdg_post_eq_variance");
  if (int rc = check_fmt(fmt)) return rc;
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "post_eq_variance: empty channel block");
  if (!(n0 > 0.0) || !(ex > 0.0)) return fail(DCDG_EINVAL, "post_eq_variance: need N0 > 0 and E_x > 0");
  if (U > 32) return fail(DCDG_EINVAL, "dcdg_post_eq_variance: U > 32 not supported");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  if (int rc = check_ctx(ctx)) return rc;  // after the device-independent argument checks
  if (P <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  return launch_post_eq(ctx, H, P, Bc, U, n0, ex, fmt, sigma2, as_stream(stream));
}

int dcdg_fuse(dcdg_ctx* ctx, const void* x_local, const float* sigma2, int S, int C, int C_total, int U, int fmt,
              int fusion, float* xhat, float* wsum, void* stream) {
  if (int rc = check_fmt(fmt)) return rc;
  if (C <= 0) return fail(DCDG_EINVAL, "fusion_weights: no clusters");
  if (C_total < C) return fail(DCDG_EINVAL, "dcdg_fuse: C_total must be >= C");
  const bool optimal = fusion == DCDG_FUSION_OPTIMAL;
  if (optimal && !sigma2) return fail(DCDG_EINVAL, "dcdg_fuse: optimal fusion needs sigma2");
  if (int rc = check_ctx(ctx)) return rc;  // after the device-independent argument checks
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  return launch_fuse(ctx, x_local, sigma2, S, C, C_total, U, fmt, optimal, xhat, wsum, as_stream(stream));
}

int dcdg_gain_part(dcdg_ctx* ctx, const void* H, const void* x_dl, const void* s, int S, int C, int Bc, int U, int fmt,
                   float* gain_part, void* stream) {
  if (int rc = check_fmt(fmt)) return rc;
  if (C <= 0 || S < 0 || Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "dcdg_gain_part: empty batch");
  if (!H || !x_dl || !s || !gain_part) return fail(DCDG_EINVAL, "dcdg_gain_part: null buffer");
  const long long P = static_cast<long long>(S) * C;
  if (P > 0x7fffffffLL) return fail(DCDG_EINVAL, "dcdg_gain_part: batch too large (S*C must fit in int32)");
  if (int rc = check_ctx(ctx)) return rc;
  if (P == 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const unsigned blocks = static_cast<unsigned>((P + 3) / 4);
  cudaStream_t st = as_stream(stream);
  if (fmt == DCDG_FP16)
    dcdg::gain_part_kernel<__half2><<<blocks, 128, 0, st>>>(static_cast<const __half2*>(H),
                                                            static_cast<const __half2*>(x_dl),
                                                            static_cast<const __half2*>(s), static_cast<int>(P), C, Bc,
                                                            U, gain_part);
  else
    dcdg::gain_part_kernel<float2><<<blocks, 128, 0, st>>>(static_cast<const float2*>(H),
                                                           static_cast<const float2*>(x_dl),
                                                           static_cast<const float2*>(s), static_cast<int>(P), C, Bc, U,
                                                           gain_part);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "gain_part launch");
  return DCDG_OK;
}

int dcdg_fuse_finalize(dcdg_ctx* ctx, float* xhat, const float* wsum, int S, int U, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const long long n = static_cast<long long>(S) * U;
  dcdg::fuse_finalize_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(reinterpret_cast<float2*>(xhat), wsum, S,
                                                                              U);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "fuse_finalize launch");
  return DCDG_OK;
}

int dcdg_gain_reduce(dcdg_ctx* ctx, const float* gain_part, const void* s, int S, int C, int U, int fmt, float* gain,
                     void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_fmt(fmt)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const unsigned blocks = static_cast<unsigned>((S + dcdg::kGainSubs - 1) / dcdg::kGainSubs);
  const size_t smem = dcdg::gain_reduce_smem(U, C);
  if (smem > 227 * 1024) return fail(DCDG_EINVAL, "dcdg_gain_reduce: U or C too large");
  if (fmt == DCDG_FP16) {
    auto k = dcdg::gain_reduce_kernel<__half2>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    CUDA_TRY(launch_dependent(k, blocks, 128, smem, as_stream(stream), gain_part, static_cast<const __half2*>(s), S, C,
                              U, gain),
             "gain_reduce launch");
  } else {
    auto k = dcdg::gain_reduce_kernel<float2>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    CUDA_TRY(launch_dependent(k, blocks, 128, smem, as_stream(stream), gain_part, static_cast<const float2*>(s), S, C,
                              U, gain),
             "gain_reduce launch");
  }
  ++ctx->launches;
  return DCDG_OK;
}

int dcdg_power_scale(dcdg_ctx* ctx, void* x, int P, int n, double rho, int fmt, void* stream) {
  if (int rc = check_fmt(fmt)) return rc;
  if (!(rho > 0.0)) return fail(DCDG_EINVAL, "power_scale: amplitude must be positive");
  if (n <= 0) return fail(DCDG_EINVAL, "power_scale: empty beamformer");
  if (int rc = check_ctx(ctx)) return rc;  // after the device-independent argument checks
  if (P <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int blocks = (P + 3) / 4;
  if (fmt == DCDG_FP16)
    dcdg::power_scale_kernel<__half2><<<blocks, 128, 0, as_stream(stream)>>>(static_cast<__half2*>(x), P, n,
                                                                             static_cast<float>(rho), ctx->d_status);
  else
    dcdg::power_scale_kernel<float2><<<blocks, 128, 0, as_stream(stream)>>>(static_cast<float2*>(x), P, n,
                                                                            static_cast<float>(rho), ctx->d_status);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "power_scale launch");
  return DCDG_OK;
}

int dcdg_fusion_weights(dcdg_ctx* ctx, const float* sigma2, int S, int C, float* w, void* stream) {
  if (C <= 0) return fail(DCDG_EINVAL, "fusion_weights: no clusters");
  if (int rc = check_ctx(ctx)) return rc;  // after the device-independent argument checks
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  dcdg::fusion_weights_kernel<<<(S + 127) / 128, 128, 0, as_stream(stream)>>>(sigma2, S, C, w, ctx->d_status);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "fusion_weights launch");
  return DCDG_OK;
}

namespace {
int check_qam(int qam, double ex) {
  if (qam != 4 && qam != 16 && qam != 64) return fail(DCDG_EINVAL, "Constellation::qam: order must be 4, 16 or 64");
  if (!(ex > 0.0)) return fail(DCDG_EINVAL, "Constellation::qam: symbol energy must be positive");
  return DCDG_OK;
}
int bps_of(int qam) { return qam == 4 ? 2 : qam == 16 ? 4 : 6; }
}  // namespace

int dcdg_mmse_bias(dcdg_ctx* ctx, const void* H, int S, int C, int Bc, int U, double n0, double ex, int fmt,
                   float* beta, void* stream) {
  if (int rc = check_fmt(fmt)) return rc;
  if (C <= 0 || Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "detector: empty channel matrix");
  if (n0 < 0.0 || !(ex > 0.0)) return fail(DCDG_EINVAL, "detector: need N0 >= 0 and E_x > 0");
  if (U > 32) return fail(DCDG_EINVAL, "dcdg_mmse_bias: U > 32 not supported");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  if (int rc = check_ctx(ctx)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);
  const double kappa = n0 / ex;
  if (kappa == 0.0) {  // detect.cpp:232: no shrinkage
    const long long n = static_cast<long long>(S) * U;
    dcdg::fill_kernel<<<static_cast<int>(std::min<long long>((n + 255) / 256, 2368)), 256, 0, st>>>(beta, n, 1.f);
    ++ctx->launches;
    CUDA_TRY(cudaGetLastError(), "fill launch");
    return DCDG_OK;
  }
  return launch_gram_chol<dcdg::kBias>(ctx, H, S, C, Bc, U, static_cast<float>(kappa), 1.f, 0.f, fmt, beta, st);
}

int dcdg_slice(dcdg_ctx* ctx, const void* x, int fmt, const float* beta, int64_t n, int qam, double ex,
               uint8_t* labels, void* stream) {
  if (int rc = check_fmt(fmt)) return rc;
  if (int rc = check_qam(qam, ex)) return rc;
  if (int rc = check_ctx(ctx)) return rc;
  if (n <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
  if (fmt == DCDG_FP16)
    dcdg::slice_kernel<__half2><<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const __half2*>(x), beta, n, qam,
                                                                       ex, labels);
  else
    dcdg::slice_kernel<float2><<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const float2*>(x), beta, n, qam, ex,
                                                                      labels);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "slice launch");
  return DCDG_OK;
}

int dcdg_bit_errors(dcdg_ctx* ctx, const uint8_t* labels, const uint8_t* bits, int64_t n, int qam,
                    unsigned long long* errors, void* stream) {
  if (int rc = check_qam(qam, 1.0)) return rc;
  if (int rc = check_ctx(ctx)) return rc;
  if (n <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 8));
  dcdg::bit_errors_kernel<<<blocks, 256, 0, as_stream(stream)>>>(labels, bits, n, bps_of(qam), errors);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "bit_errors launch");
  return DCDG_OK;
}

int dcdg_dl_receive(dcdg_ctx* ctx, const void* H, const void* x_dl, const void* s, const float* noise, int S, int C,
                    int Bc, int U, int fmt, int qam, double ex, uint8_t* labels, float* beta, uint8_t* flagged,
                    void* stream) {
  if (int rc = check_fmt(fmt)) return rc;
  if (int rc = check_qam(qam, ex)) return rc;
  if (C <= 0 || Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "precoder: empty channel matrix");
  if (U > 32) return fail(DCDG_EINVAL, "dcdg_dl_receive: U > 32 not supported");
  if (int rc = check_ctx(ctx)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int blocks = (S + 3) / 4;
  if (fmt == DCDG_FP16)
    dcdg::dl_receive_kernel<__half2><<<blocks, 128, 0, as_stream(stream)>>>(
        static_cast<const __half2*>(H), static_cast<const __half2*>(x_dl), static_cast<const __half2*>(s),
        reinterpret_cast<const float2*>(noise), S, C, Bc, U, qam, ex, labels, beta, flagged);
  else
    dcdg::dl_receive_kernel<float2><<<blocks, 128, 0, as_stream(stream)>>>(
        static_cast<const float2*>(H), static_cast<const float2*>(x_dl), static_cast<const float2*>(s),
        reinterpret_cast<const float2*>(noise), S, C, Bc, U, qam, ex, labels, beta, flagged);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "dl_receive launch");
  return DCDG_OK;
}

int dcdg_round_fp16(dcdg_ctx* ctx, float* x, int64_t n, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (n <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
  dcdg::round_fp16_kernel<<<blocks, 256, 0, as_stream(stream)>>>(x, n);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "round_fp16 launch");
  return DCDG_OK;
}

int dcdg_convert(dcdg_ctx* ctx, const void* src, int src_fmt, void* dst, int dst_fmt, int64_t n_complex,
                 void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  auto ok = [](int f) { return f == DCDG_FP32 || f == DCDG_FP16 || f == DCDG_FP16_PAIRS; };
  if (!ok(src_fmt) || !ok(dst_fmt)) return fail(DCDG_EINVAL, "dcdg: unknown storage format");
  if (n_complex <= 0) return DCDG_OK;
  if ((src_fmt == DCDG_FP16_PAIRS || dst_fmt == DCDG_FP16_PAIRS) && (n_complex & 1))
    return fail(DCDG_EINVAL, "dcdg_convert: row-pair planar fp16 needs an even element count");
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);
  const long long n = 2 * n_complex;
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
  if (src_fmt == dst_fmt) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, static_cast<size_t>(n_complex) * esize(src_fmt == DCDG_FP32 ? DCDG_FP32 : DCDG_FP16),
                             cudaMemcpyDeviceToDevice, st),
             "convert copy");
    return DCDG_OK;
  }
  if (src_fmt == DCDG_FP32 && dst_fmt == DCDG_FP16)
    dcdg::f32_to_f16_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(src), static_cast<__half*>(dst), n);
  else if (src_fmt == DCDG_FP16 && dst_fmt == DCDG_FP32)
    dcdg::f16_to_f32_kernel<<<blocks, 256, 0, st>>>(static_cast<const __half*>(src), static_cast<float*>(dst), n);
  else if (src_fmt == DCDG_FP32 && dst_fmt == DCDG_FP16_PAIRS)
    dcdg::f32_to_f16_pairs_kernel<<<blocks, 256, 0, st>>>(static_cast<const float4*>(src), static_cast<uint2*>(dst),
                                                          n_complex / 2);
  else if (src_fmt == DCDG_FP16_PAIRS && dst_fmt == DCDG_FP32)
    dcdg::f16_pairs_to_f32_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint2*>(src), static_cast<float4*>(dst),
                                                          n_complex / 2);
  else
    return fail(DCDG_EINVAL, "dcdg_convert: unsupported conversion (go through DCDG_FP32)");
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "convert launch");
  return DCDG_OK;
}

// ---------------------------------------------------------------------------
// BER-sweep building blocks
// ---------------------------------------------------------------------------
int dcdg_synth(dcdg_ctx* ctx, int S, int C, int Bc, int U, int qam, double ex, double n0, uint64_t seed,
               uint64_t first_trial, void* H, void* y, uint8_t* bits, void* sym, void* noise_dl, void* stream) {
  if (C <= 0 || Bc <= 0) return fail(DCDG_EINVAL, "make_batch: empty layout");
  if (U <= 0 || static_cast<long long>(C) * Bc < U) return fail(DCDG_EINVAL, "make_batch: need B >= U >= 1");
  if (int rc = check_qam(qam, ex)) return rc;
  if (n0 < 0.0) return fail(DCDG_EINVAL, "awgn: noise power must be nonnegative");
  if (!H || !bits) return fail(DCDG_EINVAL, "dcdg_synth: null buffer");
  if (int rc = check_ctx(ctx)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const long long n = static_cast<long long>(S) * C * Bc;
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, static_cast<long long>(ctx->sms) * 8));
  dcdg::synth_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      S, C, Bc, U, seed, first_trial, static_cast<float>(n0), static_cast<unsigned>(qam), ex, static_cast<float2*>(H),
      static_cast<float2*>(y), bits, static_cast<float2*>(sym), static_cast<float2*>(noise_dl));
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "synth launch");
  return DCDG_OK;
}

int dcdg_mf_detect(dcdg_ctx* ctx, const void* H, const void* y, int S, int C, int Bc, int U, float* xhat,
                   void* stream) {
  if (C <= 0) return fail(DCDG_EINVAL, "mf_detect: no clusters");
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "detector: empty channel matrix");
  if (U > 32) return fail(DCDG_EINVAL, "dcdg_mf_detect: U > 32 not supported");
  if (!H || !y || !xhat) return fail(DCDG_EINVAL, "dcdg_mf_detect: null buffer");
  if (int rc = check_ctx(ctx)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  dcdg::mf_detect_kernel<<<(S + 3) / 4, 128, 0, as_stream(stream)>>>(
      static_cast<const float2*>(H), static_cast<const float2*>(y), S, C, Bc, U, reinterpret_cast<float2*>(xhat),
      ctx->d_status);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "mf_detect launch");
  return DCDG_OK;
}

int dcdg_mf_precode(dcdg_ctx* ctx, const void* H, const void* s, int S, int C, int Bc, int U, double rho,
                    float* x_dl, void* stream) {
  if (C <= 0) return fail(DCDG_EINVAL, "mf_precode: no clusters");
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "precoder: empty channel matrix");
  if (!(rho > 0.0)) return fail(DCDG_EINVAL, "power_scale: amplitude must be positive");
  if (!H || !s || !x_dl) return fail(DCDG_EINVAL, "dcdg_mf_precode: null buffer");
  if (int rc = check_ctx(ctx)) return rc;
  const long long P = static_cast<long long>(S) * C;
  if (P <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  const float rho_c = static_cast<float>(rho / std::sqrt(static_cast<double>(C)));
  dcdg::mf_precode_kernel<<<static_cast<int>((P + 3) / 4), 128, 0, as_stream(stream)>>>(
      static_cast<const float2*>(H), static_cast<const float2*>(s), static_cast<int>(P), C, Bc, U, rho_c,
      reinterpret_cast<float2*>(x_dl), ctx->d_status);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "mf_precode launch");
  return DCDG_OK;
}

int dcdg_lmmse_exact(dcdg_ctx* ctx, const void* H, const void* y, int S, int C, int Bc, int U, double n0,
                     double ex, float* xhat, void* stream) {
  if (C <= 0 || Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "detector: empty channel matrix");
  if (n0 < 0.0 || !(ex > 0.0)) return fail(DCDG_EINVAL, "detector: need N0 >= 0 and E_x > 0");
  if (U > 32) return fail(DCDG_EINVAL, "dcdg_lmmse_exact: U > 32 not supported");
  if (!H || !y || !xhat) return fail(DCDG_EINVAL, "dcdg_lmmse_exact: null buffer");
  if (int rc = check_ctx(ctx)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  return launch_solve<dcdg::kSolve>(ctx, H, y, S, C, Bc, U, static_cast<float>(n0 / ex), 0.f,
                                    reinterpret_cast<float2*>(xhat), as_stream(stream));
}

int dcdg_zf_exact(dcdg_ctx* ctx, const void* H, const void* s, int S, int C, int Bc, int U, double rho,
                  float* x_dl, void* stream) {
  if (C <= 0 || Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "precoder: empty channel matrix");
  if (rho < 0.0 || std::isnan(rho)) return fail(DCDG_EINVAL, "power_scale: amplitude must be positive");
  if (U > 32) return fail(DCDG_EINVAL, "dcdg_zf_exact: U > 32 not supported");
  if (!H || !s || !x_dl) return fail(DCDG_EINVAL, "dcdg_zf_exact: null buffer");
  if (int rc = check_ctx(ctx)) return rc;
  if (S <= 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  return launch_solve<dcdg::kZf>(ctx, H, s, S, C, Bc, U, 0.f, static_cast<float>(rho),
                                 reinterpret_cast<float2*>(x_dl), as_stream(stream));
}

/* ---- fused cross-GPU exchange over peer memory ---------------------------- */
int dcdg_xwin_create(dcdg_ctx* ctx, int world, int rank, int64_t buf_bytes, dcdg_xwin** out) {
  if (!out) return fail(DCDG_EINVAL, "dcdg_xwin_create: null output");
  *out = nullptr;
  if (world < 1 || world > dcdg::kXchgMaxRanks || rank < 0 || rank >= world)
    return fail(DCDG_EINVAL, "dcdg_xwin_create: need 1 <= world <= 8 and 0 <= rank < world");
  if (buf_bytes <= 0) return fail(DCDG_EINVAL, "dcdg_xwin_create: empty window");
  if (int rc = check_ctx(ctx)) return rc;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  auto* w = new dcdg_xwin;
  w->ctx = ctx;
  w->world = world;
  w->rank = rank;
  w->buf_bytes = (buf_bytes + 255) & ~int64_t(255);
  const size_t total = dcdg::kXchgFlagBytes + 2 * static_cast<size_t>(w->buf_bytes);
  cudaError_t e = cudaMalloc(&w->base, total);
  if (e == cudaSuccess) e = cudaMemset(w->base, 0, dcdg::kXchgFlagBytes);
  if (e == cudaSuccess) e = cudaMalloc(&w->counter, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(w->counter, 0, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&w->d_epoch, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(w->d_epoch, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (w->base) cudaFree(w->base);
    if (w->counter) cudaFree(w->counter);
    if (w->d_epoch) cudaFree(w->d_epoch);
    delete w;
    return cuda_fail(e, "dcdg_xwin_create");
  }
  w->peer[rank] = w->base;
  w->opened[rank] = true;
  *out = w;
  return DCDG_OK;
}

int dcdg_xwin_handle(dcdg_xwin* w, void* handle) {
  if (!w || !handle) return fail(DCDG_EINVAL, "dcdg_xwin_handle: null argument");
  CUDA_TRY(cudaSetDevice(w->ctx->device), "cudaSetDevice");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, w->base), "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == DCDG_XWIN_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof h);
  return DCDG_OK;
}

int dcdg_xwin_open(dcdg_xwin* w, int peer, const void* handle) {
  if (!w || !handle) return fail(DCDG_EINVAL, "dcdg_xwin_open: null argument");
  if (peer < 0 || peer >= w->world) return fail(DCDG_EINVAL, "dcdg_xwin_open: peer out of range");
  if (peer == w->rank || w->opened[peer]) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(w->ctx->device), "cudaSetDevice");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  w->peer[peer] = static_cast<unsigned char*>(p);
  w->opened[peer] = true;
  return DCDG_OK;
}

int dcdg_xwin_set_timeout(dcdg_xwin* w, int64_t timeout_ns) {
  if (!w || timeout_ns <= 0) return fail(DCDG_EINVAL, "dcdg_xwin_set_timeout: need a window and a positive timeout");
  w->timeout_ns = timeout_ns;
  return DCDG_OK;
}

int dcdg_xwin_destroy(dcdg_xwin* w) {
  if (!w) return DCDG_OK;
  cudaSetDevice(w->ctx->device);
  cudaDeviceSynchronize();
  for (int q = 0; q < w->world; ++q)
    if (q != w->rank && w->opened[q] && w->peer[q]) cudaIpcCloseMemHandle(w->peer[q]);
  if (w->base) cudaFree(w->base);
  if (w->counter) cudaFree(w->counter);
  if (w->d_epoch) cudaFree(w->d_epoch);
  delete w;
  return DCDG_OK;
}

int dcdg_ul_detect_xchg(dcdg_ctx* ctx, dcdg_xwin* w, const void* H, const void* y, int S, int C, int c0,
                        int C_total, int Bc, int U, int K, double n0, double ex, int fmt, int fusion, float* xhat,
                        void* stream) {
  NvtxRange nvtx_("dcdg_ul_detect_xchg");
  if (int rc = check_fmt(fmt)) return rc;
  // the reference's argument checks first (as dcdg_ul_detect), then the exchange's own
  if (C <= 0 || S < 0) return fail(DCDG_EINVAL, "decentralized_cd_detect: no clusters");
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "detector: empty channel matrix");
  if (n0 < 0.0 || !(ex > 0.0)) return fail(DCDG_EINVAL, "detector: need N0 >= 0 and E_x > 0");
  if (K <= 0) return fail(DCDG_EINVAL, "cd_detect: need at least one sweep");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  const bool optimal = fusion == DCDG_FUSION_OPTIMAL;
  if (fusion != DCDG_FUSION_OPTIMAL && fusion != DCDG_FUSION_UNIFORM)
    return fail(DCDG_EINVAL, "dcdg_ul_detect: unknown fusion mode");
  if (optimal && !(n0 > 0.0)) return fail(DCDG_EINVAL, "post_eq_variance: need N0 > 0 and E_x > 0");
  if (optimal && U > 32) return fail(DCDG_EINVAL, "dcdg_post_eq_variance: U > 32 not supported");
  if (!w) return fail(DCDG_EINVAL, "dcdg_ul_detect_xchg: null exchange window");
  if (c0 < 0 || c0 + C > C_total) return fail(DCDG_EINVAL, "dcdg_ul_detect_xchg: clusters [c0, c0+C) outside C_total");
  if (S % w->world) return fail(DCDG_EINVAL, "dcdg_ul_detect_xchg: S must divide over the ranks");
  for (int q = 0; q < w->world; ++q)
    if (!w->opened[q]) return fail(DCDG_EINVAL, "dcdg_ul_detect_xchg: peer window " + std::to_string(q) + " not open");
  const int S_own = S / w->world;
  const long long xbytes = static_cast<long long>(S_own) * C_total * U * static_cast<long long>(esize(fmt));
  const long long sig_off = (xbytes + 255) & ~255LL;
  const long long need = sig_off + (optimal ? static_cast<long long>(S_own) * C_total * 4 : 0);
  if (need > w->buf_bytes) return fail(DCDG_EINVAL, "dcdg_ul_detect_xchg: exchange window too small for this batch");
  if (!H || !y || !xhat) return fail(DCDG_EINVAL, "dcdg_ul_detect_xchg: null buffer");
  const long long P = static_cast<long long>(S) * C;
  if (P > 0x7fffffffLL) return fail(DCDG_EINVAL, "dcdg_ul_detect: batch too large (S*C must fit in int32)");
  if (int rc = check_ctx(ctx)) return rc;
  if (P == 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);

  dcdg::XMap m{};
  for (int q = 0; q < w->world; ++q) m.win[q] = w->peer[q];
  m.counter = w->counter;
  m.epoch_dev = w->d_epoch;
  m.flag_slot = 0;  // uplink: rank q publishes to slot q
  m.per_rank = 1;
  m.buf_bytes = w->buf_bytes;
  m.sig_off = sig_off;
  m.world = w->world;
  m.rank = w->rank;
  m.S_own = S_own;
  m.C_local = C;
  m.c0 = c0;
  m.C_total = C_total;
  m.U = U;
  m.esz = static_cast<int>(esize(fmt));
  dcdg::xchg_advance_kernel<<<1, 1, 0, st>>>(w->d_epoch);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "xchg_advance launch");

  const float kappa = static_cast<float>(n0 / ex);
  const Spec* spec = find_spec(Bc, U, fmt);
  const bool gram = ctx->fp16_alg == DCDG_ALG_GRAM && gram_shape(Bc, U, fmt);  // no exchange epilogue
  if (spec && spec->ulk.kind == kReg && !optimal && !gram) {
    // fused: the CD kernel stores into the owners' windows and signals
    CUDA_TRY(spec->ul(ctx, H, y, static_cast<int>(P), K, kappa, nullptr, &m, st), "ul_detect_xchg launch");
    ++ctx->launches;
  } else {
    // CD (+ variances) locally, then one put kernel moves the rows and signals
    const size_t xl_bytes = static_cast<size_t>(P) * U * esize(fmt);
    const size_t s2_off = (xl_bytes + 255) & ~size_t(255);
    if (int rc = ensure_scratch(ctx, s2_off + (optimal ? static_cast<size_t>(P) * 4 : 0))) return rc;
    void* xl = ctx->scratch;
    float* s2 = optimal ? reinterpret_cast<float*>(static_cast<unsigned char*>(ctx->scratch) + s2_off) : nullptr;
    if (int rc = dcdg_ul_detect(ctx, H, y, S, C, C_total, Bc, U, K, n0, ex, fmt, fusion, xl, s2, nullptr, nullptr,
                                stream))
      return rc;
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<long long>((P * U + P + threads - 1) / threads, 4LL * ctx->sms));
    if (fmt == DCDG_FP16)
      dcdg::xchg_put_kernel<__half2><<<blocks, threads, 0, st>>>(static_cast<const __half2*>(xl), s2, P, m);
    else
      dcdg::xchg_put_kernel<float2><<<blocks, threads, 0, st>>>(static_cast<const float2*>(xl), s2, P, m);
    ++ctx->launches;
    CUDA_TRY(cudaGetLastError(), "xchg_put launch");
  }
  // owner side: wait for every rank's epoch, then the ascending-cluster fusion
  const long long n = static_cast<long long>(S_own) * U;
  const int threads = 256;
  const long long blocks = std::max(1LL, std::min<long long>((n + threads - 1) / threads, 2LL * ctx->sms));
#define XFUSE(T)                                                                                               \
  dcdg::xchg_fuse_kernel<T><<<blocks, threads, 0, st>>>(w->base, w->d_epoch, w->world, w->buf_bytes,           \
                                                        sig_off, S_own, C_total, U, optimal, w->timeout_ns,     \
                                                        reinterpret_cast<float2*>(xhat), ctx->d_status)
  if (fmt == DCDG_FP16)
    XFUSE(__half2);
  else
    XFUSE(float2);
#undef XFUSE
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "xchg_fuse launch");
  return DCDG_OK;
}

int dcdg_dl_precode_xchg(dcdg_ctx* ctx, dcdg_xwin* w, int root, const void* H, const void* s, int S, int C, int c0,
                         int C_total, int Bc, int U, int K, double rho, int fmt, void* x_dl, float* gain,
                         void* stream) {
  NvtxRange nvtx_("dcdg_dl_precode_xchg");
  if (int rc = check_fmt(fmt)) return rc;
  // the reference's checks (as dcdg_dl_precode), then the exchange's own
  if (C <= 0 || S < 0) return fail(DCDG_EINVAL, "decentralized_cd_precode: no clusters");
  if (Bc <= 0 || U <= 0) return fail(DCDG_EINVAL, "precoder: empty channel matrix");
  if (Bc < U)
    return fail(DCDG_EINVAL, "decentralized_cd_precode: cluster " + std::to_string(c0) + " has " +
                                 std::to_string(Bc) + " antennas for " + std::to_string(U) +
                                 " users; local zero-forcing needs B_c >= U");
  if (K <= 0) return fail(DCDG_EINVAL, "cd_precode: need at least one sweep");
  if (fmt == DCDG_FP16 && (Bc & 1))
    return fail(DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c");
  if (rho < 0.0 || std::isnan(rho)) return fail(DCDG_EINVAL, "power_scale: amplitude must be positive");
  if (!w) return fail(DCDG_EINVAL, "dcdg_dl_precode_xchg: null exchange window");
  if (root < 0 || root >= w->world) return fail(DCDG_EINVAL, "dcdg_dl_precode_xchg: root out of range");
  if (c0 < 0 || c0 + C > C_total) return fail(DCDG_EINVAL, "dcdg_dl_precode_xchg: clusters [c0, c0+C) outside C_total");
  for (int q = 0; q < w->world; ++q)
    if (!w->opened[q]) return fail(DCDG_EINVAL, "dcdg_dl_precode_xchg: peer window " + std::to_string(q) + " not open");
  const long long sbytes = static_cast<long long>(S) * U * static_cast<long long>(esize(fmt));
  const long long gain_off = (sbytes + 255) & ~255LL;
  if (gain_off + static_cast<long long>(S) * C_total * 4 > w->buf_bytes)
    return fail(DCDG_EINVAL, "dcdg_dl_precode_xchg: exchange window too small for this batch");
  if (!H || !x_dl || (w->rank == root && !s)) return fail(DCDG_EINVAL, "dcdg_dl_precode_xchg: null buffer");
  const long long P = static_cast<long long>(S) * C;
  if (P > 0x7fffffffLL) return fail(DCDG_EINVAL, "dcdg_dl_precode: batch too large (S*C must fit in int32)");
  if (int rc = check_ctx(ctx)) return rc;
  if (P == 0) return DCDG_OK;
  CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = as_stream(stream);

  dcdg::XMap m{};
  for (int q = 0; q < w->world; ++q) m.win[q] = w->peer[q];
  m.counter = w->counter;
  m.epoch_dev = w->d_epoch;
  m.buf_bytes = w->buf_bytes;
  m.sig_off = gain_off;
  m.world = w->world;
  m.rank = w->rank;
  m.C_local = C;
  m.c0 = c0;
  m.C_total = C_total;
  m.U = U;
  m.esz = static_cast<int>(esize(fmt));
  const int threads = 256;
  dcdg::xchg_advance_kernel<<<1, 1, 0, st>>>(w->d_epoch);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "xchg_advance launch");
  // 1. root: the centre -> cluster symbol broadcast as stores into every window
  if (w->rank == root) {
    m.flag_slot = dcdg::kSlotSymbols;
    m.per_rank = 0;
    const long long n = static_cast<long long>(S) * U;
    const int blocks = static_cast<int>(std::max(1LL, std::min<long long>((n + threads - 1) / threads, 4LL * ctx->sms)));
    if (fmt == DCDG_FP16)
      dcdg::xchg_symbols_push_kernel<__half2><<<blocks, threads, 0, st>>>(static_cast<const __half2*>(s), n, m);
    else
      dcdg::xchg_symbols_push_kernel<float2><<<blocks, threads, 0, st>>>(static_cast<const float2*>(s), n, m);
    ++ctx->launches;
    CUDA_TRY(cudaGetLastError(), "xchg_symbols_push launch");
  }
  // 2. every rank: wait for the symbols, precode from its own window
  dcdg::xchg_wait_kernel<<<1, 32, 0, st>>>(w->base, dcdg::kSlotSymbols, 1, w->d_epoch, w->timeout_ns, ctx->d_status);
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "xchg_wait launch");
  const size_t gp_bytes = (static_cast<size_t>(P) * sizeof(float) + 255) & ~size_t(255);
  const size_t sy_bytes = (static_cast<size_t>(sbytes) + 15) & ~size_t(15);
  if (int rc = ensure_scratch(ctx, gp_bytes + sy_bytes)) return rc;
  float* gp = static_cast<float*>(ctx->scratch);
  void* Sy = static_cast<unsigned char*>(ctx->scratch) + gp_bytes;
  {
    const long long n16 = static_cast<long long>(sy_bytes / 16);
    const int blocks = static_cast<int>(std::max(1LL, std::min<long long>((n16 + threads - 1) / threads, 4LL * ctx->sms)));
    dcdg::xchg_symbols_fetch_kernel<<<blocks, threads, 0, st>>>(w->base, w->d_epoch, w->buf_bytes, n16,
                                                                  static_cast<uint4*>(Sy));
    ++ctx->launches;
    CUDA_TRY(cudaGetLastError(), "xchg_symbols_fetch launch");
  }
  if (int rc = dcdg_dl_precode(ctx, H, Sy, S, C, C_total, Bc, U, K, rho, fmt, x_dl, gp, nullptr, stream)) return rc;
  // 3. gain shares into every window, then the ascending-cluster effective gain.
  //    (Always run: the gain exchange is also the acknowledgement that lets the
  //    root reuse this parity's symbol buffer two calls later.)
  m.flag_slot = dcdg::kSlotGain;
  m.per_rank = 1;
  {
    const int blocks = static_cast<int>(std::max(1LL, std::min<long long>((P + threads - 1) / threads, 4LL * ctx->sms)));
    dcdg::xchg_gain_put_kernel<<<blocks, threads, 0, st>>>(gp, P, m);
    ++ctx->launches;
    CUDA_TRY(cudaGetLastError(), "xchg_gain_put launch");
  }
  const int gblocks = gain ? std::max(1, std::min((S + threads - 1) / threads, 2 * ctx->sms)) : 1;
#define XGAIN(T)                                                                                                \
  dcdg::xchg_gain_fuse_kernel<T><<<gblocks, threads, 0, st>>>(w->base, w->d_epoch, w->world, w->buf_bytes,      \
                                                              gain_off, S, C_total, U, w->timeout_ns, gain,      \
                                                              ctx->d_status)
  if (fmt == DCDG_FP16)
    XGAIN(__half2);
  else
    XGAIN(float2);
#undef XGAIN
  ++ctx->launches;
  CUDA_TRY(cudaGetLastError(), "xchg_gain_fuse launch");
  return DCDG_OK;
}

}  // extern "C"
