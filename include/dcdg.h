/*
 * dcdg.h — C ABI of the B200-native decentralized coordinate-descent (CD)
 * baseband: per-cluster L-MMSE uplink detection (Alg. 1) with feed-forward
 * fusion, and per-cluster ZF downlink precoding (Alg. 2) with the rho/sqrt(C)
 * power split, batched over thousands of (subcarrier, cluster) problems.
 *
 * Plain pointers and sizes only — no torch, no C++ types.  This is the
 * boundary a host binding (C++ wrapper include/dcd_gpu.hpp, ctypes, cgo, …)
 * calls; INTEGRATION.md shows the bindings.  Reference interfaces replaced
 * (paths relative to /root/reference/proj):
 *
 *   dcdg_ul_detect     <- dcd::decentralized_cd_detect  include/dcd/detect.hpp:84-86
 *                         (per cluster dcd::cd_detect   include/dcd/detect.hpp:60-63,
 *                          dcd::post_eq_variance        detect.hpp:67,
 *                          dcd::fusion_weights          detect.hpp:70)
 *   dcdg_dl_precode    <- dcd::decentralized_cd_precode include/dcd/precode.hpp:72-75
 *                         (per cluster dcd::cd_precode  precode.hpp:58-60,
 *                          dcd::power_scale             precode.hpp:63)
 *   dcdg_fuse          <- the ascending-cluster fusion sum, src/detect.cpp:180-187
 *   dcdg_post_eq_variance <- dcd::post_eq_variance      src/detect.cpp:112-130
 *   dcdg_gain_reduce   <- assemble_blocks' effective_gain, src/precode.cpp:123-131
 *
 * The reference's kernels::Backend table (include/dcd/kernels.hpp:34-46) is a
 * per-vector (n = B_c) plugin point far too fine-grained for a GPU; this ABI
 * plugs in one level up, at the batched decentralized calls.
 *
 * DEVICE BATCH LAYOUT (all pointers are device pointers):
 *   problem p = s*C + c  (subcarrier s, local cluster c; subcarrier-major)
 *   H   [P][U][B_c]  complex; each tile is the cluster's B_c x U UPLINK block,
 *                    column-major exactly like dcd::ComplexMatrix
 *                    (numerics.hpp:35-40).  The downlink uses the same tiles:
 *                    conj_rows(H_dl)[u] is uplink column u (precode.cpp:19-27).
 *   y   [P][B_c]     uplink receive samples of each cluster
 *   s   [S][U]       downlink symbols (one vector per subcarrier, broadcast)
 *   x_local [P][U]   per-cluster uplink estimates (the wire payload)
 *   xhat [S][U]      fused uplink estimate (always complex fp32)
 *   x_dl [P][B_c]    per-cluster beamformers, already power-scaled
 * "complex" is interleaved (re, im): float2 for DCDG_FP32, two IEEE binary16
 * for DCDG_FP16 (the paper's half-precision path) — except the DCDG_FP16
 * channel tiles H and receive vectors y, which are stored ROW-PAIR PLANAR:
 * rows (2i, 2i+1) of a column/vector occupy 8 bytes as
 * {re_2i, re_2i+1, im_2i, im_2i+1}, so the half2 kernels load planar half2
 * pairs directly (B_c must be even; dcdg_convert(..., DCDG_FP16_PAIRS, ...)
 * produces this layout from complex fp32).  Buffers must be 16-byte aligned.
 *
 * Errors: every call returns a dcdg_status.  Argument errors are detected on
 * the host before any launch and carry the reference's exception text
 * (dcdg_last_error).  Numerical errors that the reference throws from inside
 * a cluster worker (all-zero channel row, zero beamformer, singular Gram) are
 * recorded on the device per batch; dcdg_sync_status() waits for the stream
 * and returns them with the reference's text.  There is no CPU fallback: with
 * no usable CUDA device every call returns DCDG_ECUDA.
 */
#ifndef DCDG_H
#define DCDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DCDG_ABI_VERSION 1

typedef enum {
  DCDG_OK = 0,
  DCDG_EINVAL = 1,   /* std::invalid_argument in the reference */
  DCDG_ENUMERIC = 2, /* std::runtime_error in the reference     */
  DCDG_ECUDA = 3,
  DCDG_ENCCL = 4
} dcdg_status;

typedef enum { DCDG_FP32 = 0, DCDG_FP16 = 1, DCDG_FP16_PAIRS = 2 /* conversion only */ } dcdg_format;
typedef enum { DCDG_FUSION_OPTIMAL = 0, DCDG_FUSION_UNIFORM = 1 } dcdg_fusion; /* detect.hpp:24 */

typedef struct dcdg_ctx dcdg_ctx;

int dcdg_abi_version(void);
/* Number of visible CUDA devices (0 when none). */
int dcdg_device_count(void);
/* Create a context bound to `device`; *out receives it. */
int dcdg_init(int device, dcdg_ctx** out);
int dcdg_destroy(dcdg_ctx* ctx);
/* Text of the last error raised on this thread (reference wording). */
const char* dcdg_last_error(void);
/* Streams are passed as void* (cudaStream_t); NULL = legacy default stream. */

/*
 * Uplink: per-cluster CD L-MMSE (detect.cpp:67-110) over P = S*C problems,
 * then fusion (detect.cpp:180-187).
 *   C_total   clusters in the whole system (C_total >= C; C_total > C when the
 *             other clusters live on other GPUs).  Uniform weights are
 *             1/C_total.
 *   x_local   optional [P][U] in `fmt` (NULL = not returned).
 *   sigma2    optional [P] fp32: optimal-fusion variances (post_eq_variance);
 *             required scratch when fusion == OPTIMAL (NULL = internal).
 *             Optimal fusion supports U <= 32 (DCDG_EINVAL otherwise, as
 *             dcdg_post_eq_variance); uniform fusion takes any U.
 *   xhat      optional [S][U] fp32 complex.  With C == C_total it is the
 *             reference's fused estimate (ascending-cluster order).  With
 *             C < C_total it is this GPU's partial: uniform: sum_c x_c/C_total;
 *             optimal: sum_c x_c/sigma2_c, with the matching partial weight
 *             sums written to wsum [S] (fp32) for the cross-GPU reduction.
 */
int dcdg_ul_detect(dcdg_ctx* ctx, const void* H, const void* y, int S, int C, int C_total,
                   int Bc, int U, int K, double n0, double ex, int fmt, int fusion,
                   void* x_local, float* sigma2, float* xhat, float* wsum, void* stream);

/*
 * Downlink: per-cluster CD ZF precoding (precode.cpp:52-99) plus
 * power_scale to rho/sqrt(C_total) (precode.cpp:101-111,155).
 *   rho       total amplitude; rho == 0 returns the raw (unnormalised)
 *             cd_precode beamformer, rho < 0 is an error.
 *   s         [S][U] symbols in `fmt` (the broadcast payload).
 *   x_dl      [P][B_c] beamformers in `fmt`.
 *   gain_part optional [P] fp32: Re(s^H H_dl,c x_c) per cluster, the
 *             cluster's share of assemble_blocks' effective_gain numerator.
 *   gain      optional [S] fp32: effective_gain (requires C == C_total).
 */
int dcdg_dl_precode(dcdg_ctx* ctx, const void* H, const void* s, int S, int C, int C_total,
                    int Bc, int U, int K, double rho, int fmt, void* x_dl, float* gain_part,
                    float* gain, void* stream);

/* Per-update traces of ONE problem (the SweepObserver debug path,
 * include/dcd/detect.hpp:28-36): the CD iterates after every coordinate
 * update, in the reference's order (sweep t, coordinate j -> entry t*U + j),
 * from the one-warp generic kernels (fp32 arithmetic on the stored inputs).
 *   dcdg_ul_trace: x_trace [K*U][U], r_trace [K*U][Bc] complex fp32
 *                  (x and the maintained residual, detect.cpp:106);
 *   dcdg_dl_trace: x_trace [K*U][Bc] complex fp32 (the unscaled beamformer,
 *                  precode.cpp:95).
 * H / y / s as one problem of dcdg_ul_detect / dcdg_dl_precode; same checks. */
int dcdg_ul_trace(dcdg_ctx* ctx, const void* H, const void* y, int Bc, int U, int K, double n0,
                  double ex, int fmt, float* x_trace, float* r_trace, void* stream);
int dcdg_dl_trace(dcdg_ctx* ctx, const void* H, const void* s, int Bc, int U, int K, int fmt,
                  float* x_trace, void* stream);

/* sigma2[p] = (E_x/U) tr((I + (E_x/N0) H_p^H H_p)^-1)  (detect.cpp:112-130). */
int dcdg_post_eq_variance(dcdg_ctx* ctx, const void* H, int P, int Bc, int U, double n0,
                          double ex, int fmt, float* sigma2, void* stream);

/* xhat[s] = sum_c w_c x_local[s][c] in ascending c (detect.cpp:180-187);
 * w from sigma2 (optimal, fusion_weights detect.cpp:132-145) or 1/C_total. */
int dcdg_fuse(dcdg_ctx* ctx, const void* x_local, const float* sigma2, int S, int C,
              int C_total, int U, int fmt, int fusion, float* xhat, float* wsum, void* stream);

/* gain[s] = (sum_c gain_part[s][c]) / ||s_s||^2  (precode.cpp:123-131). */
int dcdg_gain_reduce(dcdg_ctx* ctx, const float* gain_part, const void* s, int S, int C, int U,
                     int fmt, float* gain, void* stream);

/* gain_part[p] = Re(s^H H_dl,c x_c) of finished beamformers x_dl [P][Bc]
 * (assemble_blocks' per-cluster share, precode.cpp:123-131); feeds
 * dcdg_gain_reduce when the gain must use a different s than the precoder saw
 * (fp16 messages_only: the clusters precode the rounded broadcast). */
int dcdg_gain_part(dcdg_ctx* ctx, const void* H, const void* x_dl, const void* s, int S, int C, int Bc,
                   int U, int fmt, float* gain_part, void* stream);

/* Finalize a cross-GPU optimal-fusion reduction: xhat[s] /= wsum[s]. */
int dcdg_fuse_finalize(dcdg_ctx* ctx, float* xhat, const float* wsum, int S, int U, void* stream);

/* x[p] <- rho * x[p] / ||x[p]|| for P vectors of n complex in `fmt`
 * (power_scale, precode.cpp:101-111; zero vectors are recorded as numerical
 * errors, "power_scale: zero beamformer cannot be scaled"). */
int dcdg_power_scale(dcdg_ctx* ctx, void* x, int P, int n, double rho, int fmt, void* stream);

/* w[s][c] = (1/sigma2[s][c]) / sum_c' (1/sigma2[s][c'])  (fusion_weights,
 * detect.cpp:132-145), for S independent sets of C variances. */
int dcdg_fusion_weights(dcdg_ctx* ctx, const float* sigma2, int S, int C, float* w, void* stream);

/* Waits for `stream`, then returns and clears the first numerical error the
 * kernels recorded since the last call (DCDG_OK if none).  The message
 * (dcdg_last_error) is the reference's exception text; the failing problem
 * index is available from dcdg_last_error_problem(). */
int dcdg_sync_status(dcdg_ctx* ctx, void* stream);

/* The same check without a blocking read: dcdg_status_enqueue copies the
 * device status word to `host_word` (pinned memory) on `stream` (capturable
 * into a CUDA graph with the call it follows); after the caller has
 * synchronised the stream, dcdg_status_decode(ctx, *host_word) returns and
 * clears the recorded error exactly as dcdg_sync_status does. */
int dcdg_status_enqueue(dcdg_ctx* ctx, unsigned long long* host_word, void* stream);
int dcdg_status_decode(dcdg_ctx* ctx, unsigned long long key);
long long dcdg_last_error_problem(void);

/* Number of kernel launches issued through this context (for bench.py). */
uint64_t dcdg_launch_count(dcdg_ctx* ctx);

/* ---- hard decisions and BER --------------------------------- */
/* Full-H MMSE bias factors of S subcarriers whose C cluster tiles are local
 * (mmse_bias_factors, detect.cpp:227-242): beta [S][U] fp32,
 * beta_u = 1 - kappa [(H^H H + kappa I)^-1]_uu, H the stacked C*B_c x U
 * channel, kappa = N0/E_x (kappa == 0 gives 1).  U <= 32. */
int dcdg_mmse_bias(dcdg_ctx* ctx, const void* H, int S, int C, int Bc, int U, double n0, double ex,
                   int fmt, float* beta, void* stream);

/* labels[i] = Constellation::slice(x[i] / beta[i]) (mimo.cpp:111-122; beta
 * may be NULL): nearest Gray QAM point (qam 4/16/64, energy ex) computed in
 * fp64, distance ties to the lowest label. */
int dcdg_slice(dcdg_ctx* ctx, const void* x, int fmt, const float* beta, int64_t n, int qam,
               double ex, uint8_t* labels, void* stream);

/* *errors += number of bits where labels differ from `bits` (log2(qam) bits
 * per symbol, MSB first, one byte per bit as dcd::make_batch stores them). */
int dcdg_bit_errors(dcdg_ctx* ctx, const uint8_t* labels, const uint8_t* bits, int64_t n, int qam,
                    unsigned long long* errors, void* stream);

/* Downlink receive (downlink_receive_and_ber, precode.cpp:204-233) with every
 * cluster local: y0 = sum_c H_dl,c x_c, beta[s] = Re(s^H y0)/||s||^2,
 * labels of (y0 + noise)/beta (noise [S][U] complex fp32 or NULL);
 * flagged[s] = 1 (labels 0xff) when beta <= 0 or non-finite. */
int dcdg_dl_receive(dcdg_ctx* ctx, const void* H, const void* x_dl, const void* s,
                    const float* noise, int S, int C, int Bc, int U, int fmt, int qam, double ex,
                    uint8_t* labels, float* beta, uint8_t* flagged, void* stream);

/* ---- BER-sweep building blocks (fp32 only) ---- */

/* Device-side batch synthesis (make_batch + run_uplink_round's observation,
 * cluster.cpp:80-105,142-145) with a counter-based generator (Philox-4x32-10)
 * keyed by (seed, purpose, trial = first_trial + s, element): the channel
 * tiles H [S][C][U][Bc] ~ CN(0,1), y = H x + n [S][C][Bc] with n ~ CN(0,n0)
 * (y may be NULL), payload bits [S][U*log2(qam)] (one byte per bit, MSB first),
 * the QAM symbols x [S][U] (sym may be NULL) and downlink receiver noise
 * [S][U] ~ CN(0,n0) (noise_dl may be NULL).  The channel of global antenna
 * row b = c*Bc + i does not depend on the cluster split. */
int dcdg_synth(dcdg_ctx* ctx, int S, int C, int Bc, int U, int qam, double ex, double n0, uint64_t seed,
               uint64_t first_trial, void* H, void* y, uint8_t* bits, void* sym, void* noise_dl, void* stream);

/* Matched-filter detector over all C clusters of each subcarrier (mf_detect,
 * detect.cpp:191-218): xhat[s][u] = sum_c h_cu^H y_c / sum_c ||h_cu||^2. */
int dcdg_mf_detect(dcdg_ctx* ctx, const void* H, const void* y, int S, int C, int Bc, int U, float* xhat,
                   void* stream);

/* Matched-filter precoder (mf_precode, precode.cpp:171-202): per cluster
 * x_c = (rho/sqrt(C)) H_c s / ||H_c s||, x_dl [S][C][Bc]. */
int dcdg_mf_precode(dcdg_ctx* ctx, const void* H, const void* s, int S, int C, int Bc, int U, double rho,
                    float* x_dl, void* stream);

/* Exact L-MMSE on the full channel of each subcarrier (lmmse_exact,
 * detect.cpp:54-65): xhat = (H^H H + n0/ex I)^-1 H^H y, Cholesky solve
 * (numerics.cpp:30-75), the C tiles stacked.  U <= 32. */
int dcdg_lmmse_exact(dcdg_ctx* ctx, const void* H, const void* y, int S, int C, int Bc, int U, double n0,
                     double ex, float* xhat, void* stream);

/* Exact min-norm zero-forcing precoder on the full channel (zf_exact,
 * precode.cpp:31-50) followed by power_scale(x, rho) (rho == 0: raw),
 * x_dl [S][C][Bc] in the tile order of H.  U <= 32. */
int dcdg_zf_exact(dcdg_ctx* ctx, const void* H, const void* s, int S, int C, int Bc, int U, double rho,
                  float* x_dl, void* stream);

/* In-place round of n fp32 values to the nearest binary16 (RNE), widened
 * back: the wire-format rounding of PrecisionScope::messages_only
 * (precision.cpp:43-72, detect.cpp:170-173, precode.cpp:159-160). */
int dcdg_round_fp16(dcdg_ctx* ctx, float* x, int64_t n, void* stream);

/* Format conversion on the device: fp32 complex <-> fp16 complex (RNE),
 * interleaved (DCDG_FP16) or row-pair planar (DCDG_FP16_PAIRS, n_complex
 * even) — the latter is the DCDG_FP16 layout of H and y. */
int dcdg_convert(dcdg_ctx* ctx, const void* src, int src_fmt, void* dst, int dst_fmt,
                 int64_t n_complex, void* stream);

/* fp16 algorithm of a context (DCDG_FP16 batches of dcdg_ul_detect and
 * dcdg_dl_precode):
 *   DCDG_ALG_SWEEP  the half2 residual sweep kernels (h_j^H r dots and rank-1
 *                   r / x updates in half2 arithmetic, the paper's
 *                   half-precision path: detect.cpp:67-110 and
 *                   precode.cpp:52-99 with fp16 arithmetic);
 *   DCDG_ALG_GRAM   fp16 storage, fp32 arithmetic: G = H^H H (and z = H^H y)
 *                   on the tensor cores (mma.sync, fp32 accumulation), then
 *                   the same sweeps in the U-dimensional spaces c = H^H r
 *                   (uplink) and w = H^H x = G a (downlink, x = H a formed at
 *                   the end) (B_c = 32, U = 16; other shapes use the sweep
 *                   kernels).
 * Both meet the fp16 tolerance against the reference; GRAM is the default. */
#define DCDG_ALG_SWEEP 0
#define DCDG_ALG_GRAM 1
int dcdg_set_fp16_algorithm(dcdg_ctx* ctx, int alg);

/* Which kernel variant a (direction, Bc, U, fmt) problem shape dispatches to:
 * writes a short name ("ul_f32_reg<32,16,8>", "ul_generic_f32", …). */
int dcdg_kernel_name(int direction /*0 UL, 1 DL*/, int Bc, int U, int fmt, char* buf, int len);
/* As dcdg_kernel_name, for the fp16 algorithm a context selects. */
int dcdg_ctx_kernel_name(dcdg_ctx* ctx, int direction, int Bc, int U, int fmt, char* buf, int len);

/* ---- fused cross-GPU exchange over peer memory (NVLink P2P) ----------------
 * Replaces "CD kernel, then an NCCL collective" for the uplink fusion of
 * decentralized_cd_detect (detect.cpp:164-187) across the GPUs of one node:
 * the CD kernel's epilogue stores each cluster estimate x_c of subcarrier s
 * straight into the exchange window of the rank that owns s, its last CTA
 * publishes the batch epoch to every owner (system-scope release), and the
 * owner's fusion kernel waits for all ranks' epochs and sums the C_total
 * estimates in ascending cluster order — bitwise the single-GPU result.
 * One process per GPU; windows are exported with CUDA IPC.
 *
 *   dcdg_xwin_create  allocate this rank's window: 2 parity buffers of
 *                     buf_bytes >= S_own*C_total*U*bytes_per_complex (+256-B
 *                     pad + S_own*C_total*4 for optimal fusion), S_own = S/world
 *                     (uplink), see dcdg_dl_precode_xchg for the downlink
 *   dcdg_xwin_handle  DCDG_XWIN_HANDLE_BYTES opaque bytes to send to the peers
 *   dcdg_xwin_open    map peer `peer`'s window from its handle
 * Every rank must issue the same sequence of dcdg_ul_detect_xchg /
 * dcdg_dl_precode_xchg calls (the epochs are per-window call counters), on one
 * stream per window.  A rank whose
 * peers never publish gets DCDG_ECUDA from dcdg_sync_status after the window
 * timeout (default 20 s), not a hang. */
#define DCDG_XWIN_HANDLE_BYTES 64
typedef struct dcdg_xwin dcdg_xwin;
int dcdg_xwin_create(dcdg_ctx* ctx, int world, int rank, int64_t buf_bytes, dcdg_xwin** out);
int dcdg_xwin_handle(dcdg_xwin* w, void* handle);
int dcdg_xwin_open(dcdg_xwin* w, int peer, const void* handle);
int dcdg_xwin_set_timeout(dcdg_xwin* w, int64_t timeout_ns);
int dcdg_xwin_destroy(dcdg_xwin* w);
/* Uplink detection of this rank's C clusters [c0, c0+C) of C_total over all S
 * subcarriers (H [S][C][U][B_c], y [S][C][B_c] as in dcdg_ul_detect), fused
 * through the windows: xhat [S/world][U] receives the fused estimates of the
 * subcarriers this rank owns, [rank*S/world, (rank+1)*S/world). */
int dcdg_ul_detect_xchg(dcdg_ctx* ctx, dcdg_xwin* w, const void* H, const void* y, int S, int C, int c0,
                        int C_total, int Bc, int U, int K, double n0, double ex, int fmt, int fusion,
                        float* xhat, void* stream);
/* Downlink precoding of this rank's clusters [c0, c0+C) with decentralized_cd_precode's
 * exchanges (precode.cpp:136-169) over the windows: the root's symbols s [S][U]
 * (read on rank `root` only) are stored into every rank's window (the centre ->
 * cluster broadcast), each rank precodes from its own window into x_dl [S*C][B_c]
 * (power-scaled to rho/sqrt(C_total)), publishes its per-cluster gain shares
 * into every window, and gain [S] (optional, every rank) is the effective gain
 * summed over all C_total clusters in ascending order — bitwise the single-GPU
 * value.  Window size: S*U*bytes_per_complex (+256-B pad) + S*C_total*4. */
int dcdg_dl_precode_xchg(dcdg_ctx* ctx, dcdg_xwin* w, int root, const void* H, const void* s, int S, int C,
                         int c0, int C_total, int Bc, int U, int K, double rho, int fmt, void* x_dl,
                         float* gain, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DCDG_H */
