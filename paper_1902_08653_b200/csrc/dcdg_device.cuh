// Device-side building blocks shared by the CD kernels: sm_100a PTX wrappers
// for the bulk-copy (TMA 1-D) staging pipeline, sub-warp reductions, complex
// load/convert helpers and the numerical-status word.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dcdg {

// ---------------------------------------------------------------------------
// shared-memory async bulk copy (cp.async.bulk, SASS UBLKCP) + mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Orders this thread's prior generic-proxy shared-memory accesses before
// subsequent async-proxy (bulk copy) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16-B aligned).
// The data is streamed exactly once, so it is marked evict-first in L2.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// 32-bit shared loads that ptxas may not merge into a vector load: used to
// place interleaved (re, im) data directly into planar register pairs.
__device__ __forceinline__ float lds_f32(const void* p) {
  float v;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(const void* p) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// ---------------------------------------------------------------------------
// reductions over a group of G consecutive lanes (xor butterfly: every lane of
// the group ends with the bitwise-identical sum, so redundant per-lane scalar
// updates stay consistent)
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ float gsum(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
__device__ __forceinline__ __half2 gsum_h2(__half2 v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = __hadd2(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) { return gsum<32>(v); }

// ---------------------------------------------------------------------------
// packed fp32x2 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2: one instruction for
// two lanes of fp32, scalar operands broadcast, negation folded)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 ffma2(float s, float2 b, float2 c) { return __ffma2_rn(make_float2(s, s), b, c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float s, float2 b) { return __fmul2_rn(make_float2(s, s), b); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
// Build the planar register pair (a, b) once: x + (+0.0) is not an identity
// under IEEE (it maps -0 to +0), so ptxas keeps the FADD2 result instead of
// re-pairing the source registers with MOVs before every later use.
#ifndef DCDG_PAIR_MODE
#define DCDG_PAIR_MODE 0
#endif
__device__ __forceinline__ float2 pair(float a, float b) {
#if DCDG_PAIR_MODE == 1
  // (a, b) = a*(1,0) + b*(0,1) with broadcast operands: 2 packed ops, no MOVs
  return __ffma2_rn(make_float2(b, b), make_float2(0.f, 1.f), __fmul2_rn(make_float2(a, a), make_float2(1.f, 0.f)));
#else
  // x + (+0.0) is not an IEEE identity (-0 -> +0), so ptxas keeps the result
  return __fadd2_rn(make_float2(a, b), make_float2(0.f, 0.f));
#endif
}
__device__ __forceinline__ float hsum(float2 a) { return a.x + a.y; }
__device__ __forceinline__ float2 shfl_xor2(float2 v, int o) {
  return make_float2(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
}

// Group-wide sums of NV float2 values over aligned groups of G lanes, every
// lane of a group ending with bitwise the same sums.  DCDG_BFLY_SHALLOW
// levels at the bottom of the xor butterfly are replaced by one gather round:
// the remaining 2^L partners are read with independent shuffles and summed
// as a pairwise tree, so the dependency chain has L - 1 fewer shuffle
// latencies for (2^L - 1) / L times the shuffles of those levels.  Every lane
// adds the same partial sums in a commuted order, so the results agree.
#ifndef DCDG_BFLY_SHALLOW
#define DCDG_BFLY_SHALLOW 0
#endif
template <int G, int NV>
__device__ __forceinline__ void group_allreduce2(float2 (&d)[NV]) {
  constexpr int L = (DCDG_BFLY_SHALLOW >= 2 && G >= 4) ? 2 : 0;  // gathered bottom levels (xor 1, 2)
#pragma unroll
  for (int o = G / 2; o >= (L ? 4 : 1); o >>= 1)
#pragma unroll
    for (int a = 0; a < NV; ++a) d[a] = fadd2(d[a], shfl_xor2(d[a], o));
  if constexpr (L == 2) {
#pragma unroll
    for (int a = 0; a < NV; ++a) {
      const float2 s1 = shfl_xor2(d[a], 1), s2 = shfl_xor2(d[a], 2), s3 = shfl_xor2(d[a], 3);
      d[a] = fadd2(fadd2(d[a], s1), fadd2(s2, s3));
    }
  }
}

// ---------------------------------------------------------------------------
// complex element access for the two storage formats
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 ldc(const float2* p, size_t i) { return __ldg(p + i); }
__device__ __forceinline__ float2 ldc(const __half2* p, size_t i) { return __half22float2(__ldg(p + i)); }
__device__ __forceinline__ void stc(float2* p, size_t i, float2 v) { p[i] = v; }
__device__ __forceinline__ void stc(__half2* p, size_t i, float2 v) { p[i] = __floats2half2_rn(v.x, v.y); }

// Element i of a B_c-vector stored in the fp16 row-pair planar layout
// ({re_2i, re_2i+1, im_2i, im_2i+1}); fp32 vectors are plain interleaved.
__device__ __forceinline__ float2 ldv(const float2* v, int i) { return __ldg(v + i); }
__device__ __forceinline__ float2 ldv(const __half2* v, int i) {
  const __half* h = reinterpret_cast<const __half*>(v) + (i >> 1) * 4 + (i & 1);
  return make_float2(__half2float(h[0]), __half2float(h[2]));
}

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization starts while its
// predecessor drains and waits here until the predecessor's results are
// visible; without the attribute this is a no-op.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ __half2 u32_as_h2(uint32_t u) {
  __half2 h;
  memcpy(&h, &u, 4);
  return h;
}
__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) {
  uint32_t u;
  memcpy(&u, &h, 4);
  return u;
}

// ---------------------------------------------------------------------------
// numerical status: the first (lowest problem index) error of a batch wins,
// mirroring the reference's in-order cluster loop that throws at the first
// failing cluster (src/detect.cpp:32-52, src/precode.cpp:62-78,101-111).
// key = problem << 24 | code << 16 | detail
// ---------------------------------------------------------------------------
enum StatusCode : uint32_t {
  ST_ZERO_ROW = 1,        // precode.cpp:74-76   runtime_error
  ST_ZERO_BEAMFORMER = 2, // precode.cpp:107-108 runtime_error
  ST_SINGULAR = 3,        // numerics.cpp:55-56  runtime_error
  ST_BAD_VARIANCE = 4,    // detect.cpp:138-139  invalid_argument
  ST_RANK_DEFICIENT = 5,  // precode.cpp:42-43   runtime_error (zf_exact)
  ST_MF_ZERO_ENERGY = 6,  // detect.cpp:213-215  runtime_error (mf_detect)
  ST_MF_ZERO_BEAMFORMER = 7,  // precode.cpp:193-196 runtime_error (mf_precode)
  ST_XCHG_TIMEOUT = 8,        // fused exchange: a peer's signal never arrived (detail = peer rank)
};

__device__ __forceinline__ void record_status(unsigned long long* st, long long p, uint32_t code, uint32_t detail) {
  if (st) atomicMin(st, (static_cast<unsigned long long>(p) << 24) | (code << 16) | (detail & 0xffffu));
}

// ---------------------------------------------------------------------------
// fused cross-GPU exchange over peer memory (NVLink P2P): the uplink kernels
// store each cluster estimate straight into the exchange window of the GPU
// that owns the subcarrier, then the last CTA of the launch signals every
// owner with a system-scope release store of the batch epoch.
// Window layout (per rank): [flags: kXchgMaxRanks u64][pad to 256 B]
//   [parity 0: x [S_own][C_total][U] | sigma2 [S_own][C_total]]
//   [parity 1: same]
// ---------------------------------------------------------------------------
constexpr int kXchgMaxRanks = 8;
constexpr int kXchgFlagBytes = 256;

// Flag slots (u64) at the start of every window: uplink estimates published by
// rank q -> slot q; downlink symbols pushed by the root -> kSlotSymbols;
// downlink gain shares published by rank q -> kSlotGain + q.
constexpr int kSlotSymbols = 8;
constexpr int kSlotGain = 16;

struct XMap {
  unsigned char* win[kXchgMaxRanks];  // every rank's window base (self included), in this process's address space
  unsigned int* counter;              // local CTA-completion counter (reset by the last CTA)
  const unsigned long long* epoch_dev;  // this call's batch epoch, in device memory (xchg_advance_kernel):
                                       // read by the kernels, so a captured call replays with fresh epochs
  int flag_slot;                      // xchg_cta_done publishes to slot flag_slot (+ rank if per_rank)
  int per_rank;
  long long buf_bytes;                // bytes of one parity buffer
  long long sig_off;                  // offset of the sigma2 region inside a parity buffer
  int world, rank;
  int S_own;                          // subcarriers owned per rank
  int C_local, c0, C_total, U;
  int esz;                            // bytes per complex of x (8 fp32, 4 fp16)
};

// The call's batch epoch (written by the previous kernel on the stream) and
// its parity buffer.
__device__ __forceinline__ unsigned long long xchg_epoch(const unsigned long long* e) { return __ldcg(e); }
__device__ __forceinline__ unsigned long long xchg_epoch(const XMap& m) { return xchg_epoch(m.epoch_dev); }

// Destination of problem p's estimate (p = s*C_local + c, s global over the batch).
// (P = S*C_local < 2^31 is checked on the host: 32-bit index math.)
__device__ __forceinline__ unsigned char* xchg_x_dst(const XMap& m, int p, int parity) {
  const int s = p / m.C_local;
  const int c = p - s * m.C_local;
  const int owner = s / m.S_own;
  const int s_in = s - owner * m.S_own;
  return m.win[owner] + kXchgFlagBytes + parity * m.buf_bytes +
         static_cast<long long>((s_in * m.C_total + m.c0 + c) * m.U) * m.esz;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread 0 of the block waits until slots [slot0, slot0 + n) of the local
// window's flags reach `epoch` (acquire, system scope); a peer that never
// publishes within timeout_ns is recorded as ST_XCHG_TIMEOUT.  Returns false
// (for the whole block) on timeout.
__device__ __forceinline__ bool xchg_block_wait(const unsigned char* win, int slot0, int n, unsigned long long epoch,
                                                long long timeout_ns, unsigned long long* status) {
  __shared__ int ok_;
  if (threadIdx.x == 0) {
    ok_ = 1;
    const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(win);
    for (int q = 0; q < n && ok_; ++q) {
      const unsigned long long t0 = globaltimer_ns();
      while (ld_acquire_sys(flags + slot0 + q) < epoch) {
        if (static_cast<long long>(globaltimer_ns() - t0) > timeout_ns) {
          if (blockIdx.x == 0) record_status(status, 0, ST_XCHG_TIMEOUT, q);
          ok_ = 0;
          break;
        }
        __nanosleep(200);
      }
    }
  }
  __syncthreads();
  return ok_ != 0;
}

// Called by every thread of every CTA after its last remote store: the last
// CTA to finish publishes the epoch to flag slot flag_slot (+ rank) of every
// rank's window.
__device__ __forceinline__ void xchg_cta_done(const XMap& m) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(m.counter, 1u);
    if (t == gridDim.x - 1) {
      __threadfence_system();
      const int slot = m.flag_slot + (m.per_rank ? m.rank : 0);
      const unsigned long long e = xchg_epoch(m);
      for (int q = 0; q < m.world; ++q)
        st_release_sys(reinterpret_cast<unsigned long long*>(m.win[q]) + slot, e);
      *m.counter = 0u;  // next launch on this stream starts from zero
    }
  }
}

// D += A B, mma.sync m16n8k16, fp16 operands, fp32 accumulate
__device__ __forceinline__ void mma_f16f32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// x = hi + lo in binary16 pairs (the split operands of an fp32-accurate Gram
// on the fp16 tensor cores): hi = rn(x), lo = rn(x - hi)
__device__ __forceinline__ void split_h2(float2 x, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __float22half2_rn(x);
  const float2 hf = __half22float2(h);
  hi = h2_as_u32(h);
  lo = h2_as_u32(__float22half2_rn(make_float2(x.x - hf.x, x.y - hf.y)));
}
// W' word of an interleaved (re, im) binary16 pair: (im, -re)
__device__ __forceinline__ uint32_t wprime(uint32_t w) { return __byte_perm(w, 0, 0x1032) ^ 0x80000000u; }

// complex c -= a * b
__device__ __forceinline__ void csub_mul(float& cr, float& ci, float ar, float ai, float br, float bi) {
  cr = fmaf(-ar, br, fmaf(ai, bi, cr));
  ci = fmaf(-ar, bi, fmaf(-ai, br, ci));
}

// post_eq_variance of a problem from the Gram rows its 8 lanes hold
// (detect.cpp:112-130): sigma^2 = (E_x/U) tr (I + (E_x/N0) G)^-1.  The
// inverse's trace comes from the sweep operator in place on the lanes' rows
// (lane k: rows 2k, 2k+1 of A = I + gam G): pivot kk in ascending order, its
// row broadcast through shared memory,
//     d = a_kk,kk;  a_ij -= (a_i,kk / d) a_kk,j  (i, j != kk);
//     a_i,kk <- a_i,kk / d;  a_kk,j <- a_kk,j / d;  a_kk,kk <- -1/d,
// after which A holds -A^-1.  The pivots are the Cholesky pivots of the
// reference's hermitian_solve, so its singularity test (d > 1e-14 max A_jj,
// numerics.cpp:38-41,55-56) applies unchanged.  Returns tr A^-1 (on every lane
// of the problem); `singular` is set on the lanes that saw a failing pivot.
template <int U>
__device__ __forceinline__ float gram_trace_inverse(float (&ar0)[U], float (&ai0)[U], float (&ar1)[U],
                                                    float (&ai1)[U], int k, float gam, float4* prow,
                                                    bool& singular, bool rows_hold_a = false) {
  // A = I + gam G in place over the Gram rows (they are dead after the sweeps),
  // unless the rows already hold A
  if (!rows_hold_a) {
#pragma unroll
    for (int j = 0; j < U; ++j) {
      ar0[j] = fmaf(gam, ar0[j], j == 2 * k ? 1.f : 0.f);
      ai0[j] *= gam;
      ar1[j] = fmaf(gam, ar1[j], j == 2 * k + 1 ? 1.f : 0.f);
      ai1[j] *= gam;
    }
  }
  float dmax = 0.f;
#pragma unroll
  for (int jp = 0; jp < U / 2; ++jp)
    if (k == jp) dmax = fmaxf(ar0[2 * jp], ar1[2 * jp + 1]);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const float floor_ = 1e-14f * dmax;
#pragma unroll
  for (int kk = 0; kk < U; ++kk) {
    float4* slot = prow + (kk & 1) * (U / 2);  // alternating [U/2] float4 rows (pairs of entries)
    if (k == kk / 2) {
#pragma unroll
      for (int j = 0; j < U / 2; ++j)
        slot[j] = (kk & 1) ? make_float4(ar1[2 * j], ai1[2 * j], ar1[2 * j + 1], ai1[2 * j + 1])
                           : make_float4(ar0[2 * j], ai0[2 * j], ar0[2 * j + 1], ai0[2 * j + 1]);
    }
    __syncwarp();
    const float d = reinterpret_cast<const float*>(slot)[2 * kk];
    if (!(d > floor_)) singular = true;
    const float inv = __frcp_rn(d);
    const bool piv0 = (2 * k == kk), piv1 = (2 * k + 1 == kk);
    // pivot row: a_kk,j - (1 - 1/d) a_kk,j = a_kk,j / d with the same update
    const float f0r = piv0 ? 1.f - inv : ar0[kk] * inv, f0i = piv0 ? 0.f : ai0[kk] * inv;
    const float f1r = piv1 ? 1.f - inv : ar1[kk] * inv, f1i = piv1 ? 0.f : ai1[kk] * inv;
#pragma unroll
    for (int jq = 0; jq < U / 2; ++jq) {
      const float4 v = slot[jq];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * jq + h;
        if (j == kk) continue;
        const float br = h ? v.z : v.x, bi = h ? v.w : v.y;
        csub_mul(ar0[j], ai0[j], f0r, f0i, br, bi);
        csub_mul(ar1[j], ai1[j], f1r, f1i, br, bi);
      }
    }
    ar0[kk] = piv0 ? -inv : f0r;
    ai0[kk] = piv0 ? 0.f : f0i;
    ar1[kk] = piv1 ? -inv : f1r;
    ai1[kk] = piv1 ? 0.f : f1i;
  }
  float t = 0.f;
#pragma unroll
  for (int jp = 0; jp < U / 2; ++jp)
    if (k == jp) t = -(ar0[2 * jp] + ar1[2 * jp + 1]);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}


// Shared-memory image of A = I + gam G for the paired sweep operator below:
// row i, column pair jq (columns 2jq, 2jq+1) at float4 slot
// i*U/2 + (jq ^ ((i >> 1) & 7)):
//     (Re A[i][2jq], Re A[i][2jq+1], Im A[i][2jq], Im A[i][2jq+1]).
// The XOR skew makes the 8 lanes' reads of rows 2k (or 2k+1) conflict-free.
template <int U>
__device__ __forceinline__ int apair_slot(int i, int jq) {
  return i * (U / 2) + (jq ^ ((i >> 1) & 7));
}

// post_eq_variance from A = I + gam G held as COLUMN PAIRS
// (detect.cpp:112-130): lane k of the problem's U/2 lanes keeps rows 2k and
// 2k+1 as R?r[jq] = (Re A[i][2jq], Re A[i][2jq+1]) and R?i[jq] likewise, so
// every update of the sweep operator (same pivots and arithmetic as
// gram_trace_inverse above) is 4 FFMA2 per column pair and row, the row's
// coefficient a broadcast .F32 operand:
//     a_ij -= (a_i,kk / d) a_kk,j   (i != kk; column kk is overwritten after).
// The pivot row is broadcast through `prow` (2 x U/2 float4 per problem) in
// the same column-pair layout.  Returns tr A^-1 on every lane of the problem;
// `singular` as in gram_trace_inverse.
template <int U>
__device__ __forceinline__ float gram_trace_inverse_cpairs(float2 (&R0r)[U / 2], float2 (&R0i)[U / 2],
                                                           float2 (&R1r)[U / 2], float2 (&R1i)[U / 2], int k,
                                                           float4* prow, bool& singular) {
  constexpr int NQ = U / 2;
  float dmax = 0.f;
#pragma unroll
  for (int jq = 0; jq < NQ; ++jq)
    if (k == jq) dmax = fmaxf(R0r[jq].x, R1r[jq].y);
#pragma unroll
  for (int o = U / 4; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const float floor_ = 1e-14f * dmax;
#pragma unroll
  for (int kk = 0; kk < U; ++kk) {
    const int h = kk & 1, qk = kk >> 1;  // owner's row h; the pivot column is in pair qk, half h
    float4* slot = prow + h * NQ;        // alternating broadcast rows
    if (k == qk) {  // two 8-B stores per slot straight from the register pairs (asm: no merged 16-B
                    // store, which costs four re-pairing moves per slot)
      const uint32_t a = smem_u32(slot);
#pragma unroll
      for (int jq = 0; jq < NQ; ++jq) {
        const float2 r = h ? R1r[jq] : R0r[jq], i = h ? R1i[jq] : R0i[jq];
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a + 16 * jq), "f"(r.x), "f"(r.y) : "memory");
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a + 16 * jq + 8), "f"(i.x), "f"(i.y) : "memory");
      }
    }
    __syncwarp();
    const float d = reinterpret_cast<const float*>(slot + qk)[h];
    if (!(d > floor_)) singular = true;
    const float inv = __frcp_rn(d);
    const bool piv0 = (2 * k == kk), piv1 = (2 * k + 1 == kk);
    // row coefficients f_i = a_i,kk / d; the pivot row's is 1 - 1/d (a_kk,j / d
    // with the same update)
    const float a0r = h ? R0r[qk].y : R0r[qk].x, a0i = h ? R0i[qk].y : R0i[qk].x;
    const float a1r = h ? R1r[qk].y : R1r[qk].x, a1i = h ? R1i[qk].y : R1i[qk].x;
    const float f0r = piv0 ? 1.f - inv : a0r * inv, f0i = piv0 ? 0.f : a0i * inv;
    const float f1r = piv1 ? 1.f - inv : a1r * inv, f1i = piv1 ? 0.f : a1i * inv;
#pragma unroll
    for (int jq = 0; jq < NQ; ++jq) {
      const float4 v = slot[jq];
      const float2 br = make_float2(v.x, v.y), bi = make_float2(v.z, v.w);
      // (ar + i ai) -= (fr + i fi)(br + i bi) over the column pair
      R0r[jq] = ffma2(f0i, bi, ffma2(-f0r, br, R0r[jq]));
      R0i[jq] = ffma2(-f0i, br, ffma2(-f0r, bi, R0i[jq]));
      R1r[jq] = ffma2(f1i, bi, ffma2(-f1r, br, R1r[jq]));
      R1i[jq] = ffma2(-f1i, br, ffma2(-f1r, bi, R1i[jq]));
    }
    // column kk: a_i,kk <- a_i,kk / d, the pivot's own entry -1/d
    const float n0r = piv0 ? -inv : f0r, n0i = piv0 ? 0.f : f0i;
    const float n1r = piv1 ? -inv : f1r, n1i = piv1 ? 0.f : f1i;
    if (h) {
      R0r[qk].y = n0r;
      R0i[qk].y = n0i;
      R1r[qk].y = n1r;
      R1i[qk].y = n1i;
    } else {
      R0r[qk].x = n0r;
      R0i[qk].x = n0i;
      R1r[qk].x = n1r;
      R1i[qk].x = n1i;
    }
  }
  float t = 0.f;
#pragma unroll
  for (int jq = 0; jq < NQ; ++jq)
    if (k == jq) t = -(R0r[jq].x + R1r[jq].y);
#pragma unroll
  for (int o = U / 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// Sweep operator with 2x2 block pivots (1) or single pivots (0): measured per
// kernel (profiles/lab/README.md) -- the fused fp32 variance keeps single
// pivots (0.402 vs 0.420 ms), the tensor-core variance kernel takes block
// pivots at U <= 16 (U=16: 0.366 -> 0.314 ms) and single pivots at U = 32.
#ifndef DCDG_SIG_BLOCK2
#define DCDG_SIG_BLOCK2 0
#endif
#ifndef DCDG_PEV_TC_BLOCK2_MAXU
#define DCDG_PEV_TC_BLOCK2_MAXU 16
#endif
// The same sweep operator two pivots at a time (a 2x2 block pivot on the
// column pair qk = rows 2qk, 2qk+1 = the pair lane qk owns): with
// P = A[{2qk,2qk+1}][{2qk,2qk+1}] = [[d0, c], [conj c, e]],
//     a_ij -= A_iP P^-1 A_Pj  (i, j outside P),  A_iP <- A_iP P^-1,
//     A_Pj <- P^-1 A_Pj,  A_PP <- -P^-1,
// which is the two single sweeps composed, so A still ends as -A^-1.  The
// pivots checked against the floor are those of the sequential sweep
// (d0, then the Schur complement e - |c|^2/d0), as hermitian_solve's.  Half the
// pivot chain (broadcast, barrier, reciprocal) per sweep; the same FFMA2 count.
// `prow`: 2 x U/2 float4 per problem (both pivot rows of the block).
template <int U>
__device__ __forceinline__ float gram_trace_inverse_cpairs2(float2 (&R0r)[U / 2], float2 (&R0i)[U / 2],
                                                            float2 (&R1r)[U / 2], float2 (&R1i)[U / 2], int k,
                                                            float4* prow, bool& singular) {
  constexpr int NQ = U / 2;
  float dmax = 0.f;
#pragma unroll
  for (int jq = 0; jq < NQ; ++jq)
    if (k == jq) dmax = fmaxf(R0r[jq].x, R1r[jq].y);
#pragma unroll
  for (int o = U / 4; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const float floor_ = 1e-14f * dmax;
  float4* slot0 = prow;
  float4* slot1 = prow + NQ;
#pragma unroll
  for (int qk = 0; qk < NQ; ++qk) {
    const bool own = (k == qk);
    if (own) {  // both pivot rows, 8-B stores straight from the register pairs
      const uint32_t a0 = smem_u32(slot0), a1 = smem_u32(slot1);
#pragma unroll
      for (int jq = 0; jq < NQ; ++jq) {
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a0 + 16 * jq), "f"(R0r[jq].x), "f"(R0r[jq].y) : "memory");
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a0 + 16 * jq + 8), "f"(R0i[jq].x), "f"(R0i[jq].y)
                     : "memory");
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a1 + 16 * jq), "f"(R1r[jq].x), "f"(R1r[jq].y) : "memory");
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a1 + 16 * jq + 8), "f"(R1i[jq].x), "f"(R1i[jq].y)
                     : "memory");
      }
    }
    __syncwarp();
    const float4 p0 = slot0[qk], p1 = slot1[qk];
    const float d0 = p0.x, cr = p0.y, ci = p0.w, e = p1.y;  // P = [[d0, c], [conj c, e]]
    const float cc = fmaf(cr, cr, ci * ci);
    if (!(d0 > floor_)) singular = true;
    const float det = fmaf(d0, e, -cc);                      // d0 (e - |c|^2 / d0)
    if (!(det > floor_ * d0)) singular = true;
    const float id = __frcp_rn(det);
    // P^-1 = id [[e, -c], [-conj c, d0]]
    const float q00 = id * e, q11 = id * d0, q01r = -id * cr, q01i = -id * ci;  // (P^-1)_01 = -id c
    // row coefficients: f = A_iP P^-1 (i outside P) or I - P^-1 (the owner's rows)
    float f00r, f00i, f01r, f01i, f10r, f10i, f11r, f11i;
    {
      // row 2k: a0 = A[2k][2qk], a1 = A[2k][2qk+1]
      const float a0r = R0r[qk].x, a0i = R0i[qk].x, a1r = R0r[qk].y, a1i = R0i[qk].y;
      // f0 = a0 q00 + a1 conj(q01) ;  f1 = a0 q01 + a1 q11   ((P^-1)_10 = conj((P^-1)_01))
      f00r = fmaf(a0r, q00, fmaf(a1r, q01r, a1i * q01i));
      f00i = fmaf(a0i, q00, fmaf(a1i, q01r, -a1r * q01i));
      f01r = fmaf(a0r, q01r, fmaf(-a0i, q01i, a1r * q11));
      f01i = fmaf(a0r, q01i, fmaf(a0i, q01r, a1i * q11));
      const float b0r = R1r[qk].x, b0i = R1i[qk].x, b1r = R1r[qk].y, b1i = R1i[qk].y;
      f10r = fmaf(b0r, q00, fmaf(b1r, q01r, b1i * q01i));
      f10i = fmaf(b0i, q00, fmaf(b1i, q01r, -b1r * q01i));
      f11r = fmaf(b0r, q01r, fmaf(-b0i, q01i, b1r * q11));
      f11i = fmaf(b0r, q01i, fmaf(b0i, q01r, b1i * q11));
    }
    if (own) {  // I - P^-1
      f00r = 1.f - q00;
      f00i = 0.f;
      f01r = -q01r;
      f01i = -q01i;
      f10r = -q01r;   // -(P^-1)_10 = -conj(q01)
      f10i = q01i;
      f11r = 1.f - q11;
      f11i = 0.f;
    }
#pragma unroll
    for (int jq = 0; jq < NQ; ++jq) {
      const float4 v0 = slot0[jq], v1 = slot1[jq];
      const float2 b0r = make_float2(v0.x, v0.y), b0i = make_float2(v0.z, v0.w);
      const float2 b1r = make_float2(v1.x, v1.y), b1i = make_float2(v1.z, v1.w);
      // (ar + i ai) -= f0 b0 + f1 b1 over the column pair, both rows
      R0r[jq] = ffma2(f01i, b1i, ffma2(-f01r, b1r, ffma2(f00i, b0i, ffma2(-f00r, b0r, R0r[jq]))));
      R0i[jq] = ffma2(-f01i, b1r, ffma2(-f01r, b1i, ffma2(-f00i, b0r, ffma2(-f00r, b0i, R0i[jq]))));
      R1r[jq] = ffma2(f11i, b1i, ffma2(-f11r, b1r, ffma2(f10i, b0i, ffma2(-f10r, b0r, R1r[jq]))));
      R1i[jq] = ffma2(-f11i, b1r, ffma2(-f11r, b1i, ffma2(-f10i, b0r, ffma2(-f10r, b0i, R1i[jq]))));
    }
    // the pivot columns: A_iP <- f (outside P), A_PP <- -P^-1 (the owner)
    if (own) {
      R0r[qk] = make_float2(-q00, -q01r);
      R0i[qk] = make_float2(0.f, -q01i);
      R1r[qk] = make_float2(-q01r, -q11);
      R1i[qk] = make_float2(q01i, 0.f);
    } else {
      R0r[qk] = make_float2(f00r, f01r);
      R0i[qk] = make_float2(f00i, f01i);
      R1r[qk] = make_float2(f10r, f11r);
      R1i[qk] = make_float2(f10i, f11i);
    }
    __syncwarp();  // every lane has read this block's rows before the next owner stores
  }
  float t = 0.f;
#pragma unroll
  for (int jq = 0; jq < NQ; ++jq)
    if (k == jq) t = -(R0r[jq].x + R1r[jq].y);
#pragma unroll
  for (int o = U / 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// Which factorisation the variance kernels run: 1 = forward elimination on
// column pairs (gram_trace_inverse_cols below), 0 = the sweep operators above.
#ifndef DCDG_SIG_COLS
#define DCDG_SIG_COLS 1
#endif
#ifndef DCDG_SIG_COLS_STS32
#define DCDG_SIG_COLS_STS32 0
#endif
// 1: the owner's pivot column is left as -d_kk M (no per-row selects), rescaled
// in the trace.  Measured per site (profiles/lab/README.md): on in the variance
// kernel and the fp16 Gram kernel, off in the fused fp32 CD kernel.
#ifndef DCDG_SIG_COLS_SCALED
#define DCDG_SIG_COLS_SCALED 1
#endif
#ifndef DCDG_SIG_COLS_SCALED_FUSED
#define DCDG_SIG_COLS_SCALED_FUSED 0
#endif

// post_eq_variance (detect.cpp:112-130) by forward elimination of [A | I]
// held as COLUMN PAIRS: lane k of the problem's U/2 lanes keeps columns 2k,
// 2k+1 of A = I + gam G for every row i as Cr[i] = (Re A[i][2k], Re A[i][2k+1]),
// Ci[i] likewise.  Pivot kk (ascending, as hermitian_solve's Cholesky,
// numerics.cpp:51-66) updates only the rows below it,
//     a_ij -= f_i a_kk,j   (i > kk, every column j),   f_i = a_i,kk / d_kk,
// and the in-place column kk of those rows becomes -f_i.  Stored in place the
// right half of [A | I] fills exactly the columns the left half vacates, so
// at the end row i holds M = L^-1 (unit lower, A = L D L^H) left of the
// diagonal and d_i on it, and
//     tr A^-1 = sum_i (1 + sum_{j<i} |M_ij|^2) / d_i.
// The pivots d_kk are the Schur complements the reference's Cholesky checks
// against 1e-14 max_i A_ii.  Each lane's rows below kk are lane-uniform, so a
// pivot costs 4 FFMA2 per row below it (480 per lane at U = 16, against 1024
// for the in-place sweep operator), and only pivot COLUMN kk is broadcast
// (`prow`: 2 x U float2 per problem, alternating by pivot parity) -- the pivot
// row of a lane's columns is its own register.  Returns tr A^-1 on every lane
// of the problem.
// SCALED: instead of selecting -f_i into the owner's column kk row by row,
// the owner's copy of its pivot entry is zeroed, so that column keeps
// a_i,kk = -d_kk M_i,kk and stays that multiple through every later update
// (they are linear in it); the trace divides its |.|^2 by d_kk^2.
template <int U, bool SCALED = DCDG_SIG_COLS_SCALED != 0>
__device__ __forceinline__ float gram_trace_inverse_cols(float2 (&Cr)[U], float2 (&Ci)[U], int k, float4* prow,
                                                         bool& singular) {
  constexpr int NQ = U / 2;
  float dmax = 0.f;
#pragma unroll
  for (int jq = 0; jq < NQ; ++jq)
    if (k == jq) dmax = fmaxf(Cr[2 * jq].x, Cr[2 * jq + 1].y);
#pragma unroll
  for (int o = U / 4; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const float floor_ = 1e-14f * dmax;
  float invd[U];
#pragma unroll
  for (int kk = 0; kk < U; ++kk) {
    const int h = kk & 1, qk = kk >> 1;  // pivot column kk = half h of lane qk's pair
    const bool own = (k == qk);
    float2* col = reinterpret_cast<float2*>(prow) + h * U;  // (re, im) of rows kk..U-1
    if (own) {
      const uint32_t a = smem_u32(col);
#pragma unroll
      for (int i = 0; i < U; ++i)  // constant bounds: fully unrolled with the pivot loop
        if (i >= kk) {
#if DCDG_SIG_COLS_STS32
          // two 4-B stores: re and im sit in different register pairs, a
          // vector store would need two re-pairing moves per row
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + 8 * i), "f"(h ? Cr[i].y : Cr[i].x) : "memory");
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + 8 * i + 4), "f"(h ? Ci[i].y : Ci[i].x) : "memory");
#else
          asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a + 8 * i), "f"(h ? Cr[i].y : Cr[i].x),
                       "f"(h ? Ci[i].y : Ci[i].x)
                       : "memory");
#endif
        }
    }
    __syncwarp();
    const float d = col[kk].x;
    if (!(d > floor_)) singular = true;
    float inv;  // MUFU.RCP alone (<= 1 ulp): the IEEE __frcp_rn adds a Newton step and a slow-path branch to the chain
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(d));
    invd[kk] = inv;
    float2 pr = Cr[kk], pi = Ci[kk];  // pivot row kk over this lane's column pair
    // SCALED: the owner's pivot entry taken as 0: its column kk keeps
    // a_i,kk = -d_kk M_i,kk below the pivot, and every later update of that
    // column is linear in it
    if (SCALED && own) {
      if (h) {
        pr.y = 0.f;
        pi.y = 0.f;
      } else {
        pr.x = 0.f;
        pi.x = 0.f;
      }
    }
#pragma unroll
    for (int i = 1; i < U; ++i) {
      if (i <= kk) continue;
      const float2 f = fmul2(inv, col[i]);  // f_i = a_i,kk / d
      Cr[i] = ffma2(f.y, pi, ffma2(-f.x, pr, Cr[i]));
      Ci[i] = ffma2(-f.y, pr, ffma2(-f.x, pi, Ci[i]));
      if (!SCALED && own) {  // M_i,kk = -f_i
        if (h) {
          Cr[i].y = -f.x;
          Ci[i].y = -f.y;
        } else {
          Cr[i].x = -f.x;
          Ci[i].x = -f.y;
        }
      }
    }
  }
  // SCALED: column j below the diagonal holds -d_j M_ij, |M_ij|^2 = |a_ij|^2 / d_j^2
  float s0 = 1.f, s1 = 1.f;
  if (SCALED) {
#pragma unroll
    for (int jq = 0; jq < NQ; ++jq)
      if (k == jq) {
        s0 = invd[2 * jq] * invd[2 * jq];
        s1 = invd[2 * jq + 1] * invd[2 * jq + 1];
      }
  }
  // (1 + sum_j |M_ij|^2) / d_i: the 1 from the lane's own diagonal rows, the
  // |M_ij|^2 of its two columns below the diagonal
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < U; ++i) {
    const float2 m = ffma2(Cr[i], Cr[i], fmul2(Ci[i], Ci[i]));
    const float s = SCALED ? (2 * k < i ? m.x * s0 : 0.f) + (2 * k + 1 < i ? m.y * s1 : 0.f) +
                                 (2 * k == i || 2 * k + 1 == i ? 1.f : 0.f)
                           : (2 * k < i ? m.x : 0.f) + (2 * k + 1 < i ? m.y : 0.f) +
                                 (2 * k == i || 2 * k + 1 == i ? 1.f : 0.f);
    t = fmaf(s, invd[i], t);
  }
#pragma unroll
  for (int o = U / 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

}  // namespace dcdg
