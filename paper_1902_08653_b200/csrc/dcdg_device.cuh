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
  unsigned long long epoch;           // batch epoch written to the owners' flags
  int flag_slot;                      // xchg_cta_done publishes to slot flag_slot (+ rank if per_rank)
  int per_rank;
  long long buf_bytes;                // bytes of one parity buffer
  long long sig_off;                  // offset of the sigma2 region inside a parity buffer
  int world, rank;
  int S_own;                          // subcarriers owned per rank
  int C_local, c0, C_total, U;
  int esz;                            // bytes per complex of x (8 fp32, 4 fp16)
  int parity;
};

// Destination of problem p's estimate (p = s*C_local + c, s global over the batch).
// (P = S*C_local < 2^31 is checked on the host: 32-bit index math.)
__device__ __forceinline__ unsigned char* xchg_x_dst(const XMap& m, int p) {
  const int s = p / m.C_local;
  const int c = p - s * m.C_local;
  const int owner = s / m.S_own;
  const int s_in = s - owner * m.S_own;
  return m.win[owner] + kXchgFlagBytes + m.parity * m.buf_bytes +
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
      for (int q = 0; q < m.world; ++q)
        st_release_sys(reinterpret_cast<unsigned long long*>(m.win[q]) + slot, m.epoch);
      *m.counter = 0u;  // next launch on this stream starts from zero
    }
  }
}

}  // namespace dcdg
