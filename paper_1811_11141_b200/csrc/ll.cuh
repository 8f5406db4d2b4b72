// ll.cuh -- push-based low-latency one-shot for small, startup-dominated groups
// (same result as ring_allreduce, allreduce_net.py:370-411, for the group's bucket).
//
// The messages MG-WFBP creates by merging are small: their cost is the startup `a`
// (paper Eq. 8), not bandwidth.  The pull one-shot pays a flag round trip (signal +
// poll) and then a remote-read round trip.  Here every rank *pushes* its packed
// values into every peer's LL receive area as 8-byte words (epoch << 32 | fp32 bits):
// a word is data and flag at once (single-copy atomic 64-bit store), so a receiver
// only polls its own local memory and folds as soon as all N words of an element
// carry the current epoch.  One NVLink crossing, no separate barrier.  Twice the bytes
// on the wire, which is irrelevant at these sizes.
//
// Fold order is the reference's (start at the element's `_segments` segment), so the
// result is bit-identical to K2/K3.  Disagreement: CTA 0 of every rank also pushes a
// header (epoch << 32 | collective_tag) and checks every peer's header before folding;
// a mismatch raises the sticky abort flag that every poll loop watches.
#pragma once

#include "fused.cuh"

namespace mgw {

constexpr int64_t kLLMaxElems = kLLElems;  // per rank per parity (1 MB of fp32 payload)

struct LLArgs {
  FusedArgs f;                   // rows (layer tensors), scale, comm pointers, epochs
  uint64_t* ll[kMaxRanks];       // per-rank LL receive area base: [2 parity][kMaxRanks src][kLLMaxElems]
  uint64_t* hdr[kMaxRanks];      // per-rank header words: [2 parity][... src]; a communicator
                                 // points them at its arrive barrier flags of CTA 0, so an LL
                                 // header and a barrier flag of a rank running another kernel
                                 // meet in the same word and the tag check sees the mismatch
  int64_t hdr_stride;            // words from parity 0 to parity 1 of hdr
};

__device__ __forceinline__ void st_relaxed_sys_v2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t a) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void ld_relaxed_sys_v2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// Re-poll a pair of words until both carry `epoch`.  Bounded; watches the abort flag and
// the source's header word `hdr`: a peer running a different collective (length, kernel,
// group ...) never sends these words, and its header tells us so without the timeout.
__device__ __forceinline__ void ll_wait2(const uint64_t* p, const uint64_t* hdr, uint32_t epoch, const ArArgs& a,
                                         int& status, uint64_t& w0, uint64_t& w1) {
  const uint64_t start = global_ns();
  for (uint32_t spin = 0;; ++spin) {
    ld_relaxed_sys_v2(p, w0, w1);
    if ((uint32_t)(w0 >> 32) == epoch && (uint32_t)(w1 >> 32) == epoch) return;
    if ((spin & 31) == 31) {
      const uint64_t h = ld_relaxed_sys_u64(hdr);
      if ((uint32_t)(h >> 32) == epoch && (uint32_t)h != a.tag) {
        status = MGW_DEV_MISMATCH;
        return;
      }
      if (load_relaxed_sys32(a.abort_flag[a.rank]) != 0u) {
        status = MGW_DEV_PEER_ABORT;
        return;
      }
      if (global_ns() - start > a.timeout_ns) {
        status = MGW_DEV_TIMEOUT;
        return;
      }
    }
  }
}

// error word + abort flags (a peer abort is only recorded)
__device__ __forceinline__ void ll_report(const ArArgs& a, int status) {
  atomicCAS(a.err, 0, status);
  if (status != MGW_DEV_PEER_ABORT)
    for (int r = 0; r < a.world; ++r) store_release_sys32(a.abort_flag[r], 1u);
}

// CTA 0's threads < N wait for every peer's header of this epoch and compare its tag (the
// peer's length / kernel / dtype / group); the other CTAs pass straight through.  Returns
// the CTA-uniform status; reports errors.
__device__ __forceinline__ int ll_header_check(const LLArgs& l, uint32_t epoch, int parity, bool active, int status,
                                               int* s_status) {
  const ArArgs& a = l.f.ar;
  const int me = a.rank;
  if (threadIdx.x == 0) *s_status = MGW_DEV_OK;
  __syncthreads();
  if (status != MGW_DEV_OK) atomicCAS(s_status, 0, status);  // a fold thread's error
  if (active && status == MGW_DEV_OK && threadIdx.x < a.world) {
    const uint64_t* p = l.hdr[me] + parity * l.hdr_stride + threadIdx.x;
    uint64_t v = ld_relaxed_sys_u64(p);
    const uint64_t start = global_ns();
    int st = MGW_DEV_OK;
    for (uint32_t spin = 0; (uint32_t)(v >> 32) != epoch; ++spin) {
      if ((spin & 31) == 31) {
        if (load_relaxed_sys32(a.abort_flag[me]) != 0u) {
          st = MGW_DEV_PEER_ABORT;
          break;
        }
        if (global_ns() - start > a.timeout_ns) {
          st = MGW_DEV_TIMEOUT;
          break;
        }
      }
      v = ld_relaxed_sys_u64(p);
    }
    if (st == MGW_DEV_OK && (uint32_t)v != a.tag) st = MGW_DEV_MISMATCH;
    if (st != MGW_DEV_OK) atomicCAS(s_status, 0, st);
  }
  __syncthreads();
  const int out = *s_status;
  if (out != MGW_DEV_OK && threadIdx.x == 0) ll_report(a, out);
  return out;
}

__device__ __forceinline__ uint64_t ll_word(uint32_t epoch, float x) {
  return ((uint64_t)epoch << 32) | (uint64_t)__float_as_uint(x);
}

__device__ __forceinline__ float* ll_tensor(const FusedArgs& f, int& k, int64_t e) {
  const Row r = walk_row(f, k, e);
  return r.ptr + (e - r.offset);
}

template <int N>
__device__ __forceinline__ void ll_oneshot_body(const LLArgs& l, const int cta, const int ctas) {
  const FusedArgs& f = l.f;
  const ArArgs& a = f.ar;
  grid_dep_wait();
  stamp_enter(a.stamp);
  __shared__ int64_t s_end[kMaxRanks];
  __shared__ int s_status;
  const uint32_t epoch = load_volatile32(a.state) + 1u;
  const int parity = (int)(epoch & 1u);
  const int me = a.rank;
  const int64_t n = a.n;
  if (threadIdx.x < N) {
    const int t = threadIdx.x;
    const int64_t q = n / N, r = n % N;
    s_end[t] = (int64_t)(t + 1) * q + (t + 1 < r ? t + 1 : r);
  }
  if (threadIdx.x == 0) s_status = MGW_DEV_OK;
  // header: (epoch, n) to every rank (CTA 0).  kSkipPack / kSkipPhase1 split the push
  // and the fold into separate launches (emulated ranks on one device, tests only).
  const bool do_push = !(a.flags & kSkipPack), do_fold = !(a.flags & kSkipPhase1);
  if (do_push && cta == 0 && threadIdx.x < N)
    st_relaxed_sys_u64(l.hdr[threadIdx.x] + parity * l.hdr_stride + me, ((uint64_t)epoch << 32) | a.tag);
  __syncthreads();

  // element pairs of this CTA: [p0, p1) (pair j = elements 2j, 2j+1)
  const int64_t pairs = (n + 1) >> 1;
  const int64_t per = (pairs + ctas - 1) / ctas;
  const int64_t p0 = (int64_t)cta * per;
  const int64_t p1 = p0 + per < pairs ? p0 + per : pairs;
  const float scale = f.scale;
  const size_t my_off = ((size_t)parity * kMaxRanks + me) * kLLMaxElems;

  phase_mark(a, 0, cta);
  // 1. pack and push: my two elements of each pair to every rank's LL area
  int k = 0;
  if (p0 < p1) k = fused_row_covering(f, (p0 + threadIdx.x) * 2 < n ? (p0 + threadIdx.x) * 2 : 0);
  for (int64_t j = p0 + threadIdx.x; do_push && j < p1; j += kThreads) {
    const int64_t e = 2 * j;
    float x0 = *ll_tensor(f, k, e);
    float x1 = e + 1 < n ? *ll_tensor(f, k, e + 1) : 0.f;
    if (scale != 1.0f) {
      x0 = __fmul_rn(x0, scale);
      x1 = __fmul_rn(x1, scale);
    }
    const uint64_t w0 = ll_word(epoch, x0), w1 = ll_word(epoch, x1);
#pragma unroll
    for (int r = 0; r < N; ++r) st_relaxed_sys_v2(l.ll[r] + my_off + e, w0, w1);
  }

  phase_mark(a, 1, cta);
  // 2. CTA 0 checks every peer's header first (length / collective agreement); measured:
  //    checking after the fold was slower (512 threads polling data words that are still in
  //    flight instead of N threads polling headers)
  int status = do_fold ? ll_header_check(l, epoch, parity, cta == 0, MGW_DEV_OK, &s_status) : MGW_DEV_OK;
  phase_mark(a, 2, cta);

  // 3. fold every element of my pairs from the N local LL areas, write the tensors.
  //    The N sources' words of a pair are fetched as N independent 16-B loads issued
  //    back to back (one memory latency, not 2N serial ones); only words that do not yet
  //    carry this epoch are polled again.
  const uint64_t* hdr_mine = l.hdr[me] + parity * l.hdr_stride;
  if (do_fold && status == MGW_DEV_OK) {
    const uint64_t* base = l.ll[me] + (size_t)parity * kMaxRanks * kLLMaxElems;
    int seg = 0;
    k = 0;
    if (p0 < p1) k = fused_row_covering(f, (p0 + threadIdx.x) * 2 < n ? (p0 + threadIdx.x) * 2 : 0);
    for (int64_t j = p0 + threadIdx.x; j < p1 && status == MGW_DEV_OK; j += kThreads) {
      const int64_t e = 2 * j;
      uint64_t w0[N], w1[N];
#pragma unroll
      for (int src = 0; src < N; ++src) ld_relaxed_sys_v2(base + (size_t)src * kLLMaxElems + e, w0[src], w1[src]);
#pragma unroll
      for (int src = 0; src < N; ++src) {
        if ((uint32_t)(w0[src] >> 32) != epoch || (uint32_t)(w1[src] >> 32) != epoch)
          ll_wait2(base + (size_t)src * kLLMaxElems + e, hdr_mine + src, epoch, a, status, w0[src], w1[src]);
      }
      if (status != MGW_DEV_OK) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t eh = e + h;
        if (eh >= n) break;
        seg = advance_segment(seg, eh, s_end);
        float acc = 0.f;
#pragma unroll
        for (int kk = 0; kk < N; ++kk) {
          int src = seg + kk;
          src = src >= N ? src - N : src;
          // select the word of source `src` without dynamic register indexing
          uint64_t w = 0;
#pragma unroll
          for (int q = 0; q < N; ++q) w = q == src ? (h ? w1[q] : w0[q]) : w;
          const float x = __uint_as_float((uint32_t)w);
          acc = kk == 0 ? x : __fadd_rn(acc, x);
        }
        *ll_tensor(f, k, eh) = acc;
      }
    }
  }
  if (status != MGW_DEV_OK && status != s_status) ll_report(a, status);  // a fold thread's own error
  phase_mark(a, 3, cta);
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(ll_oneshot, LLArgs)

}  // namespace mgw
