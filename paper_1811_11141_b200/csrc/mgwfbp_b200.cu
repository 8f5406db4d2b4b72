// mgwfbp_b200.cu -- sm_100a kernels and C ABI of the MG-WFBP merged-gradient data path.
//
//   K1 pack+scale   gather a merge group's layer gradients into one contiguous
//                   bucket (layer `high` at offset 0; allreduce_net.py:495-509)
//   K2 one-shot     every rank pulls all N peer buckets over NVLink (CUDA IPC)
//                   and folds them in the reference ring's per-element order
//   K3 two-shot     reduce-scatter of the rank's own `_segments` slice, then
//                   all-gather of the peers' reduced slices, same fold order
//   K4 unpack       scatter the reduced bucket back to the layer tensors
//   K5 spin         simulated backward on the compute stream (%globaltimer)
//
// Fold order (bit-exact with allreduce_net.py:360-411): element e of the bucket
// lies in segment s = seg(e) of `_segments(n, N)`; the ring accumulates it as
// ((x_s + x_{s+1}) + x_{s+2}) + ... + x_{s+N-1} (ranks mod N).  Both K2 and K3
// reproduce exactly that left fold with __fadd_rn (no contraction).
//
// Synchronisation: per-block flag barriers in the IPC control area of every
// rank (system-scope release/acquire), epochs taken from a device-side call
// counter so the whole iteration can be replayed from a CUDA graph, bounded
// spins that set a device error word (-> ProtocolError on the host).

#include "mgwfbp_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

// ------------------------------------------------------------------ errors

thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define MGW_CUDA(call)                                                                            \
  do {                                                                                            \
    cudaError_t err_ = (call);                                                                    \
    if (err_ != cudaSuccess)                                                                      \
      return set_error(MGW_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(err_), __FILE__, __LINE__); \
  } while (0)

#define MGW_CHECK_LAUNCH()                                                                        \
  do {                                                                                            \
    cudaError_t err_ = cudaGetLastError();                                                        \
    if (err_ != cudaSuccess)                                                                      \
      return set_error(MGW_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(err_), __FILE__, __LINE__); \
  } while (0)

// --------------------------------------------------------------- constants

constexpr int kMaxRanks = MGW_MAX_RANKS;
constexpr int kMaxBlocks = 256;          // per-block barrier slots per parity
constexpr int kThreads = 512;            // threads per CTA for every bulk kernel
constexpr int64_t kTile = 16384;         // pack/unpack tile: 64 KB of bucket per CTA step
constexpr int kSMs = 148;

// IPC region layout (per rank):  [arrive | mid | abort | pad] [slot 0] [slot 1]
constexpr size_t kFlagsPerParity = (size_t)kMaxBlocks * kMaxRanks;
constexpr size_t kArriveOff = 0;
constexpr size_t kMidOff = kArriveOff + 2 * kFlagsPerParity * sizeof(uint64_t);
constexpr size_t kAbortOff = kMidOff + 2 * kFlagsPerParity * sizeof(uint64_t);
constexpr size_t kCtrlBytes = 131072;
static_assert(kAbortOff + 256 <= kCtrlBytes, "control area overflow");

enum : int { kNoBarrier = 1, kSkipPhase1 = 2, kSkipPhase2 = 4 };

struct Row {  // identical layout to mgw_tensor_desc
  float* ptr;
  int64_t count;
  int64_t offset;
};
static_assert(sizeof(Row) == sizeof(mgw_tensor_desc), "Row must mirror mgw_tensor_desc");

// ------------------------------------------------------------ device utils

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void store_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void store_relaxed_sys32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t load_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t load_acquire_sys32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t load_volatile32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Kernel span stamps: every CTA folds its entry time into stamp[0] (min) and its
// exit time into stamp[1] (max), so [stamp[0], stamp[1]] is the kernel's execution
// span without the ~6.5 us an event record pair costs inside a CUDA graph.
__device__ __forceinline__ void stamp_enter(uint64_t* stamp) {
  if (stamp != nullptr && threadIdx.x == 0) atomicMin(reinterpret_cast<unsigned long long*>(stamp), (unsigned long long)global_ns());
}

__device__ __forceinline__ void stamp_exit(uint64_t* stamp) {
  if (stamp != nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(stamp + 1), (unsigned long long)global_ns());
  }
}

__device__ __forceinline__ float4 fadd4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

__device__ __forceinline__ float4 fmul4(float4 a, float s) {
  return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}

// ======================================================== K1 / K4: pack, unpack
//
// The bucket of a group is tiled in kTile-element steps; a CTA binary-searches
// the first descriptor row overlapping its tile and walks the rows it covers.
// Each (row, tile) span is copied block-cooperatively: 128-bit accesses when
// tensor and bucket addresses agree modulo 16 B (true for every torch
// allocation and every profile whose layer sizes are multiples of 4), scalar
// coalesced accesses otherwise.

enum class RowOp { kPack, kUnpack, kFill, kCheck };

template <RowOp kOp, bool kScale>
__device__ __forceinline__ void span_op(float* __restrict__ tensor, float* __restrict__ bucket, int64_t len,
                                        float scale, float value, unsigned long long* mismatches) {
  const int t = threadIdx.x;
  const int nt = blockDim.x;
  if constexpr (kOp == RowOp::kFill) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(tensor);
    int64_t head = (int64_t)(((16 - (a & 15)) & 15) >> 2);
    head = head < len ? head : len;
    for (int64_t i = t; i < head; i += nt) tensor[i] = value;
    float4* d4 = reinterpret_cast<float4*>(tensor + head);
    const int64_t nv = (len - head) >> 2;
    const float4 v4 = make_float4(value, value, value, value);
    for (int64_t i = t; i < nv; i += nt) d4[i] = v4;
    for (int64_t i = head + (nv << 2) + t; i < len; i += nt) tensor[i] = value;
  } else if constexpr (kOp == RowOp::kCheck) {
    unsigned long long bad = 0;
    for (int64_t i = t; i < len; i += nt) bad += (tensor[i] != value);
    if (bad) atomicAdd(mismatches, bad);
  } else {
    const float* __restrict__ src = (kOp == RowOp::kUnpack) ? bucket : tensor;
    float* __restrict__ dst = (kOp == RowOp::kUnpack) ? tensor : bucket;
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
    const uintptr_t da = reinterpret_cast<uintptr_t>(dst);
    if (((sa ^ da) & 15) == 0) {
      int64_t head = (int64_t)(((16 - (da & 15)) & 15) >> 2);
      head = head < len ? head : len;
      for (int64_t i = t; i < head; i += nt) dst[i] = kScale ? __fmul_rn(src[i], scale) : src[i];
      const float4* __restrict__ s4 = reinterpret_cast<const float4*>(src + head);
      float4* __restrict__ d4 = reinterpret_cast<float4*>(dst + head);
      const int64_t nv = (len - head) >> 2;
      int64_t i = t;
      for (; i + 3 * nt < nv; i += 4 * nt) {
        float4 r0 = s4[i], r1 = s4[i + nt], r2 = s4[i + 2 * nt], r3 = s4[i + 3 * nt];
        if (kScale) {
          r0 = fmul4(r0, scale);
          r1 = fmul4(r1, scale);
          r2 = fmul4(r2, scale);
          r3 = fmul4(r3, scale);
        }
        d4[i] = r0;
        d4[i + nt] = r1;
        d4[i + 2 * nt] = r2;
        d4[i + 3 * nt] = r3;
      }
      for (; i < nv; i += nt) d4[i] = kScale ? fmul4(s4[i], scale) : s4[i];
      for (int64_t j = head + (nv << 2) + t; j < len; j += nt) dst[j] = kScale ? __fmul_rn(src[j], scale) : src[j];
    } else {
      for (int64_t i = t; i < len; i += nt) dst[i] = kScale ? __fmul_rn(src[i], scale) : src[i];
    }
  }
}

__device__ __forceinline__ int first_row_covering(const Row* __restrict__ rows, int n, int64_t e) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rows[mid].offset + rows[mid].count > e)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

template <RowOp kOp, bool kScale>
__global__ void __launch_bounds__(kThreads) rows_kernel(const Row* __restrict__ rows, int n_rows, float* bucket,
                                                        int64_t total, float scale, const float* __restrict__ values,
                                                        const uint32_t* calls, int64_t slot_stride_elems,
                                                        unsigned long long* mismatches, uint64_t* stamp) {
  stamp_enter(stamp);
  if (calls != nullptr) {
    // epoch of the collective this pack feeds = completed calls + 1
    const uint32_t epoch = load_volatile32(calls) + 1u;
    bucket += (int64_t)(epoch & 1u) * slot_stride_elems;
  }
  for (int64_t t0 = (int64_t)blockIdx.x * kTile; t0 < total; t0 += (int64_t)gridDim.x * kTile) {
    const int64_t t1 = t0 + kTile < total ? t0 + kTile : total;
    for (int k = first_row_covering(rows, n_rows, t0); k < n_rows; ++k) {
      const Row r = rows[k];
      if (r.offset >= t1) break;
      const int64_t lo = r.offset > t0 ? r.offset : t0;
      const int64_t hi = (r.offset + r.count) < t1 ? (r.offset + r.count) : t1;
      if (hi <= lo) continue;
      const float v = values ? values[k] : 0.f;
      span_op<kOp, kScale>(r.ptr + (lo - r.offset), bucket + lo, hi - lo, scale, v, mismatches);
    }
  }
  stamp_exit(stamp);
}

int rows_grid(int64_t total) {
  int64_t tiles = (total + kTile - 1) / kTile;
  int64_t cap = (int64_t)kSMs * 4;
  return (int)std::max<int64_t>(1, std::min(tiles, cap));
}

template <RowOp kOp>
int launch_rows(const void* table, int n, float* bucket, int64_t total, float scale, const float* values,
                const uint32_t* calls, int64_t slot_stride_elems, unsigned long long* mismatches,
                cudaStream_t stream, uint64_t* stamp = nullptr) {
  if (total <= 0 || n <= 0) return MGW_OK;
  const Row* rows = static_cast<const Row*>(table);
  const int grid = rows_grid(total);
  if (kOp == RowOp::kPack && scale != 1.0f)
    rows_kernel<kOp, true><<<grid, kThreads, 0, stream>>>(rows, n, bucket, total, scale, values, calls,
                                                          slot_stride_elems, mismatches, stamp);
  else
    rows_kernel<kOp, false><<<grid, kThreads, 0, stream>>>(rows, n, bucket, total, scale, values, calls,
                                                           slot_stride_elems, mismatches, stamp);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

// ============================================================ K5: spin kernels

__global__ void spin_relative_kernel(int64_t ns) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = global_ns();
  while ((int64_t)(global_ns() - t0) < ns) __nanosleep(128);
}

__global__ void stamps_reset_kernel(uint64_t* stamps, int pairs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += gridDim.x * blockDim.x) {
    stamps[2 * i] = ~0ull;
    stamps[2 * i + 1] = 0ull;
  }
}

__global__ void clock_mark_kernel(uint64_t* clock) {
  if (threadIdx.x == 0) *clock = global_ns();
}

__global__ void spin_until_kernel(const uint64_t* clock, int64_t deadline_ns) {
  if (threadIdx.x != 0) return;
  const uint64_t until = *reinterpret_cast<const volatile uint64_t*>(clock) + (uint64_t)deadline_ns;
  while (global_ns() < until) __nanosleep(128);
}

// ====================================================== K2 / K3: all-reduce

struct ArArgs {
  char* slot[kMaxRanks];       // slot-0 base of every rank (peer mapped; own at [rank])
  uint64_t* arrive[kMaxRanks]; // per-rank entry-barrier flags  [2][kMaxBlocks][kMaxRanks]
  uint64_t* mid[kMaxRanks];    // per-rank mid-barrier flags    [2][kMaxBlocks][kMaxRanks]
  uint32_t* abort_flag[kMaxRanks];
  float* out[kMaxRanks];       // result buffer (real mode uses out[rank])
  uint32_t* state;             // local device [completed calls, finished CTAs]; null = no epochs
  int* err;                    // local device error word
  uint64_t* stamp;             // optional kernel span stamps [2]
  int64_t slot_stride;         // bytes from slot 0 to slot 1
  int64_t n;                   // elements
  uint64_t timeout_ns;
  int rank;
  int world;
  int flags;
};

// segment of bucket element e under _segments(n, N): q, r = divmod(n, N); the
// first r segments hold q+1 elements (allreduce_net.py:360-367)
__device__ __forceinline__ int segment_of(int64_t e, int64_t q, int64_t r) {
  const int64_t big = r * (q + 1);
  return e < big ? (int)(e / (q + 1)) : (int)(r + (e - big) / q);
}

__device__ __forceinline__ void segment_range(int s, int64_t q, int64_t r, int64_t& off, int64_t& len) {
  len = q + (s < r ? 1 : 0);
  off = (int64_t)s * q + (s < r ? s : r);
}

// Work a CTA owns inside one segment: a scalar head (CTA 0), a slice of the
// 16-B aligned vector body, and a scalar tail (last CTA).  Deterministic in
// (segment, cta, grid) so a CTA on another rank can find what this CTA wrote.
struct Chunk {
  int64_t v0, v1;  // vector indices (4 floats each) into the bucket
  int64_t h0, h1;  // scalar head elements
  int64_t t0, t1;  // scalar tail elements
};

__device__ __forceinline__ Chunk chunk_of(int64_t off, int64_t len, int b, int G) {
  Chunk c{0, 0, 0, 0, 0, 0};
  const int64_t end = off + len;
  const int64_t a0 = (off + 3) & ~int64_t(3);
  const int64_t a1 = end & ~int64_t(3);
  if (a0 >= a1) {
    if (b == 0) {
      c.h0 = off;
      c.h1 = end;
    }
    return c;
  }
  if (b == 0) {
    c.h0 = off;
    c.h1 = a0;
  }
  if (b == G - 1) {
    c.t0 = a1;
    c.t1 = end;
  }
  const int64_t nv = (a1 - a0) >> 2;
  const int64_t per = (nv + G - 1) / G;
  const int64_t lo = (int64_t)b * per < nv ? (int64_t)b * per : nv;
  const int64_t hi = (int64_t)(b + 1) * per < nv ? (int64_t)(b + 1) * per : nv;
  c.v0 = (a0 >> 2) + lo;
  c.v1 = (a0 >> 2) + hi;
  return c;
}

// Per-CTA barrier across ranks.  Thread t < world signals rank t and waits for
// rank t's matching CTA.  Flags carry (epoch << 32 | n mod 2^32) so a length
// disagreement is detected at the barrier (replaces the frame header check,
// allreduce_net.py:342-347).  Parity-split slots keep epoch e's flags intact
// until every rank has passed e.
__device__ int cta_barrier(uint64_t* const* flags, int parity, uint32_t epoch, uint32_t tag, const ArArgs& a) {
  __shared__ int s_status;
  if (threadIdx.x == 0) s_status = 0;
  __syncthreads();
  const int t = threadIdx.x;
  if (t < a.world) {
    const size_t base = ((size_t)parity * kMaxBlocks + blockIdx.x) * kMaxRanks;
    __threadfence_system();
    store_relaxed_sys(flags[t] + base + a.rank, ((uint64_t)epoch << 32) | tag);
    const uint64_t* mine = flags[a.rank] + base + t;
    const uint64_t start = global_ns();
    int status = MGW_DEV_OK;
    for (;;) {
      const uint64_t v = load_acquire_sys(mine);
      if ((uint32_t)(v >> 32) == epoch) {
        if ((uint32_t)v != tag) status = MGW_DEV_LENGTH_MISMATCH;
        break;
      }
      if (load_acquire_sys32(a.abort_flag[a.rank]) != 0u) {
        status = MGW_DEV_PEER_ABORT;
        break;
      }
      if (global_ns() - start > a.timeout_ns) {
        status = MGW_DEV_TIMEOUT;
        break;
      }
    }
    __threadfence_system();
    if (status != MGW_DEV_OK) atomicCAS(&s_status, 0, status);
  }
  __syncthreads();
  const int status = s_status;
  if (status != MGW_DEV_OK && threadIdx.x == 0) {
    atomicCAS(a.err, 0, status);
    if (status != MGW_DEV_PEER_ABORT)
      for (int r = 0; r < a.world; ++r) store_relaxed_sys32(a.abort_flag[r], 1u);
  }
  return status;
}

// Last CTA out advances the call counter (epochs and slot parity come from it).
__device__ __forceinline__ void finish_call(const ArArgs& a) {
  stamp_exit(a.stamp);
  if (a.state == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t ticket = atomicAdd(&a.state[1], 1u);
    if (ticket == gridDim.x - 1) {
      a.state[1] = 0u;
      __threadfence();
      atomicAdd(&a.state[0], 1u);
    }
  }
}

template <int N>
__device__ __forceinline__ float4 fold4(const float* const* in, int s, int64_t e) {
  float4 x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int src = s + k;
    src = src >= N ? src - N : src;
    x[k] = __ldcg(reinterpret_cast<const float4*>(in[src] + e));
  }
  float4 acc = x[0];
#pragma unroll
  for (int k = 1; k < N; ++k) acc = fadd4(acc, x[k]);
  return acc;
}

template <int N>
__device__ __forceinline__ float fold1(const float* const* in, int s, int64_t e) {
  float x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int src = s + k;
    src = src >= N ? src - N : src;
    x[k] = __ldcg(in[src] + e);
  }
  float acc = x[0];
#pragma unroll
  for (int k = 1; k < N; ++k) acc = __fadd_rn(acc, x[k]);
  return acc;
}

template <int N>
__device__ __forceinline__ void load_slots(const ArArgs& a, int parity, const float** s_in) {
  if (threadIdx.x < N) s_in[threadIdx.x] = reinterpret_cast<const float*>(a.slot[threadIdx.x] + (int64_t)parity * a.slot_stride);
  __syncthreads();
}

// K2: every rank reads all N buckets and writes the full reduced vector.
template <int N>
__global__ void __launch_bounds__(kThreads) oneshot_kernel(ArArgs a) {
  __shared__ const float* s_in[kMaxRanks];
  stamp_enter(a.stamp);
  uint32_t epoch = 0;
  if (a.state != nullptr) epoch = load_volatile32(a.state) + 1u;
  const int parity = (int)(epoch & 1u);
  load_slots<N>(a, parity, s_in);
  int status = MGW_DEV_OK;
  if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, (uint32_t)a.n, a);
  if (status == MGW_DEV_OK) {
    float* __restrict__ out = a.out[a.rank];
    const int64_t n = a.n, q = n / N, r = n % N;
    const int64_t nv = n >> 2;
    const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
    const int64_t v0 = (int64_t)blockIdx.x * per;
    const int64_t v1 = v0 + per < nv ? v0 + per : nv;
    int64_t v = v0 + threadIdx.x;
    for (; v + blockDim.x < v1; v += 2 * blockDim.x) {
      const int64_t e0 = v << 2, e1 = (v + blockDim.x) << 2;
      const int s0 = segment_of(e0, q, r), s1 = segment_of(e1, q, r);
      if (s0 == segment_of(e0 + 3, q, r) && s1 == segment_of(e1 + 3, q, r)) {
        const float4 y0 = fold4<N>(s_in, s0, e0);
        const float4 y1 = fold4<N>(s_in, s1, e1);
        *reinterpret_cast<float4*>(out + e0) = y0;
        *reinterpret_cast<float4*>(out + e1) = y1;
      } else {
        for (int j = 0; j < 4; ++j) out[e0 + j] = fold1<N>(s_in, segment_of(e0 + j, q, r), e0 + j);
        for (int j = 0; j < 4; ++j) out[e1 + j] = fold1<N>(s_in, segment_of(e1 + j, q, r), e1 + j);
      }
    }
    for (; v < v1; v += blockDim.x) {
      const int64_t e = v << 2;
      const int s = segment_of(e, q, r);
      if (s == segment_of(e + 3, q, r)) {
        *reinterpret_cast<float4*>(out + e) = fold4<N>(s_in, s, e);
      } else {
        for (int j = 0; j < 4; ++j) out[e + j] = fold1<N>(s_in, segment_of(e + j, q, r), e + j);
      }
    }
    if (blockIdx.x == gridDim.x - 1)
      for (int64_t e = (nv << 2) + threadIdx.x; e < n; e += blockDim.x) out[e] = fold1<N>(s_in, segment_of(e, q, r), e);
  }
  finish_call(a);
}

// K3: reduce-scatter own segment (in place in the own slot, copy to out), then
// all-gather the peers' reduced segments into out.
template <int N>
__global__ void __launch_bounds__(kThreads) twoshot_kernel(ArArgs a) {
  __shared__ const float* s_in[kMaxRanks];
  stamp_enter(a.stamp);
  uint32_t epoch = 0;
  if (a.state != nullptr) epoch = load_volatile32(a.state) + 1u;
  const int parity = (int)(epoch & 1u);
  load_slots<N>(a, parity, s_in);
  const int me = a.rank;
  const int b = blockIdx.x, G = gridDim.x;
  const int64_t n = a.n, q = n / N, r = n % N;
  float* __restrict__ out = a.out[me];
  float* own = const_cast<float*>(s_in[me]);
  const bool copy_out = out != own;
  int status = MGW_DEV_OK;

  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, (uint32_t)a.n, a);
    if (status == MGW_DEV_OK) {
      int64_t off, len;
      segment_range(me, q, r, off, len);
      const Chunk c = chunk_of(off, len, b, G);
      for (int64_t e = c.h0 + threadIdx.x; e < c.h1; e += blockDim.x) {
        const float y = fold1<N>(s_in, me, e);
        own[e] = y;
        if (copy_out) out[e] = y;
      }
      int64_t v = c.v0 + threadIdx.x;
      for (; v + blockDim.x < c.v1; v += 2 * blockDim.x) {
        const int64_t e0 = v << 2, e1 = (v + blockDim.x) << 2;
        const float4 y0 = fold4<N>(s_in, me, e0);
        const float4 y1 = fold4<N>(s_in, me, e1);
        *reinterpret_cast<float4*>(own + e0) = y0;
        *reinterpret_cast<float4*>(own + e1) = y1;
        if (copy_out) {
          *reinterpret_cast<float4*>(out + e0) = y0;
          *reinterpret_cast<float4*>(out + e1) = y1;
        }
      }
      for (; v < c.v1; v += blockDim.x) {
        const int64_t e = v << 2;
        const float4 y = fold4<N>(s_in, me, e);
        *reinterpret_cast<float4*>(own + e) = y;
        if (copy_out) *reinterpret_cast<float4*>(out + e) = y;
      }
      for (int64_t e = c.t0 + threadIdx.x; e < c.t1; e += blockDim.x) {
        const float y = fold1<N>(s_in, me, e);
        own[e] = y;
        if (copy_out) out[e] = y;
      }
    }
  }

  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase2)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.mid, parity, epoch, (uint32_t)a.n, a);
    if (status == MGW_DEV_OK) {
#pragma unroll 1
      for (int k = 1; k < N; ++k) {
        int s = me + k;
        s = s >= N ? s - N : s;
        int64_t off, len;
        segment_range(s, q, r, off, len);
        const Chunk c = chunk_of(off, len, b, G);
        const float* __restrict__ src = s_in[s];
        for (int64_t e = c.h0 + threadIdx.x; e < c.h1; e += blockDim.x) out[e] = __ldcg(src + e);
        const float4* __restrict__ s4 = reinterpret_cast<const float4*>(src);
        float4* __restrict__ d4 = reinterpret_cast<float4*>(out);
        const int64_t step = blockDim.x;
        int64_t v = c.v0 + threadIdx.x;
        for (; v + 3 * step < c.v1; v += 4 * step) {
          const float4 x0 = __ldcg(s4 + v), x1 = __ldcg(s4 + v + step), x2 = __ldcg(s4 + v + 2 * step),
                       x3 = __ldcg(s4 + v + 3 * step);
          d4[v] = x0;
          d4[v + step] = x1;
          d4[v + 2 * step] = x2;
          d4[v + 3 * step] = x3;
        }
        for (; v < c.v1; v += step) d4[v] = __ldcg(s4 + v);
        for (int64_t e = c.t0 + threadIdx.x; e < c.t1; e += blockDim.x) out[e] = __ldcg(src + e);
      }
    }
  }
  finish_call(a);
}

int grid_for(int64_t vectors_per_cta_work, int64_t min_per_cta, int max_ctas) {
  int64_t g = (vectors_per_cta_work + min_per_cta - 1) / min_per_cta;
  g = std::max<int64_t>(1, std::min<int64_t>(g, max_ctas));
  return (int)g;
}

int launch_allreduce(const ArArgs& a, int algo, int max_ctas, cudaStream_t stream) {
  const int64_t nv = a.n >> 2;
  max_ctas = std::min(max_ctas, kMaxBlocks);  // one barrier flag slot per CTA
  if (algo == MGW_ALGO_ONESHOT) {
    const int grid = grid_for(nv, 1024, max_ctas);
#define MGW_ONESHOT_CASE(NN) \
  case NN:                   \
    oneshot_kernel<NN><<<grid, kThreads, 0, stream>>>(a); \
    break;
    switch (a.world) {
      MGW_ONESHOT_CASE(1)
      MGW_ONESHOT_CASE(2)
      MGW_ONESHOT_CASE(3)
      MGW_ONESHOT_CASE(4)
      MGW_ONESHOT_CASE(5)
      MGW_ONESHOT_CASE(6)
      MGW_ONESHOT_CASE(7)
      MGW_ONESHOT_CASE(8)
      default:
        return set_error(MGW_EINVAL, "world %d outside 1..%d", a.world, kMaxRanks);
    }
#undef MGW_ONESHOT_CASE
  } else {
    const int grid = grid_for(nv / std::max(1, a.world), 1024, max_ctas);
#define MGW_TWOSHOT_CASE(NN) \
  case NN:                   \
    twoshot_kernel<NN><<<grid, kThreads, 0, stream>>>(a); \
    break;
    switch (a.world) {
      MGW_TWOSHOT_CASE(1)
      MGW_TWOSHOT_CASE(2)
      MGW_TWOSHOT_CASE(3)
      MGW_TWOSHOT_CASE(4)
      MGW_TWOSHOT_CASE(5)
      MGW_TWOSHOT_CASE(6)
      MGW_TWOSHOT_CASE(7)
      MGW_TWOSHOT_CASE(8)
      default:
        return set_error(MGW_EINVAL, "world %d outside 1..%d", a.world, kMaxRanks);
    }
#undef MGW_TWOSHOT_CASE
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

}  // namespace

// =================================================================== C ABI

struct mgw_comm {
  int rank = 0;
  int world = 1;
  int device = 0;
  int64_t capacity = 0;    // bytes per slot as requested
  int64_t slot_bytes = 0;  // rounded to 256 B
  char* region = nullptr;  // own IPC region
  char* peer[kMaxRanks] = {};
  bool peers_open = false;
  uint32_t* state = nullptr;  // [calls, finished]
  int* err = nullptr;
  float* result = nullptr;
  uint64_t timeout_ns = 30ull * 1000000000ull;
  int64_t oneshot_max_bytes = 1 << 20;
  int max_ctas = kSMs;
};

struct mgw_sched {
  mgw_comm* comm = nullptr;
  int world = 1;
  std::vector<Row> rows;
  Row* d_rows = nullptr;
  std::vector<mgw_group> groups;
  float* d_fill = nullptr;
  float* local_bucket = nullptr;  // single-rank bucket
  uint64_t* d_clock = nullptr;
  uint64_t* d_stamps = nullptr;   // per group: pack, all-reduce, unpack spans (3 x [start, end])
  std::vector<uint64_t> h_stamps;
  float scale = 1.f;
  uint32_t flags = 0;
  std::vector<float*> host_src, host_dst;
  // dependency events (fork/join) and the three timing events of an iteration
  cudaEvent_t dep_fork = nullptr, dep_join = nullptr, dep_compute = nullptr;
  std::vector<cudaEvent_t> dep_ready;
  cudaEvent_t t_start = nullptr, t_compute = nullptr, t_end = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaGraph_t graph = nullptr;
  int launches = 0;
  bool capturing = false;
};

namespace {

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

ArArgs make_args(const mgw_comm* c, int64_t n) {
  ArArgs a;
  memset(&a, 0, sizeof(a));
  for (int s = 0; s < c->world; ++s) {
    char* base = c->peer[s];
    a.slot[s] = base + kCtrlBytes;
    a.arrive[s] = reinterpret_cast<uint64_t*>(base + kArriveOff);
    a.mid[s] = reinterpret_cast<uint64_t*>(base + kMidOff);
    a.abort_flag[s] = reinterpret_cast<uint32_t*>(base + kAbortOff);
  }
  a.out[c->rank] = c->result;
  a.state = c->state;
  a.err = c->err;
  a.slot_stride = c->slot_bytes;
  a.n = n;
  a.timeout_ns = c->timeout_ns;
  a.rank = c->rank;
  a.world = c->world;
  a.flags = 0;
  return a;
}

int pick_algo(const mgw_comm* c, int64_t n, int algo) {
  if (algo != MGW_ALGO_AUTO) return algo;
  return n * 4 <= c->oneshot_max_bytes ? MGW_ALGO_ONESHOT : MGW_ALGO_TWOSHOT;
}

int comm_allreduce(mgw_comm* c, int64_t n, int algo, cudaStream_t stream, uint64_t* stamp = nullptr) {
  if (n < 0 || n * 4 > c->slot_bytes) return set_error(MGW_EINVAL, "bucket of %lld elements exceeds slot capacity %lld B", (long long)n, (long long)c->slot_bytes);
  if (c->world == 1) {
    if (n > 0) MGW_CUDA(cudaMemcpyAsync(c->result, c->region + kCtrlBytes, n * 4, cudaMemcpyDeviceToDevice, stream));
    return MGW_OK;
  }
  if (!c->peers_open) return set_error(MGW_EINVAL, "peers not opened (call mgw_comm_open_peers)");
  ArArgs a = make_args(c, n);
  a.stamp = stamp;
  return launch_allreduce(a, pick_algo(c, n, algo), c->max_ctas, stream);
}

int comm_pack(mgw_comm* c, const void* table, int n_rows, int64_t n, float scale, cudaStream_t stream,
              uint64_t* stamp = nullptr) {
  if (n * 4 > c->slot_bytes) return set_error(MGW_EINVAL, "bucket of %lld elements exceeds slot capacity %lld B", (long long)n, (long long)c->slot_bytes);
  float* slot0 = reinterpret_cast<float*>(c->region + kCtrlBytes);
  const uint32_t* calls = c->world > 1 ? c->state : nullptr;
  return launch_rows<RowOp::kPack>(table, n_rows, slot0, n, scale, nullptr, calls, c->slot_bytes / 4, nullptr, stream,
                                   stamp);
}

}  // namespace

extern "C" {

const char* mgw_version(void) { return "mgwfbp_b200 0.1.0 (sm_100a)"; }

int mgw_last_error(char* buf, size_t len) {
  if (buf && len) {
    strncpy(buf, g_last_error.c_str(), len - 1);
    buf[len - 1] = '\0';
  }
  return (int)g_last_error.size();
}

int mgw_device_count(int* out) {
  if (!out) return set_error(MGW_EINVAL, "out is null");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return set_error(MGW_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *out = n;
  return MGW_OK;
}

int mgw_spin_ns(int64_t ns, void* stream) {
  if (ns < 0) return set_error(MGW_EINVAL, "spin time must be >= 0, got %lld", (long long)ns);
  spin_relative_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ns);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int mgw_desc_upload(const mgw_tensor_desc* rows, int n, void** dev_table) {
  if (!dev_table || n < 0 || (n > 0 && !rows)) return set_error(MGW_EINVAL, "bad descriptor table arguments");
  for (int i = 0; i < n; ++i) {
    if (rows[i].count < 0 || rows[i].offset < 0) return set_error(MGW_EINVAL, "row %d: negative count/offset", i);
    if (i > 0 && rows[i].offset < rows[i - 1].offset + rows[i - 1].count)
      return set_error(MGW_EINVAL, "row %d: rows must be sorted by offset and non-overlapping", i);
  }
  void* p = nullptr;
  MGW_CUDA(cudaMalloc(&p, std::max<size_t>(1, sizeof(Row) * (size_t)n)));
  if (n) MGW_CUDA(cudaMemcpy(p, rows, sizeof(Row) * (size_t)n, cudaMemcpyHostToDevice));
  *dev_table = p;
  return MGW_OK;
}

int mgw_desc_free(void* dev_table) {
  if (dev_table) MGW_CUDA(cudaFree(dev_table));
  return MGW_OK;
}

int mgw_pack(const void* dev_table, int n, float* bucket, int64_t bucket_elems, float scale, void* stream) {
  if (!dev_table || !bucket || bucket_elems < 0) return set_error(MGW_EINVAL, "bad pack arguments");
  return launch_rows<RowOp::kPack>(dev_table, n, bucket, bucket_elems, scale, nullptr, nullptr, 0, nullptr,
                                   static_cast<cudaStream_t>(stream));
}

int mgw_unpack(const void* dev_table, int n, const float* bucket, int64_t bucket_elems, void* stream) {
  if (!dev_table || !bucket || bucket_elems < 0) return set_error(MGW_EINVAL, "bad unpack arguments");
  return launch_rows<RowOp::kUnpack>(dev_table, n, const_cast<float*>(bucket), bucket_elems, 1.f, nullptr, nullptr,
                                     0, nullptr, static_cast<cudaStream_t>(stream));
}

static int table_extent(const void* dev_table, int n, cudaStream_t stream, int64_t* out) {
  // extent of a device table = last row's offset + count (read back once)
  if (n <= 0) {
    *out = 0;
    return MGW_OK;
  }
  Row last;
  MGW_CUDA(cudaMemcpyAsync(&last, static_cast<const Row*>(dev_table) + (n - 1), sizeof(Row), cudaMemcpyDeviceToHost, stream));
  MGW_CUDA(cudaStreamSynchronize(stream));
  *out = last.offset + last.count;
  return MGW_OK;
}

int mgw_fill_const(const void* dev_table, int n, const float* values_dev, void* stream) {
  if (!dev_table || !values_dev) return set_error(MGW_EINVAL, "bad fill arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t total = 0;
  int rc = table_extent(dev_table, n, s, &total);
  if (rc) return rc;
  return launch_rows<RowOp::kFill>(dev_table, n, nullptr, total, 1.f, values_dev, nullptr, 0, nullptr, s);
}

int mgw_check_const(const void* dev_table, int n, const float* values_dev, int64_t* mismatches, void* stream) {
  if (!dev_table || !values_dev || !mismatches) return set_error(MGW_EINVAL, "bad check arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t total = 0;
  int rc = table_extent(dev_table, n, s, &total);
  if (rc) return rc;
  unsigned long long* d_bad = nullptr;
  MGW_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long)));
  MGW_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), s));
  rc = launch_rows<RowOp::kCheck>(dev_table, n, nullptr, total, 1.f, values_dev, nullptr, 0, d_bad, s);
  unsigned long long bad = 0;
  if (rc == MGW_OK) {
    MGW_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
    MGW_CUDA(cudaStreamSynchronize(s));
  }
  cudaFree(d_bad);
  *mismatches = (int64_t)bad;
  return rc;
}

int mgw_comm_create(int rank, int world, int device, int64_t capacity_bytes, mgw_comm** out, uint8_t* ipc_handle_out) {
  if (!out) return set_error(MGW_EINVAL, "out is null");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks) return set_error(MGW_EINVAL, "world must lie in 1..%d, got %d", kMaxRanks, world);
  if (rank < 0 || rank >= world) return set_error(MGW_EINVAL, "rank must lie in [0, %d), got %d", world, rank);
  if (capacity_bytes < 0) return set_error(MGW_EINVAL, "capacity must be >= 0");
  MGW_CUDA(cudaSetDevice(device));
  mgw_comm* c = new mgw_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->capacity = capacity_bytes;
  c->slot_bytes = round_up(std::max<int64_t>(capacity_bytes, 256), 256);
  const size_t region_bytes = kCtrlBytes + 2 * (size_t)c->slot_bytes;
  cudaError_t e = cudaMalloc(&c->region, region_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->region, 0, kCtrlBytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->state, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(c->state, 0, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&c->result, (size_t)c->slot_bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && ipc_handle_out) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, c->region);
    if (e == cudaSuccess) memcpy(ipc_handle_out, &h, MGW_IPC_HANDLE_BYTES);
  }
  if (e != cudaSuccess) {
    mgw_comm_destroy(c);
    return set_error(MGW_ECUDA, "communicator setup on device %d: %s", device, cudaGetErrorString(e));
  }
  c->peer[rank] = c->region;
  if (world == 1) c->peers_open = true;
  *out = c;
  return MGW_OK;
}

int mgw_comm_open_peers(mgw_comm* c, const uint8_t* handles) {
  if (!c) return set_error(MGW_EINVAL, "comm is null");
  if (c->world == 1) return MGW_OK;
  if (!handles) return set_error(MGW_EINVAL, "handles is null");
  MGW_CUDA(cudaSetDevice(c->device));
  for (int s = 0; s < c->world; ++s) {
    if (s == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + (size_t)s * MGW_IPC_HANDLE_BYTES, MGW_IPC_HANDLE_BYTES);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return set_error(MGW_EPROTO, "rank %d: cannot map rank %d's bucket: %s", c->rank, s, cudaGetErrorString(e));
    c->peer[s] = static_cast<char*>(p);
  }
  c->peers_open = true;
  return MGW_OK;
}

int mgw_comm_destroy(mgw_comm* c) {
  if (!c) return MGW_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int s = 0; s < kMaxRanks; ++s)
    if (s != c->rank && c->peer[s]) cudaIpcCloseMemHandle(c->peer[s]);
  if (c->region) cudaFree(c->region);
  if (c->state) cudaFree(c->state);
  if (c->err) cudaFree(c->err);
  if (c->result) cudaFree(c->result);
  delete c;
  return MGW_OK;
}

int mgw_comm_set_timeout_ms(mgw_comm* c, int64_t ms) {
  if (!c || ms <= 0) return set_error(MGW_EINVAL, "bad timeout");
  c->timeout_ns = (uint64_t)ms * 1000000ull;
  return MGW_OK;
}

int mgw_comm_set_oneshot_max(mgw_comm* c, int64_t bytes) {
  if (!c || bytes < 0) return set_error(MGW_EINVAL, "bad one-shot threshold");
  c->oneshot_max_bytes = bytes;
  return MGW_OK;
}

int mgw_comm_input(mgw_comm* c, float** slot) {
  if (!c || !slot) return set_error(MGW_EINVAL, "bad arguments");
  uint32_t calls = 0;
  if (c->world > 1) {
    MGW_CUDA(cudaSetDevice(c->device));
    MGW_CUDA(cudaDeviceSynchronize());
    MGW_CUDA(cudaMemcpy(&calls, c->state, sizeof(calls), cudaMemcpyDeviceToHost));
  }
  const int64_t parity = c->world > 1 ? (int64_t)((calls + 1u) & 1u) : 0;
  *slot = reinterpret_cast<float*>(c->region + kCtrlBytes + parity * c->slot_bytes);
  return MGW_OK;
}

int mgw_comm_result(mgw_comm* c, float** result) {
  if (!c || !result) return set_error(MGW_EINVAL, "bad arguments");
  *result = c->result;
  return MGW_OK;
}

int mgw_comm_pack(mgw_comm* c, const void* dev_table, int n, int64_t n_elem, float scale, void* stream) {
  if (!c || !dev_table) return set_error(MGW_EINVAL, "bad arguments");
  return comm_pack(c, dev_table, n, n_elem, scale, static_cast<cudaStream_t>(stream));
}

int mgw_allreduce(mgw_comm* c, int64_t n_elem, int algo, void* stream) {
  if (!c) return set_error(MGW_EINVAL, "comm is null");
  if (algo < MGW_ALGO_AUTO || algo > MGW_ALGO_TWOSHOT) return set_error(MGW_EINVAL, "unknown algorithm %d", algo);
  return comm_allreduce(c, n_elem, algo, static_cast<cudaStream_t>(stream));
}

int mgw_comm_error(mgw_comm* c, int* code) {
  if (!c || !code) return set_error(MGW_EINVAL, "bad arguments");
  MGW_CUDA(cudaSetDevice(c->device));
  MGW_CUDA(cudaDeviceSynchronize());
  MGW_CUDA(cudaMemcpy(code, c->err, sizeof(int), cudaMemcpyDeviceToHost));
  return MGW_OK;
}

int mgw_comm_calls(mgw_comm* c, int64_t* calls) {
  if (!c || !calls) return set_error(MGW_EINVAL, "bad arguments");
  uint32_t v = 0;
  MGW_CUDA(cudaSetDevice(c->device));
  MGW_CUDA(cudaDeviceSynchronize());
  MGW_CUDA(cudaMemcpy(&v, c->state, sizeof(v), cudaMemcpyDeviceToHost));
  *calls = v;
  return MGW_OK;
}

int mgw_allreduce_emulated(float* const* ins, float* const* outs, int world, int64_t n, int algo, void* stream) {
  if (!ins || !outs || world < 1 || world > kMaxRanks || n < 0) return set_error(MGW_EINVAL, "bad emulated all-reduce arguments");
  if (algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT) return set_error(MGW_EINVAL, "emulated all-reduce needs an explicit algorithm");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ArArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < world; ++r) {
    a.slot[r] = reinterpret_cast<char*>(ins[r]);
    a.out[r] = outs[r];
    if (algo == MGW_ALGO_ONESHOT) {
      for (int q = 0; q < world; ++q)
        if (outs[r] == ins[q]) return set_error(MGW_EINVAL, "one-shot output may not alias an input");
    }
  }
  a.n = n;
  a.world = world;
  if (n == 0) return MGW_OK;
  if (algo == MGW_ALGO_ONESHOT) {
    for (int r = 0; r < world; ++r) {
      a.rank = r;
      a.flags = kNoBarrier;
      int rc = launch_allreduce(a, algo, 2 * kSMs, s);
      if (rc) return rc;
    }
    return MGW_OK;
  }
  for (int phase = 0; phase < 2; ++phase) {
    for (int r = 0; r < world; ++r) {
      a.rank = r;
      a.flags = kNoBarrier | (phase == 0 ? kSkipPhase2 : kSkipPhase1);
      int rc = launch_allreduce(a, algo, 2 * kSMs, s);
      if (rc) return rc;
    }
  }
  return MGW_OK;
}

// Device time of back-to-back group-exchange steps, timed as one event pair around
// `reps` repetitions (after `warmups` untimed ones) so no per-launch event cost
// enters the figure.  kind: 0 = pack -> all-reduce -> unpack (single rank: pack ->
// unpack into `local_bucket`), 1 = all-reduce kernel only, 2 = pack only, 3 = unpack only.
int mgw_time_exchange(mgw_comm* c, const void* table, int n_rows, int64_t n_elem, float* local_bucket, int algo,
                      int kind, int reps, int warmups, double* seconds_per_rep, void* stream) {
  if (!table || reps < 1 || warmups < 0 || !seconds_per_rep || n_elem <= 0 || kind < 0 || kind > 3)
    return set_error(MGW_EINVAL, "bad timing arguments");
  const bool multi = c && c->world > 1;
  if (!multi && !local_bucket) return set_error(MGW_EINVAL, "single-rank timing needs a local bucket");
  if (kind == 1 && !multi) return set_error(MGW_EINVAL, "all-reduce timing needs a multi-rank communicator");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto step = [&]() -> int {
    int rc = MGW_OK;
    if (multi) {
      if (kind == 0 || kind == 2) rc = comm_pack(c, table, n_rows, n_elem, 1.f, s);
      if (rc == MGW_OK && (kind == 0 || kind == 1)) rc = comm_allreduce(c, n_elem, algo, s);
      if (rc == MGW_OK && (kind == 0 || kind == 3))
        rc = launch_rows<RowOp::kUnpack>(table, n_rows, c->result, n_elem, 1.f, nullptr, nullptr, 0, nullptr, s);
    } else {
      if (kind == 0 || kind == 2)
        rc = launch_rows<RowOp::kPack>(table, n_rows, local_bucket, n_elem, 1.f, nullptr, nullptr, 0, nullptr, s);
      if (rc == MGW_OK && (kind == 0 || kind == 3))
        rc = launch_rows<RowOp::kUnpack>(table, n_rows, local_bucket, n_elem, 1.f, nullptr, nullptr, 0, nullptr, s);
    }
    return rc;
  };
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  MGW_CUDA(cudaEventCreate(&ev0));
  cudaError_t e = cudaEventCreate(&ev1);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev0);
    return set_error(MGW_ECUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
  }
  int rc = MGW_OK;
  for (int r = 0; r < warmups && rc == MGW_OK; ++r) rc = step();
  // hold the stream while the host enqueues the timed reps
  if (rc == MGW_OK) spin_relative_kernel<<<1, 32, 0, s>>>(1000000 + 20000LL * reps);
  if (rc == MGW_OK) cudaEventRecord(ev0, s);
  for (int r = 0; r < reps && rc == MGW_OK; ++r) rc = step();
  if (rc == MGW_OK) {
    cudaEventRecord(ev1, s);
    e = cudaEventSynchronize(ev1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev0, ev1);
    if (e != cudaSuccess)
      rc = set_error(MGW_ECUDA, "timing loop: %s", cudaGetErrorString(e));
    else
      *seconds_per_rep = ms * 1e-3 / reps;
  }
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  return rc;
}

// ------------------------------------------------------------ schedule engine

static void sched_release(mgw_sched* s) {
  if (!s) return;
  if (s->graph_exec) cudaGraphExecDestroy(s->graph_exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  for (auto e : s->dep_ready) cudaEventDestroy(e);
  for (cudaEvent_t e : {s->dep_fork, s->dep_join, s->dep_compute, s->t_start, s->t_compute, s->t_end})
    if (e) cudaEventDestroy(e);
  for (void* p : {(void*)s->d_rows, (void*)s->d_fill, (void*)s->local_bucket, (void*)s->d_clock, (void*)s->d_stamps})
    if (p) cudaFree(p);
  delete s;
}

int mgw_sched_create(mgw_comm* comm, const mgw_tensor_desc* rows, int n_rows, const mgw_group* groups, int n_groups,
                     float scale, uint32_t flags, const float* fill_values, float* const* host_src,
                     float* const* host_dst, mgw_sched** out) {
  if (!out || (n_rows > 0 && !rows) || !groups || n_rows < 0 || n_groups <= 0)
    return set_error(MGW_EINVAL, "bad schedule arguments");
  *out = nullptr;
  if ((flags & MGW_SCHED_FILL) && !fill_values) return set_error(MGW_EINVAL, "MGW_SCHED_FILL needs fill_values");
  if ((flags & MGW_SCHED_HOSTIO) && (!host_src || !host_dst))
    return set_error(MGW_EINVAL, "MGW_SCHED_HOSTIO needs host_src and host_dst");
  int64_t max_elems = 0;
  for (int g = 0; g < n_groups; ++g) {
    const mgw_group& gr = groups[g];
    if (gr.desc_begin < 0 || gr.desc_count < 0 || gr.desc_begin + gr.desc_count > n_rows)
      return set_error(MGW_EINVAL, "group %d: descriptor range outside the table", g);
    int64_t expect = 0;
    for (int k = gr.desc_begin; k < gr.desc_begin + gr.desc_count; ++k) {
      if (rows[k].offset != expect) return set_error(MGW_EINVAL, "group %d: rows must tile the bucket contiguously", g);
      expect += rows[k].count;
    }
    if (expect != gr.n_elem)
      return set_error(MGW_EINVAL, "group %d: n_elem %lld != rows total %lld", g, (long long)gr.n_elem, (long long)expect);
    if (gr.ready_ns < 0) return set_error(MGW_EINVAL, "group %d: negative ready time", g);
    if (g > 0 && gr.ready_ns < groups[g - 1].ready_ns) return set_error(MGW_EINVAL, "groups must be in send order");
    max_elems = std::max(max_elems, gr.n_elem);
  }
  const int world = comm ? comm->world : 1;
  if (comm && max_elems * 4 > comm->slot_bytes)
    return set_error(MGW_EINVAL, "largest group (%lld B) exceeds the communicator slot (%lld B)",
                     (long long)(max_elems * 4), (long long)comm->slot_bytes);
  mgw_sched* s = new mgw_sched();
  s->comm = comm;
  s->world = world;
  if (n_rows > 0) s->rows.assign(reinterpret_cast<const Row*>(rows), reinterpret_cast<const Row*>(rows) + n_rows);
  s->groups.assign(groups, groups + n_groups);
  s->scale = scale;
  s->flags = flags;
  if ((flags & MGW_SCHED_HOSTIO) && n_rows > 0) {
    s->host_src.assign(host_src, host_src + n_rows);
    s->host_dst.assign(host_dst, host_dst + n_rows);
  }
  s->h_stamps.assign((size_t)n_groups * 6, 0);
  cudaError_t e = cudaMalloc(&s->d_rows, sizeof(Row) * (size_t)std::max(1, n_rows));
  if (e == cudaSuccess && n_rows > 0) e = cudaMemcpy(s->d_rows, rows, sizeof(Row) * (size_t)n_rows, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && (flags & MGW_SCHED_FILL)) {
    e = cudaMalloc(&s->d_fill, sizeof(float) * (size_t)std::max(1, n_rows));
    if (e == cudaSuccess && n_rows > 0)
      e = cudaMemcpy(s->d_fill, fill_values, sizeof(float) * (size_t)n_rows, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && world == 1) e = cudaMalloc(&s->local_bucket, std::max<size_t>(256, (size_t)max_elems * 4));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_clock, sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMemset(s->d_clock, 0, sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_stamps, sizeof(uint64_t) * (size_t)n_groups * 6);
  if (e == cudaSuccess) e = cudaMemset(s->d_stamps, 0, sizeof(uint64_t) * (size_t)n_groups * 6);
  auto mk = [&](cudaEvent_t* ev, bool timing) {
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, timing ? cudaEventDefault : cudaEventDisableTiming);
  };
  mk(&s->dep_fork, false);
  mk(&s->dep_join, false);
  mk(&s->dep_compute, false);
  mk(&s->t_start, true);
  mk(&s->t_compute, true);
  mk(&s->t_end, true);
  s->dep_ready.assign(n_groups, nullptr);
  for (int g = 0; g < n_groups; ++g) mk(&s->dep_ready[g], false);
  if (e != cudaSuccess) {
    sched_release(s);
    return set_error(MGW_ECUDA, "schedule setup: %s", cudaGetErrorString(e));
  }
  int launches = 2 + (world > 1 ? 1 : 0);  // stamp reset + clock mark (+ start barrier)
  for (int g = 0; g < n_groups; ++g) {
    launches += 1;  // spin
    if (groups[g].n_elem == 0) continue;
    launches += (flags & MGW_SCHED_FILL) ? 1 : 0;  // gradient production
    launches += 2;                                 // pack + unpack
    launches += world > 1 ? 1 : 0;                 // all-reduce
  }
  s->launches = launches;
  *out = s;
  return MGW_OK;
}

// Timing events: inside a stream capture they must be external record nodes; in
// eager mode they are plain records.
static cudaError_t record_timing(const mgw_sched* s, cudaEvent_t ev, cudaStream_t st) {
  return s->capturing ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal) : cudaEventRecord(ev, st);
}

static int sched_enqueue(mgw_sched* s, cudaStream_t cs, cudaStream_t ms) {
  const Row* d_rows = s->d_rows;
  const int n_groups = (int)s->groups.size();
  if (s->world > 1) {
    // align the ranks' iteration starts: a zero-length collective is a barrier
    int rc = comm_allreduce(s->comm, 0, MGW_ALGO_ONESHOT, cs);
    if (rc) return rc;
  }
  stamps_reset_kernel<<<1, 256, 0, cs>>>(s->d_stamps, n_groups * 3);
  MGW_CHECK_LAUNCH();
  MGW_CUDA(record_timing(s, s->t_start, cs));
  MGW_CUDA(cudaEventRecord(s->dep_fork, cs));
  clock_mark_kernel<<<1, 32, 0, cs>>>(s->d_clock);
  MGW_CHECK_LAUNCH();
  for (int g = 0; g < n_groups; ++g) {
    const mgw_group& gr = s->groups[g];
    if ((s->flags & MGW_SCHED_HOSTIO) && gr.n_elem > 0) {
      for (int k = gr.desc_begin; k < gr.desc_begin + gr.desc_count; ++k)
        if (s->rows[k].count)
          MGW_CUDA(cudaMemcpyAsync(s->rows[k].ptr, s->host_src[k], s->rows[k].count * 4, cudaMemcpyHostToDevice, cs));
    }
    if ((s->flags & MGW_SCHED_FILL) && gr.n_elem > 0) {
      int rc = launch_rows<RowOp::kFill>(d_rows + gr.desc_begin, gr.desc_count, nullptr, gr.n_elem, 1.f,
                                         s->d_fill + gr.desc_begin, nullptr, 0, nullptr, cs);
      if (rc) return rc;
    }
    spin_until_kernel<<<1, 32, 0, cs>>>(s->d_clock, gr.ready_ns);
    MGW_CHECK_LAUNCH();
    MGW_CUDA(cudaEventRecord(s->dep_ready[g], cs));
  }
  MGW_CUDA(record_timing(s, s->t_compute, cs));
  MGW_CUDA(cudaEventRecord(s->dep_compute, cs));

  MGW_CUDA(cudaStreamWaitEvent(ms, s->dep_fork, 0));
  for (int g = 0; g < n_groups; ++g) {
    const mgw_group& gr = s->groups[g];
    const Row* grows = d_rows + gr.desc_begin;
    uint64_t* st = s->d_stamps + 6 * (size_t)g;
    MGW_CUDA(cudaStreamWaitEvent(ms, s->dep_ready[g], 0));
    if (gr.n_elem == 0) continue;  // silent group: nothing to send (allreduce_net.py:549)
    int rc;
    if (s->world == 1) {
      rc = launch_rows<RowOp::kPack>(grows, gr.desc_count, s->local_bucket, gr.n_elem, s->scale, nullptr, nullptr, 0,
                                     nullptr, ms, st);
      if (rc) return rc;
      rc = launch_rows<RowOp::kUnpack>(grows, gr.desc_count, s->local_bucket, gr.n_elem, 1.f, nullptr, nullptr, 0,
                                       nullptr, ms, st + 4);
      if (rc) return rc;
    } else {
      rc = comm_pack(s->comm, grows, gr.desc_count, gr.n_elem, s->scale, ms, st);
      if (rc) return rc;
      rc = comm_allreduce(s->comm, gr.n_elem, gr.algo, ms, st + 2);
      if (rc) return rc;
      rc = launch_rows<RowOp::kUnpack>(grows, gr.desc_count, s->comm->result, gr.n_elem, 1.f, nullptr, nullptr, 0,
                                       nullptr, ms, st + 4);
      if (rc) return rc;
    }
    if (s->flags & MGW_SCHED_HOSTIO) {
      for (int k = gr.desc_begin; k < gr.desc_begin + gr.desc_count; ++k)
        if (s->rows[k].count)
          MGW_CUDA(cudaMemcpyAsync(s->host_dst[k], s->rows[k].ptr, s->rows[k].count * 4, cudaMemcpyDeviceToHost, ms));
    }
  }
  MGW_CUDA(cudaStreamWaitEvent(ms, s->dep_compute, 0));  // iteration ends no earlier than backward
  MGW_CUDA(record_timing(s, s->t_end, ms));
  MGW_CUDA(cudaEventRecord(s->dep_join, ms));
  MGW_CUDA(cudaStreamWaitEvent(cs, s->dep_join, 0));
  return MGW_OK;
}

int mgw_sched_run(mgw_sched* s, void* compute_stream, void* comm_stream) {
  if (!s) return set_error(MGW_EINVAL, "schedule is null");
  cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
  cudaStream_t ms = static_cast<cudaStream_t>(comm_stream);
  if (cs == ms) return set_error(MGW_EINVAL, "compute and comm streams must differ");
  if (!(s->flags & MGW_SCHED_GRAPH)) return sched_enqueue(s, cs, ms);
  if (!s->graph_exec) {
    MGW_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    s->capturing = true;
    int rc = sched_enqueue(s, cs, ms);
    s->capturing = false;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return set_error(MGW_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    s->graph = graph;
    MGW_CUDA(cudaGraphInstantiate(&s->graph_exec, graph, 0));
  }
  MGW_CUDA(cudaGraphLaunch(s->graph_exec, cs));
  return MGW_OK;
}

static int sched_fetch_stamps(mgw_sched* s) {
  MGW_CUDA(cudaEventSynchronize(s->t_end));
  MGW_CUDA(cudaMemcpy(s->h_stamps.data(), s->d_stamps, sizeof(uint64_t) * s->h_stamps.size(), cudaMemcpyDeviceToHost));
  return MGW_OK;
}

static double span_s(const uint64_t* st) {
  return (st[0] == ~0ull || st[1] < st[0]) ? 0.0 : (double)(st[1] - st[0]) * 1e-9;
}

int mgw_sched_times(mgw_sched* s, double* t_iter_s, double* compute_s, double* group_comm_s) {
  if (!s) return set_error(MGW_EINVAL, "schedule is null");
  int rc = sched_fetch_stamps(s);
  if (rc) return rc;
  float ms = 0.f;
  if (t_iter_s) {
    MGW_CUDA(cudaEventElapsedTime(&ms, s->t_start, s->t_end));
    *t_iter_s = ms * 1e-3;
  }
  if (compute_s) {
    MGW_CUDA(cudaEventElapsedTime(&ms, s->t_start, s->t_compute));
    *compute_s = ms * 1e-3;
  }
  if (group_comm_s) {
    for (size_t g = 0; g < s->groups.size(); ++g) {
      const uint64_t* st = &s->h_stamps[6 * g];
      // pack entry .. unpack exit: the group's whole exchange on the comm stream
      group_comm_s[g] = (st[0] == ~0ull || st[5] < st[0]) ? 0.0 : (double)(st[5] - st[0]) * 1e-9;
    }
  }
  return MGW_OK;
}

int mgw_sched_kernel_times(mgw_sched* s, double* pack_s, double* allreduce_s, double* unpack_s) {
  if (!s || !pack_s || !allreduce_s || !unpack_s) return set_error(MGW_EINVAL, "bad arguments");
  int rc = sched_fetch_stamps(s);
  if (rc) return rc;
  for (size_t g = 0; g < s->groups.size(); ++g) {
    const uint64_t* st = &s->h_stamps[6 * g];
    pack_s[g] = span_s(st);
    allreduce_s[g] = span_s(st + 2);
    unpack_s[g] = span_s(st + 4);
  }
  return MGW_OK;
}

int mgw_sched_launches(mgw_sched* s, int* per_iteration) {
  if (!s || !per_iteration) return set_error(MGW_EINVAL, "bad arguments");
  *per_iteration = s->launches;
  return MGW_OK;
}

int mgw_sched_destroy(mgw_sched* s) {
  if (s) {
    cudaDeviceSynchronize();
    sched_release(s);
  }
  return MGW_OK;
}

}  // extern "C"
