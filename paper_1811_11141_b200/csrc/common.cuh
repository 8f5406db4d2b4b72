// common.cuh -- constants, error plumbing and device helpers shared by the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "mgwfbp_b200.h"

namespace mgw {

// ------------------------------------------------------------------ errors

inline std::string& last_error_slot() {
  thread_local std::string msg;
  return msg;
}

inline int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error_slot() = buf;
  return code;
}

#define MGW_CUDA(call)                                                                             \
  do {                                                                                             \
    cudaError_t err_ = (call);                                                                     \
    if (err_ != cudaSuccess)                                                                       \
      return ::mgw::set_error(MGW_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(err_), __FILE__, \
                              __LINE__);                                                           \
  } while (0)

#define MGW_CHECK_LAUNCH()                                                                         \
  do {                                                                                             \
    cudaError_t err_ = cudaGetLastError();                                                         \
    if (err_ != cudaSuccess)                                                                       \
      return ::mgw::set_error(MGW_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(err_),   \
                              __FILE__, __LINE__);                                                 \
  } while (0)

// --------------------------------------------------------------- constants

constexpr int kMaxRanks = MGW_MAX_RANKS;
constexpr int kMaxBlocks = 512;     // barrier flag slots per parity (>= any grid we launch)
constexpr int kThreads = 512;       // threads per CTA of every bulk kernel
constexpr int kSMs = 148;
constexpr int64_t kTile = 16384;    // pack/unpack tile: 64 KB of bucket per CTA step
constexpr int kInlineRows = 40;     // descriptor rows passed by value as kernel parameters

// IPC region layout (per rank): [arrive | mid | abort | pad] [slot 0] [slot 1]
constexpr size_t kFlagsPerParity = (size_t)kMaxBlocks * kMaxRanks;
constexpr size_t kArriveOff = 0;
constexpr size_t kMidOff = kArriveOff + 2 * kFlagsPerParity * sizeof(uint64_t);
constexpr size_t kAbortOff = kMidOff + 2 * kFlagsPerParity * sizeof(uint64_t);
constexpr size_t kHdrOff = kAbortOff + 1024;  // LL headers u64 [2 parity][kMaxRanks src]
constexpr size_t kDoorOff = kHdrOff + 2 * kMaxRanks * sizeof(uint64_t);  // gate u64 [kMaxRanks src]
constexpr size_t kCtrlBytes = 262144;
static_assert(kDoorOff + kMaxRanks * sizeof(uint64_t) <= kCtrlBytes, "control area overflow");
// LL receive area u64 [2 parity][kMaxRanks src][kLLElems] follows the control area,
// then the two bucket slots.
constexpr int64_t kLLElems = 262144;  // 1 MB of fp32 payload per source per parity
constexpr size_t kLLOff = kCtrlBytes;
constexpr size_t kLLBytes = 2 * (size_t)kMaxRanks * (size_t)kLLElems * sizeof(uint64_t);
// pipelined two-shot flags u64 [2 kind][2 parity][kMaxBlocks][16 warp][kPipeSub][kMaxRanks src]
constexpr int kPipeSub = 8;
constexpr size_t kPipeOff = kLLOff + kLLBytes;
constexpr size_t kPipeBytes = 2 * 2 * (size_t)kMaxBlocks * (kThreads / 32) * kPipeSub * kMaxRanks * sizeof(uint64_t);
constexpr size_t kSlotOff = kPipeOff + kPipeBytes;

struct Row {  // identical layout to mgw_tensor_desc
  float* ptr;
  int64_t count;
  int64_t offset;
};
static_assert(sizeof(Row) == sizeof(mgw_tensor_desc), "Row must mirror mgw_tensor_desc");

// ------------------------------------------------------------ checked build
// -DMGW_CHECKED (__graft_entry__.build(checked=True) -> _lib/libmgwfbp_b200_checked.so):
// every tensor row walk, bucket / slot index, barrier flag slot, LL area index and push
// row offset the kernels compute is validated against its extent, and violations are
// counted in a per-translation-unit device word (mgw_checked_violations) instead of
// trapping.  compute-sanitizer is closed on this pool; this also catches overruns that
// stay inside one allocation (a slot overrunning into the next), which memcheck cannot.
#ifdef MGW_CHECKED
static __device__ unsigned long long g_violations;
#define MGW_EXPECT(cond)                                  \
  do {                                                    \
    if (!(cond)) atomicAdd(&::mgw::g_violations, 1ull);  \
  } while (0)
#define MGW_CHECKED_ONLY(x) x
#else
#define MGW_EXPECT(cond) \
  do {                   \
  } while (0)
#define MGW_CHECKED_ONLY(x)
#endif

// host side: read (and optionally reset) this translation unit's violation count
#ifdef MGW_CHECKED
#define MGW_DEFINE_VIOLATIONS(tu)                                                               \
  int violations_##tu(unsigned long long* out, bool reset) {                                   \
    if (cudaMemcpyFromSymbol(out, g_violations, sizeof(*out)) != cudaSuccess) return MGW_ECUDA; \
    if (reset) {                                                                                \
      const unsigned long long zero = 0;                                                        \
      if (cudaMemcpyToSymbol(g_violations, &zero, sizeof(zero)) != cudaSuccess) return MGW_ECUDA; \
    }                                                                                           \
    return MGW_OK;                                                                              \
  }
#else
#define MGW_DEFINE_VIOLATIONS(tu)                               \
  int violations_##tu(unsigned long long* out, bool) {         \
    *out = 0;                                                  \
    return MGW_OK;                                             \
  }
#endif

// ------------------------------------------------------------ device utils

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void store_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void store_release_sys32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t load_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t ld_relaxed_sys64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ uint32_t load_relaxed_sys32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t load_volatile32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Programmatic dependent launch: a kernel whose producer was launched with a
// programmatic event may start while the producer still runs; it waits here for the
// producer grid's completion (and memory) before touching its inputs.  A no-op for a
// normally launched kernel.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Kernel span stamps: every CTA folds its entry time into stamp[0] (min) and its
// exit time into stamp[1] (max), so [stamp[0], stamp[1]] is the kernel's execution
// span without the ~6.5 us an event-record pair costs inside a CUDA graph.
__device__ __forceinline__ void stamp_enter(uint64_t* stamp) {
  if (stamp != nullptr && threadIdx.x == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(stamp), (unsigned long long)global_ns());
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

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace mgw
