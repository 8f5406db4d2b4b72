// nvls.cuh -- opt-in NVLink-SHARP (NVSwitch multicast) exchange for large buckets
// (stands in for ring_allreduce, allreduce_net.py:370-411, within fp32
// rounding only).
//
// Every rank's bucket is bound to one CUDA multicast object.  CTA b packs chunk b of
// every part into its own (unicast) copy, a per-CTA barrier, then reduces chunk b of
// its own part IN THE SWITCH (multimem.ld_reduce: one fp32 sum of the N copies comes
// back) and broadcasts it to every rank's copy (multimem.st), a second barrier, and
// finally unpacks chunk b of every part into the layer tensors.
//
// Per GPU NVLink traffic: in (N-1)/N·M + M/N = M, instead of two-shot's 2(N-1)/N·M,
// so the bus bandwidth can exceed the per-link ceiling.  The switch's summation order
// is not the reference ring's: results are identical on every rank and within fp32
// rounding of the exact sum, but not bit-identical to the reference -- hence opt-in
// (MGW_ALGO_NVLS), never chosen by MGW_ALGO_AUTO.
#pragma once

#include "fused.cuh"

namespace mgw {

struct NvlsArgs {
  FusedArgs f;       // rows, scale, flags/epochs (f.ar.slot unused)
  float* uc;         // this rank's unicast mapping of the multicast-bound bucket
  float* mc;         // the multicast mapping (same offsets)
};

__device__ __forceinline__ float4 multimem_ld_reduce_add4(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}

__device__ __forceinline__ float multimem_ld_reduce_add1(const float* mc) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
  return v;
}

__device__ __forceinline__ void multimem_st4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void multimem_st1(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}

template <int N>
__global__ void __launch_bounds__(kThreads, 2) nvls_kernel(const __grid_constant__ NvlsArgs x) {
  const FusedArgs& f = x.f;
  const ArArgs& a = f.ar;
  grid_dep_wait();
  stamp_enter(a.stamp);
  const uint32_t epoch = load_volatile32(a.state) + 1u;
  const int parity = (int)(epoch & 1u);
  const int me = a.rank;
  const int b = blockIdx.x, G = gridDim.x;
  const int64_t nv = a.n >> 2;
  const int64_t tail0 = nv << 2;
  const bool last = b == G - 1;
  __shared__ PartChunks<N> pc;
  if (threadIdx.x == 0) part_chunks<N>(nv, b, G, pc);
  __syncthreads();
  // 1. pack chunk b of every part into my unicast copy
  fused_pack_parts<N>(f, x.uc, pc);
  if (last) fused_pack_range(f, x.uc, 0, 0, tail0, a.n);
  int status = cta_barrier(a.arrive, parity, epoch, a.tag, a, blockIdx.x);
  if (status == MGW_DEV_OK) {
    // 2. reduce my part's chunk b in the switch and broadcast it to every copy
    constexpr int U = 4;
    const int64_t lo = pc.lo[me], len = pc.len[me];
    for (int64_t i = threadIdx.x; i < len; i += (int64_t)U * kThreads) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t ii = i + (int64_t)u * kThreads;
        if (ii < len) v[u] = multimem_ld_reduce_add4(x.mc + ((lo + ii) << 2));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t ii = i + (int64_t)u * kThreads;
        if (ii < len) multimem_st4(x.mc + ((lo + ii) << 2), v[u]);
      }
    }
    if (last && me == N - 1)
      for (int64_t e = tail0 + threadIdx.x; e < a.n; e += kThreads) multimem_st1(x.mc + e, multimem_ld_reduce_add1(x.mc + e));
    __threadfence_system();
    status = cta_barrier(a.mid, parity, epoch, a.tag, a, blockIdx.x);
  }
  if (status == MGW_DEV_OK) {
    // 3. unpack chunk b of every part (now reduced in my copy) into the tensors
    __threadfence();
    const float* uc = x.uc;
    for (int p = 0; p < N; ++p) fused_scatter_range(f, uc, pc.lo[p], pc.lo[p] + pc.len[p], 0, 0);
    if (last) fused_scatter_range(f, uc, 0, 0, tail0, a.n);
  }
  finish_call(a, gridDim.x);
}

}  // namespace mgw
