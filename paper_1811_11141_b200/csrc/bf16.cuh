// bf16.cuh -- merged-gradient exchange of bf16 gradients with fp32 accumulation
// (the reference's ModelProfile already prices element_bytes = 2,
// model_profile.py:24, but its ring only moves fp32).
//
// Wire and bucket format: bf16 (half the NVLink and HBM bytes of fp32).  Element e of
// reference segment s = seg(e) (allreduce_net.py:360-367) is reduced as
//     acc = f32(x_s); acc = acc + f32(x_{s+1}); ... ; acc = acc + f32(x_{s+N-1})   (RN)
//     out = bf16_rn(acc * scale)              (the multiply only when scale != 1)
// -- the reference ring's fold order in fp32 over exactly-upcast inputs, rounded once.
// Every rank gets the same bits (oracle: ring_oracle.ring_allreduce_bf16).
//
// Same kernel shapes as fused.cuh with 16-B slots of 8 elements:
//   one-shot: CTA b packs slot chunk b, barrier, folds chunk b of the N slots into the
//             tensors;
//   two-shot: CTA b packs chunk b of every part, barrier, folds chunk b of its own part
//             into its slot (in place, bf16) and its tensors, barrier, copies chunk b of
//             every peer's part into its tensors.
// The n % 8 tail belongs to the last CTA (and to part N-1).
#pragma once

#include <cuda_bf16.h>

#include "fused.cuh"

namespace mgw {

constexpr int kB16 = 8;  // bf16 elements per 16-B slot

__device__ __forceinline__ float b16_word_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float b16_word_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float b16_to_f32(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ uint16_t f32_to_b16(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }

// barrier tag: a rank calling the bf16 exchange while a peer calls the fp32 one (same n)
// is reported like a length mismatch
__device__ __forceinline__ uint32_t b16_tag(int64_t n) { return (uint32_t)n ^ 0x80000000u; }

__device__ __forceinline__ uint32_t b16_word(const uint4& v, int w) {
  return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

// fold one 16-B slot from the N inputs given in fold order
template <int N>
__device__ __forceinline__ uint4 b16_fold8(const uint4 (&x)[N], float scale, bool scaled) {
  uint32_t o[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    float lo = b16_word_lo(b16_word(x[0], w)), hi = b16_word_hi(b16_word(x[0], w));
#pragma unroll
    for (int k = 1; k < N; ++k) {
      lo = __fadd_rn(lo, b16_word_lo(b16_word(x[k], w)));
      hi = __fadd_rn(hi, b16_word_hi(b16_word(x[k], w)));
    }
    if (scaled) {
      lo = __fmul_rn(lo, scale);
      hi = __fmul_rn(hi, scale);
    }
    o[w] = (uint32_t)f32_to_b16(lo) | ((uint32_t)f32_to_b16(hi) << 16);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

template <int N>
__device__ __forceinline__ uint16_t b16_fold1(const uint16_t* const* in, int s, int64_t e, float scale, bool scaled) {
  float acc = b16_to_f32(__ldcg(in[s] + e));
#pragma unroll
  for (int k = 1; k < N; ++k) {
    const int src = s + k >= N ? s + k - N : s + k;
    acc = __fadd_rn(acc, b16_to_f32(__ldcg(in[src] + e)));
  }
  return f32_to_b16(scaled ? __fmul_rn(acc, scale) : acc);
}

// tensor address of bucket element e (row cursor k monotone per thread);
// fast: the 16-B slot at e lies inside one row at a 16-B aligned tensor address
__device__ __forceinline__ uint16_t* b16_tensor(const FusedArgs& f, int& k, int64_t e, bool& fast) {
  Row r = fused_row(f, k);
  while (e >= r.offset + r.count) r = fused_row(f, ++k);
  uint16_t* p = reinterpret_cast<uint16_t*>(r.ptr) + (e - r.offset);
  fast = e + kB16 <= r.offset + r.count && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  return p;
}

__device__ __forceinline__ uint16_t* b16_tensor1(const FusedArgs& f, int k, int64_t e) {
  Row r = fused_row(f, k);
  while (e >= r.offset + r.count) r = fused_row(f, ++k);
  return reinterpret_cast<uint16_t*>(r.ptr) + (e - r.offset);
}

__device__ __forceinline__ int b16_first_row(const FusedArgs& f, int64_t v0, int64_t v1) {
  const int64_t v = v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0;
  return fused_row_covering(f, v * kB16);
}

// pack slots [v0, v1) and scalar elements [t0, t1) of the tensors into `slot` (a copy:
// bf16 scaling happens after the fp32 fold)
__device__ void b16_pack_range(const FusedArgs& f, uint16_t* slot, int64_t v0, int64_t v1, int64_t t0, int64_t t1) {
  if (v0 < v1) {
    int k = b16_first_row(f, v0, v1);
    for (int64_t v = v0 + threadIdx.x; v < v1; v += kThreads) {
      const int64_t e = v * kB16;
      bool fast;
      const uint16_t* tp = b16_tensor(f, k, e, fast);
      if (fast) {
        *reinterpret_cast<uint4*>(slot + e) = *reinterpret_cast<const uint4*>(tp);
      } else {
        for (int j = 0; j < kB16; ++j) slot[e + j] = *b16_tensor1(f, k, e + j);
      }
    }
  }
  for (int64_t e = t0 + threadIdx.x; e < t1; e += kThreads) slot[e] = *b16_tensor1(f, fused_row_covering(f, e), e);
}

// fold slots [v0, v1) from the N inputs into the tensors (and own[] when non-null)
template <int N, int U>
__device__ void b16_reduce_range(const FusedArgs& f, const uint16_t* const* in, const int64_t* seg_end, int64_t v0,
                                 int64_t v1, uint16_t* own) {
  if (v0 >= v1) return;
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  int seg = advance_segment(0, (v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0) * kB16, seg_end);
  int k = b16_first_row(f, v0, v1);
  for (int64_t base = v0 + threadIdx.x; base < v1; base += (int64_t)U * kThreads) {
    uint4 x[U][N];
    int su[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vv = base + (int64_t)u * kThreads;
      ok[u] = false;
      su[u] = seg;
      if (vv < v1) {
        const int64_t e = vv * kB16;
        seg = advance_segment(seg, e, seg_end);
        su[u] = seg;
        ok[u] = e + kB16 - 1 < seg_end[seg];
        if (ok[u]) {
#pragma unroll
          for (int kk = 0; kk < N; ++kk) {
            const int src = seg + kk >= N ? seg + kk - N : seg + kk;
            x[u][kk] = __ldcg(reinterpret_cast<const uint4*>(in[src] + e));
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vv = base + (int64_t)u * kThreads;
      if (vv >= v1) continue;
      const int64_t e = vv * kB16;
      bool fast;
      uint16_t* tp = b16_tensor(f, k, e, fast);
      if (ok[u]) {
        const uint4 y = b16_fold8<N>(x[u], scale, scaled);
        if (own) *reinterpret_cast<uint4*>(own + e) = y;
        if (fast) {
          *reinterpret_cast<uint4*>(tp) = y;
        } else {
          const uint16_t* h = reinterpret_cast<const uint16_t*>(&y);
          for (int j = 0; j < kB16; ++j) *b16_tensor1(f, k, e + j) = h[j];
        }
      } else {  // the slot straddles a segment boundary: element by element
        int s = su[u];
        for (int j = 0; j < kB16; ++j) {
          s = advance_segment(s, e + j, seg_end);
          const uint16_t y = b16_fold1<N>(in, s, e + j, scale, scaled);
          if (own) own[e + j] = y;
          *b16_tensor1(f, k, e + j) = y;
        }
      }
    }
  }
}

template <int N>
__device__ void b16_reduce_tail(const FusedArgs& f, const uint16_t* const* in, const int64_t* seg_end, int64_t e0,
                                int64_t e1, uint16_t* own) {
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
    const uint16_t y = b16_fold1<N>(in, advance_segment(0, e, seg_end), e, scale, scaled);
    if (own) own[e] = y;
    *b16_tensor1(f, fused_row_covering(f, e), e) = y;
  }
}

// copy reduced slots [v0, v1) and scalars [t0, t1) of `src` into the tensors
__device__ void b16_scatter_range(const FusedArgs& f, const uint16_t* src, int64_t v0, int64_t v1, int64_t t0,
                                  int64_t t1) {
  constexpr int UC = 4;
  if (v0 < v1) {
    int k = b16_first_row(f, v0, v1);
    for (int64_t base = v0 + threadIdx.x; base < v1; base += (int64_t)UC * kThreads) {
      uint4 x[UC];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int64_t vv = base + (int64_t)u * kThreads;
        if (vv < v1) x[u] = __ldcg(reinterpret_cast<const uint4*>(src) + vv);
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int64_t vv = base + (int64_t)u * kThreads;
        if (vv >= v1) continue;
        const int64_t e = vv * kB16;
        bool fast;
        uint16_t* tp = b16_tensor(f, k, e, fast);
        if (fast) {
          *reinterpret_cast<uint4*>(tp) = x[u];
        } else {
          const uint16_t* h = reinterpret_cast<const uint16_t*>(&x[u]);
          for (int j = 0; j < kB16; ++j) *b16_tensor1(f, k, e + j) = h[j];
        }
      }
    }
  }
  for (int64_t e = t0 + threadIdx.x; e < t1; e += kThreads)
    *b16_tensor1(f, fused_row_covering(f, e), e) = __ldcg(src + e);
}

template <int N>
__global__ void __launch_bounds__(kThreads, 2) b16_oneshot_kernel(const __grid_constant__ FusedArgs f) {
  constexpr int U = Unroll<N>::value;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  const uint16_t* const* in = reinterpret_cast<const uint16_t* const*>(s_in);
  const int64_t nv = a.n / kB16;
  const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const int64_t v0 = (int64_t)blockIdx.x * per;
  const int64_t v1 = v0 + per < nv ? v0 + per : nv;
  const bool last = blockIdx.x == gridDim.x - 1;
  if (!(a.flags & kSkipPack))
    b16_pack_range(f, const_cast<uint16_t*>(in[a.rank]), v0, v1, last ? nv * kB16 : 0, last ? a.n : 0);
  int status = MGW_DEV_OK;
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, b16_tag(a.n), a);
    if (status == MGW_DEV_OK) {
      b16_reduce_range<N, U>(f, in, s_end, v0, v1, nullptr);
      if (last) b16_reduce_tail<N>(f, in, s_end, nv * kB16, a.n, nullptr);
    }
  }
  finish_call(a);
}

template <int N>
__global__ void __launch_bounds__(kThreads, 2) b16_twoshot_kernel(const __grid_constant__ FusedArgs f) {
  constexpr int U = Unroll<N>::value;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  const uint16_t* const* in = reinterpret_cast<const uint16_t* const*>(s_in);
  const int me = a.rank;
  const int b = blockIdx.x, G = gridDim.x;
  const int64_t nv = a.n / kB16;
  const bool last = b == G - 1;
  const int64_t tail0 = nv * kB16;
  uint16_t* mine = const_cast<uint16_t*>(in[me]);
  __shared__ PartChunks<N> pc;
  if (threadIdx.x == 0) part_chunks<N>(nv, b, G, pc);
  __syncthreads();
  if (!(a.flags & kSkipPack)) {
    for (int p = 0; p < N; ++p) b16_pack_range(f, mine, pc.lo[p], pc.lo[p] + pc.len[p], 0, 0);
    if (last) b16_pack_range(f, mine, 0, 0, tail0, a.n);
  }
  int status = MGW_DEV_OK;
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, b16_tag(a.n), a);
    if (status == MGW_DEV_OK) {
      b16_reduce_range<N, U>(f, in, s_end, pc.lo[me], pc.lo[me] + pc.len[me], mine);
      if (last && me == N - 1) b16_reduce_tail<N>(f, in, s_end, tail0, a.n, mine);
    }
  }
  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase2)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.mid, parity, epoch, b16_tag(a.n), a);
    if (status == MGW_DEV_OK) {
      for (int p = 0; p < N; ++p)
        if (p != me) b16_scatter_range(f, in[p], pc.lo[p], pc.lo[p] + pc.len[p], 0, 0);
      if (last && me != N - 1) b16_scatter_range(f, in[N - 1], 0, 0, tail0, a.n);
    }
  }
  finish_call(a);
}

template <int N>
int launch_b16_n(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream) {
  const int64_t nv = f.ar.n / kB16;
  if (algo == MGW_ALGO_ONESHOT)
    b16_oneshot_kernel<N><<<collective_grid<N>(nv, 0, max_ctas), kThreads, 0, stream>>>(f);
  else
    b16_twoshot_kernel<N><<<collective_grid<N>(nv / N, 0, max_ctas), kThreads, 0, stream>>>(f);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

inline int launch_b16(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream) {
  if (algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT)
    return set_error(MGW_EINVAL, "bf16 buckets support one-shot and two-shot only (algorithm %d)", algo);
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  switch (f.ar.world) {
    case 1: return launch_b16_n<1>(f, algo, max_ctas, stream);
    case 2: return launch_b16_n<2>(f, algo, max_ctas, stream);
    case 3: return launch_b16_n<3>(f, algo, max_ctas, stream);
    case 4: return launch_b16_n<4>(f, algo, max_ctas, stream);
    case 5: return launch_b16_n<5>(f, algo, max_ctas, stream);
    case 6: return launch_b16_n<6>(f, algo, max_ctas, stream);
    case 7: return launch_b16_n<7>(f, algo, max_ctas, stream);
    case 8: return launch_b16_n<8>(f, algo, max_ctas, stream);
    default: return set_error(MGW_EINVAL, "world %d outside 1..%d", f.ar.world, kMaxRanks);
  }
}

}  // namespace mgw
