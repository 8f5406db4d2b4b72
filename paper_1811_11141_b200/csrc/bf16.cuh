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

#include "ll.cuh"

namespace mgw {

constexpr int kB16 = 8;  // bf16 elements per 16-B slot

__device__ __forceinline__ float b16_word_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float b16_word_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float b16_to_f32(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ uint16_t f32_to_b16(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }


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
  const Row r = walk_row(f, k, e);
  uint16_t* p = reinterpret_cast<uint16_t*>(r.ptr) + (e - r.offset);
  fast = e + kB16 <= r.offset + r.count && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  return p;
}

__device__ __forceinline__ uint16_t* b16_tensor1(const FusedArgs& f, int k, int64_t e) {
  const Row r = walk_row(f, k, e);
  return reinterpret_cast<uint16_t*>(r.ptr) + (e - r.offset);
}

__device__ __forceinline__ int b16_first_row(const FusedArgs& f, int64_t v0, int64_t v1) {
  const int64_t v = v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0;
  return fused_row_covering(f, v * kB16);
}

// pack slots [v0, v1) and scalar elements [t0, t1) of the tensors into `slot` (a copy:
// bf16 scaling happens after the fp32 fold)
static __device__ void b16_pack_range(const FusedArgs& f, uint16_t* slot, int64_t v0, int64_t v1, int64_t t0, int64_t t1) {
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
static __device__ void b16_scatter_range(const FusedArgs& f, const uint16_t* src, int64_t v0, int64_t v1, int64_t t0,
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

// pack chunk b of every part into my slot, parts interleaved (N loads in flight)
template <int N>
__device__ void b16_pack_parts(const FusedArgs& f, uint16_t* slot, const PartChunks<N>& pc) {
  int cur[N];
#pragma unroll
  for (int p = 0; p < N; ++p) cur[p] = fused_row_covering(f, (pc.lo[p] + (threadIdx.x < pc.len[p] ? threadIdx.x : 0)) * kB16);
  for (int64_t i = threadIdx.x; i < pc.longest; i += kThreads) {
    uint4 x[N];
    bool fast[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
      fast[p] = false;
      if (i < pc.len[p]) {
        const uint16_t* tp = b16_tensor(f, cur[p], (pc.lo[p] + i) * kB16, fast[p]);
        if (fast[p]) x[p] = *reinterpret_cast<const uint4*>(tp);
      }
    }
#pragma unroll
    for (int p = 0; p < N; ++p) {
      if (i >= pc.len[p]) continue;
      const int64_t e = (pc.lo[p] + i) * kB16;
      if (fast[p]) {
        *reinterpret_cast<uint4*>(slot + e) = x[p];
      } else {
        for (int j = 0; j < kB16; ++j) slot[e + j] = *b16_tensor1(f, cur[p], e + j);
      }
    }
  }
}

// copy chunk b of every peer's reduced part into my tensors, parts interleaved
template <int N>
__device__ void b16_scatter_parts(const FusedArgs& f, const uint16_t* const* in, int me, const PartChunks<N>& pc) {
  int cur[N];
#pragma unroll
  for (int p = 0; p < N; ++p) cur[p] = fused_row_covering(f, (pc.lo[p] + (threadIdx.x < pc.len[p] ? threadIdx.x : 0)) * kB16);
  for (int64_t i = threadIdx.x; i < pc.longest; i += kThreads) {
    uint4 x[N];
#pragma unroll
    for (int p = 0; p < N; ++p)
      if (p != me && i < pc.len[p]) x[p] = __ldcg(reinterpret_cast<const uint4*>(in[p]) + pc.lo[p] + i);
#pragma unroll
    for (int p = 0; p < N; ++p) {
      if (p == me || i >= pc.len[p]) continue;
      const int64_t e = (pc.lo[p] + i) * kB16;
      bool fast;
      uint16_t* tp = b16_tensor(f, cur[p], e, fast);
      if (fast) {
        *reinterpret_cast<uint4*>(tp) = x[p];
      } else {
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&x[p]);
        for (int j = 0; j < kB16; ++j) *b16_tensor1(f, cur[p], e + j) = h[j];
      }
    }
  }
}

template <int N>
__device__ __forceinline__ void b16_oneshot_body(const FusedArgs& f, const int cta, const int ctas) {
  constexpr int U = Unroll<N>::value;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  const uint16_t* const* in = reinterpret_cast<const uint16_t* const*>(s_in);
  const int64_t nv = a.n / kB16;
  int64_t v0, v1;
  cta_chunk(0, nv, cta, ctas, v0, v1);
  const bool last = cta == ctas - 1;
  if (!(a.flags & kSkipPack))
    b16_pack_range(f, const_cast<uint16_t*>(in[a.rank]), v0, v1, last ? nv * kB16 : 0, last ? a.n : 0);
  int status = MGW_DEV_OK;
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, cta);
    if (status == MGW_DEV_OK) {
      b16_reduce_range<N, U>(f, in, s_end, v0, v1, nullptr);
      if (last) b16_reduce_tail<N>(f, in, s_end, nv * kB16, a.n, nullptr);
    }
  }
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(b16_oneshot, FusedArgs)

template <int N>
__device__ __forceinline__ void b16_twoshot_body(const FusedArgs& f, const int cta, const int ctas) {
  constexpr int U = Unroll<N>::value;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  const uint16_t* const* in = reinterpret_cast<const uint16_t* const*>(s_in);
  const int me = a.rank;
  const int b = cta, G = ctas;
  const int64_t nv = a.n / kB16;
  const bool last = b == G - 1;
  const int64_t tail0 = nv * kB16;
  uint16_t* mine = const_cast<uint16_t*>(in[me]);
  __shared__ PartChunks<N> pc;
  if (threadIdx.x == 0) part_chunks<N>(nv, b, G, pc);
  __syncthreads();
  if (!(a.flags & kSkipPack)) {
    b16_pack_parts<N>(f, mine, pc);
    if (last) b16_pack_range(f, mine, 0, 0, tail0, a.n);
  }
  int status = MGW_DEV_OK;
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, cta);
    if (status == MGW_DEV_OK) {
      b16_reduce_range<N, U>(f, in, s_end, pc.lo[me], pc.lo[me] + pc.len[me], mine);
      if (last && me == N - 1) b16_reduce_tail<N>(f, in, s_end, tail0, a.n, mine);
    }
  }
  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase2)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.mid, parity, epoch, a.tag, a, cta);
    if (status == MGW_DEV_OK) {
      b16_scatter_parts<N>(f, in, me, pc);
      if (last && me != N - 1) b16_scatter_range(f, in[N - 1], 0, 0, tail0, a.n);
    }
  }
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(b16_twoshot, FusedArgs)

// LL push one-shot for small bf16 buckets: a word carries (epoch << 32 | two bf16), a
// 16-B push carries four elements.  Same protocol as ll_oneshot_kernel (ll.cuh): header
// length check by CTA 0, batched polls of the N sources, fold in the reference order in
// fp32, one rounding.  At most 2 * kLLMaxElems elements (1 MB of bf16 per parity).
__device__ __forceinline__ uint64_t ll_b16_word(uint32_t epoch, uint16_t lo, uint16_t hi) {
  return ((uint64_t)epoch << 32) | ((uint32_t)hi << 16) | lo;
}

template <int N>
__device__ __forceinline__ void ll_b16_body(const LLArgs& l, const int cta, const int ctas) {
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
  const bool do_push = !(a.flags & kSkipPack), do_fold = !(a.flags & kSkipPhase1);  // emulation split
  if (do_push && cta == 0 && threadIdx.x < N)
    st_relaxed_sys_u64(l.hdr[threadIdx.x] + parity * l.hdr_stride + me, ((uint64_t)epoch << 32) | a.tag);
  __syncthreads();

  // element quads of this CTA: [q0, q1) (quad j = elements 4j .. 4j+3 = words 2j, 2j+1)
  const int64_t quads = (n + 3) >> 2;
  const int64_t per = (quads + ctas - 1) / ctas;
  const int64_t q0 = (int64_t)cta * per;
  const int64_t q1 = q0 + per < quads ? q0 + per : quads;
  const size_t my_off = ((size_t)parity * kMaxRanks + me) * kLLMaxElems;

  // 1. pack and push my four elements of each quad to every rank
  int k = 0;
  if (q0 < q1) k = fused_row_covering(f, (q0 + threadIdx.x) * 4 < n ? (q0 + threadIdx.x) * 4 : 0);
  for (int64_t j = q0 + threadIdx.x; do_push && j < q1; j += kThreads) {
    const int64_t e = 4 * j;
    uint16_t x[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      x[h] = 0;
      if (e + h < n) {
        Row r = fused_row(f, k);
        while (e + h >= r.offset + r.count) r = fused_row(f, ++k);
        x[h] = reinterpret_cast<const uint16_t*>(r.ptr)[e + h - r.offset];
      }
    }
    const uint64_t w0 = ll_b16_word(epoch, x[0], x[1]), w1 = ll_b16_word(epoch, x[2], x[3]);
#pragma unroll
    for (int r = 0; r < N; ++r) st_relaxed_sys_v2(l.ll[r] + my_off + 2 * j, w0, w1);
  }

  // 2. CTA 0 checks every peer's header (length and dtype agreement)
  int status = do_fold ? ll_header_check(l, epoch, parity, cta == 0, MGW_DEV_OK, &s_status) : MGW_DEV_OK;
  const uint64_t* hdr_mine = l.hdr[me] + parity * l.hdr_stride;

  // 3. fold: batched 16-B polls of the N sources, fp32 fold in the reference order
  if (do_fold && status == MGW_DEV_OK) {
    const float scale = f.scale;
    const bool scaled = scale != 1.0f;
    const uint64_t* base = l.ll[me] + (size_t)parity * kMaxRanks * kLLMaxElems;
    int seg = 0;
    k = 0;
    if (q0 < q1) k = fused_row_covering(f, (q0 + threadIdx.x) * 4 < n ? (q0 + threadIdx.x) * 4 : 0);
    for (int64_t j = q0 + threadIdx.x; j < q1 && status == MGW_DEV_OK; j += kThreads) {
      const int64_t e = 4 * j;
      uint64_t w0[N], w1[N];
#pragma unroll
      for (int src = 0; src < N; ++src) ld_relaxed_sys_v2(base + (size_t)src * kLLMaxElems + 2 * j, w0[src], w1[src]);
#pragma unroll
      for (int src = 0; src < N; ++src) {
        if ((uint32_t)(w0[src] >> 32) != epoch || (uint32_t)(w1[src] >> 32) != epoch)
          ll_wait2(base + (size_t)src * kLLMaxElems + 2 * j, hdr_mine + src, epoch, a, status, w0[src], w1[src]);
      }
      if (status != MGW_DEV_OK) break;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int64_t eh = e + h;
        if (eh >= n) break;
        seg = advance_segment(seg, eh, s_end);
        float acc = 0.f;
#pragma unroll
        for (int kk = 0; kk < N; ++kk) {
          int src = seg + kk;
          src = src >= N ? src - N : src;
          uint64_t w = 0;
#pragma unroll
          for (int q = 0; q < N; ++q) w = q == src ? (h < 2 ? w0[q] : w1[q]) : w;
          const float x = (h & 1) ? b16_word_hi((uint32_t)w) : b16_word_lo((uint32_t)w);
          acc = kk == 0 ? x : __fadd_rn(acc, x);
        }
        const uint16_t y = f32_to_b16(scaled ? __fmul_rn(acc, scale) : acc);
        Row r = fused_row(f, k);
        while (eh >= r.offset + r.count) r = fused_row(f, ++k);
        reinterpret_cast<uint16_t*>(r.ptr)[eh - r.offset] = y;
      }
    }
  }
  if (status != MGW_DEV_OK && status != s_status) ll_report(a, status);  // a fold thread's own error
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(ll_b16, LLArgs)

}  // namespace mgw
