// fused.cuh -- one kernel per merge group: K1 pack -> K2/K3 all-reduce -> K4 unpack.
// Replaces, per group, the reference's per-layer pack (allreduce_net.py:544-546) and
// ring_allreduce (allreduce_net.py:370-411) on the bucket layout of :499-509.
//
// The separate kernels cost three launches per group and a round trip of the whole
// bucket through the result buffer.  Here every CTA packs exactly the bucket chunk its
// peers' matching CTA will read (so the per-CTA barrier still suffices), folds the
// chunk from all ranks in the reference order, and writes the reduced values straight
// back into the layer tensors.  Same bits as pack + all-reduce + unpack.
//
//   one-shot: CTA b packs chunk b of its own slot, barrier, folds chunk b from the N
//             slots into the tensors.
//   two-shot: CTA b packs chunk b of every rank's part, barrier, folds chunk b of its
//             own part into its slot (in place) and the tensors, barrier, copies chunk
//             b of every peer's reduced part into the tensors.
#pragma once

#include "allreduce.cuh"
#include "rows.cuh"

namespace mgw {

struct FusedArgs {
  ArArgs ar;
  Row inline_rows[kInlineRows];
  const Row* rows;
  int n_rows;
  int use_inline;
  float scale;
};

__device__ __forceinline__ Row fused_row(const FusedArgs& f, int k) {
  return f.use_inline ? f.inline_rows[k] : f.rows[k];
}

__device__ __forceinline__ int fused_row_covering(const FusedArgs& f, int64_t e) {
  int lo = 0, hi = f.n_rows;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const Row r = fused_row(f, mid);
    if (r.offset + r.count > e)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// Tensor address of bucket element e; `k` is a monotone per-thread row cursor.
// fast4: the 16-B slot at e is inside one row at a 16-B aligned tensor address.
// Row of bucket element e, advancing the monotone cursor k (checked build: the walk never
// leaves the table and e lies inside the row and the bucket).
__device__ __forceinline__ Row walk_row(const FusedArgs& f, int& k, int64_t e) {
  Row r = fused_row(f, k);
  while (e >= r.offset + r.count) {
    MGW_CHECKED_ONLY(if (k + 1 >= f.n_rows) {
      MGW_EXPECT(false);
      break;
    })
    r = fused_row(f, ++k);
  }
  MGW_EXPECT(k < f.n_rows && e >= r.offset && e < r.offset + r.count && e < f.ar.n);
  return r;
}

__device__ __forceinline__ float* fused_tensor(const FusedArgs& f, int& k, int64_t e, bool& fast4) {
  const Row r = walk_row(f, k, e);
  float* p = r.ptr + (e - r.offset);
  fast4 = e + 4 <= r.offset + r.count && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  return p;
}

__device__ __forceinline__ float* fused_tensor1(const FusedArgs& f, int k, int64_t e) {
  const Row r = walk_row(f, k, e);
  return r.ptr + (e - r.offset);
}

// Slow paths (a 16-B slot straddling two rows or two reference segments, or sitting at a
// misaligned tensor address).  kOol = out of line: the N = 1 group kernel calls them as
// functions -- inlined into every unrolled hot loop they made it 82 KB of SASS, and a small
// group's launch runs ~2 us, so fetching a large body from L2 on cold SMs is a visible share
// of it (in-step spans -5 %, profiles/n1_group_spans_r02.json).  The N >= 2 kernels inline
// them: a call there makes the caller spill around it.
__device__ __forceinline__ void pack4_body(const FusedArgs& f, float* slot, int k, int64_t e, float scale) {
  for (int j = 0; j < 4; ++j) {
    const float y = *fused_tensor1(f, k, e + j);
    slot[e + j] = scale != 1.0f ? __fmul_rn(y, scale) : y;
  }
}

__device__ __forceinline__ void store4_body(const FusedArgs& f, int k, int64_t e, float4 v) {
  *fused_tensor1(f, k, e) = v.x;
  *fused_tensor1(f, k, e + 1) = v.y;
  *fused_tensor1(f, k, e + 2) = v.z;
  *fused_tensor1(f, k, e + 3) = v.w;
}

// four elements whose fold starts differ (the slot straddles a reference segment boundary)
template <int N>
__device__ __forceinline__ void fold4_body(const FusedArgs& f, const float* const* in, const int64_t* seg_end, int s,
                                           int k, int64_t e, float* own) {
  for (int j = 0; j < 4; ++j) {
    s = advance_segment(s, e + j, seg_end);
    const float y = fold1<N>(in, s, e + j);
    if (own) own[e + j] = y;
    *fused_tensor1(f, k, e + j) = y;
  }
}

static __device__ __noinline__ void pack4_ool(const FusedArgs& f, float* slot, int k, int64_t e, float scale) {
  pack4_body(f, slot, k, e, scale);
}
static __device__ __noinline__ void store4_ool(const FusedArgs& f, int k, int64_t e, float4 v) {
  store4_body(f, k, e, v);
}
template <int N>
__device__ __noinline__ void fold4_ool(const FusedArgs& f, const float* const* in, const int64_t* seg_end, int s, int k,
                                       int64_t e, float* own) {
  fold4_body<N>(f, in, seg_end, s, k, e, own);
}

template <bool kOol>
__device__ __forceinline__ void pack4_slow(const FusedArgs& f, float* slot, int k, int64_t e, float scale) {
  if constexpr (kOol) pack4_ool(f, slot, k, e, scale); else pack4_body(f, slot, k, e, scale);
}
template <bool kOol>
__device__ __forceinline__ void store4_slow(const FusedArgs& f, int k, int64_t e, float4 v) {
  if constexpr (kOol) store4_ool(f, k, e, v); else store4_body(f, k, e, v);
}
template <int N, bool kOol>
__device__ __forceinline__ void fold4_slow(const FusedArgs& f, const float* const* in, const int64_t* seg_end, int s,
                                           int k, int64_t e, float* own) {
  if constexpr (kOol) fold4_ool<N>(f, in, seg_end, s, k, e, own); else fold4_body<N>(f, in, seg_end, s, k, e, own);
}

// Pack bucket vectors [v0, v1) (16-B slots) plus scalar elements [t0, t1) into `slot`.
// UP slots per thread are loaded before any is stored (ncu r01: one outstanding 16-B load
// per thread left the pack phase latency-bound on long-scoreboard stalls).
template <bool kOol = false>
__device__ void fused_pack_range(const FusedArgs& f, float* slot, int64_t v0, int64_t v1, int64_t t0, int64_t t1) {
  constexpr int UP = 4;
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  if (v0 < v1) {
    int k = fused_row_covering(f, (v0 + threadIdx.x) << 2 < (v1 << 2) ? (v0 + threadIdx.x) << 2 : v0 << 2);
    for (int64_t base = v0 + threadIdx.x; base < v1; base += (int64_t)UP * kThreads) {
      float4 x[UP];
      float* tp[UP];
      bool fast[UP];
      int ku[UP];
#pragma unroll
      for (int u = 0; u < UP; ++u) {
        const int64_t vv = base + (int64_t)u * kThreads;
        fast[u] = false;
        ku[u] = k;
        if (vv < v1) {
          tp[u] = fused_tensor(f, k, vv << 2, fast[u]);
          ku[u] = k;
          if (fast[u]) x[u] = *reinterpret_cast<const float4*>(tp[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < UP; ++u) {
        const int64_t vv = base + (int64_t)u * kThreads;
        if (vv >= v1) continue;
        const int64_t e = vv << 2;
        if (fast[u])
          *reinterpret_cast<float4*>(slot + e) = scaled ? fmul4(x[u], scale) : x[u];
        else
          pack4_slow<kOol>(f, slot, ku[u], e, scale);
      }
    }
  }
  for (int64_t e = t0 + threadIdx.x; e < t1; e += kThreads) {
    const float x = *fused_tensor1(f, fused_row_covering(f, e), e);
    slot[e] = scaled ? __fmul_rn(x, scale) : x;
  }
}

// Fold bucket vectors [v0, v1) from the N slots (reference order); write to the
// tensors and, when `own` is non-null, to own[] as well.
template <int N, int U>
__device__ void fused_reduce_range(const FusedArgs& f, const float* const* in, const int64_t* seg_end, int64_t v0,
                                   int64_t v1, float* own) {
  if (v0 >= v1) return;
  int seg = advance_segment(0, (v0 + threadIdx.x) << 2 < (v1 << 2) ? (v0 + threadIdx.x) << 2 : v0 << 2, seg_end);
  int k = fused_row_covering(f, (v0 + threadIdx.x) << 2 < (v1 << 2) ? (v0 + threadIdx.x) << 2 : v0 << 2);
  for (int64_t base = v0 + threadIdx.x; base < v1; base += (int64_t)U * kThreads) {
    float4 x[U][N];
    int su[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vv = base + (int64_t)u * kThreads;
      ok[u] = false;
      su[u] = seg;
      if (vv < v1) {
        const int64_t e = vv << 2;
        seg = advance_segment(seg, e, seg_end);
        su[u] = seg;
        ok[u] = e + 3 < seg_end[seg];
        if (ok[u]) {
#pragma unroll
          for (int kk = 0; kk < N; ++kk) {
            const int src = seg + kk >= N ? seg + kk - N : seg + kk;
            x[u][kk] = __ldcg(reinterpret_cast<const float4*>(in[src] + e));
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vv = base + (int64_t)u * kThreads;
      if (vv >= v1) continue;
      const int64_t e = vv << 2;
      bool fast;
      float* tp = fused_tensor(f, k, e, fast);
      if (ok[u]) {
        float4 acc = x[u][0];
#pragma unroll
        for (int kk = 1; kk < N; ++kk) acc = fadd4(acc, x[u][kk]);
        if (own) *reinterpret_cast<float4*>(own + e) = acc;
        if (fast)
          *reinterpret_cast<float4*>(tp) = acc;
        else
          store4_slow<N == 1>(f, k, e, acc);
      } else {
        fold4_slow<N, N == 1>(f, in, seg_end, su[u], k, e, own);
      }
    }
  }
}

template <int N>
__device__ void fused_reduce_tail(const FusedArgs& f, const float* const* in, const int64_t* seg_end, int64_t e0,
                                  int64_t e1, float* own) {
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
    const int s = advance_segment(0, e, seg_end);
    const float y = fold1<N>(in, s, e);
    if (own) own[e] = y;
    *fused_tensor1(f, fused_row_covering(f, e), e) = y;
  }
}

// copy reduced bucket vectors [v0, v1) (and scalars [t0, t1)) of `src` into the tensors
static __device__ void fused_scatter_range(const FusedArgs& f, const float* src, int64_t v0, int64_t v1, int64_t t0,
                                    int64_t t1) {
  constexpr int UC = 4;
  if (v0 < v1) {
    int k = fused_row_covering(f, (v0 + threadIdx.x) << 2 < (v1 << 2) ? (v0 + threadIdx.x) << 2 : v0 << 2);
    for (int64_t base = v0 + threadIdx.x; base < v1; base += (int64_t)UC * kThreads) {
      float4 x[UC];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int64_t vv = base + (int64_t)u * kThreads;
        if (vv < v1) x[u] = __ldcg(reinterpret_cast<const float4*>(src) + vv);
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int64_t vv = base + (int64_t)u * kThreads;
        if (vv >= v1) continue;
        const int64_t e = vv << 2;
        bool fast;
        float* tp = fused_tensor(f, k, e, fast);
        if (fast)
          *reinterpret_cast<float4*>(tp) = x[u];
        else
          store4_slow<false>(f, k, e, x[u]);
      }
    }
  }
  for (int64_t e = t0 + threadIdx.x; e < t1; e += kThreads)
    *fused_tensor1(f, fused_row_covering(f, e), e) = __ldcg(src + e);
}

template <int N>
__device__ __forceinline__ void fused_oneshot_body(const FusedArgs& f, const int cta, const int ctas) {
  constexpr int U = Unroll<N>::value;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  MGW_EXPECT(a.slot_stride == 0 || a.n * 4 <= a.slot_stride);  // fp32 bucket fits its slot
  const int64_t nv = a.n >> 2;
  int64_t v0, v1;
  cta_chunk(0, nv, cta, ctas, v0, v1);
  const bool last = cta == ctas - 1;
  float* mine = const_cast<float*>(s_in[a.rank]);
  phase_mark(a, 0, cta);
  if (!(a.flags & kSkipPack)) fused_pack_range<N == 1>(f, mine, v0, v1, last ? nv << 2 : 0, last ? a.n : 0);
  phase_mark(a, 1, cta);
  int status = MGW_DEV_OK;
  if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, cta);
  phase_mark(a, 2, cta);
  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase1)) {
    fused_reduce_range<N, U>(f, s_in, s_end, v0, v1, nullptr);
    if (last) fused_reduce_tail<N>(f, s_in, s_end, nv << 2, a.n, nullptr);
  }
  phase_mark(a, 3, cta);
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(fused_oneshot, FusedArgs)

// Interleaved walk over chunk b of several parts: slot i of every part is handled in the
// same loop trip, so the parts' memory streams are in flight together (one round trip
// per trip instead of one per part).  `cur` are per-part monotone row cursors.
template <int N>
struct PartChunks {
  int64_t lo[N];   // first 16-B slot of chunk b in part p
  int64_t len[N];  // slots of chunk b in part p
  int64_t longest;
};

template <int N>
__device__ __forceinline__ void part_chunks(int64_t nv, int b, int G, PartChunks<N>& pc) {
  pc.longest = 0;
#pragma unroll
  for (int p = 0; p < N; ++p) {
    int64_t c0, c1;
    cta_chunk(part_begin(p, nv, N), part_begin(p + 1, nv, N), b, G, c0, c1);
    pc.lo[p] = c0;
    pc.len[p] = c1 > c0 ? c1 - c0 : 0;
    pc.longest = pc.len[p] > pc.longest ? pc.len[p] : pc.longest;
  }
}

// pack chunk b of every part into my slot, parts interleaved
template <int N>
__device__ void fused_pack_parts(const FusedArgs& f, float* slot, const PartChunks<N>& pc) {
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  int cur[N];
#pragma unroll
  for (int p = 0; p < N; ++p) cur[p] = fused_row_covering(f, (pc.lo[p] + (threadIdx.x < pc.len[p] ? threadIdx.x : 0)) << 2);
  constexpr int PB = N <= 4 ? N : 4;  // parts per batch of loads in flight (N = 7, 8 spilled)
  for (int64_t i = threadIdx.x; i < pc.longest; i += kThreads) {
#pragma unroll
    for (int pb = 0; pb < N; pb += PB) {
      float4 x[PB];
      bool fast[PB];
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        const int p = pb + q;
        fast[q] = false;
        if (p < N && i < pc.len[p]) {
          const float* tp = fused_tensor(f, cur[p], (pc.lo[p] + i) << 2, fast[q]);
          if (fast[q]) x[q] = *reinterpret_cast<const float4*>(tp);
        }
      }
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        const int p = pb + q;
        if (p >= N || i >= pc.len[p]) continue;
        const int64_t e = (pc.lo[p] + i) << 2;
        if (fast[q])
          *reinterpret_cast<float4*>(slot + e) = scaled ? fmul4(x[q], scale) : x[q];
        else
          pack4_slow<false>(f, slot, cur[p], e, scale);
      }
    }
  }
}

// copy chunk b of every peer's reduced part from its slot into my tensors, interleaved
template <int N>
__device__ void fused_scatter_parts(const FusedArgs& f, const float* const* in, int me, const PartChunks<N>& pc) {
  int cur[N];
#pragma unroll
  for (int p = 0; p < N; ++p) cur[p] = fused_row_covering(f, (pc.lo[p] + (threadIdx.x < pc.len[p] ? threadIdx.x : 0)) << 2);
  for (int64_t i = threadIdx.x; i < pc.longest; i += kThreads) {
    float4 x[N];
#pragma unroll
    for (int p = 0; p < N; ++p)
      if (p != me && i < pc.len[p]) x[p] = __ldcg(reinterpret_cast<const float4*>(in[p]) + pc.lo[p] + i);
#pragma unroll
    for (int p = 0; p < N; ++p) {
      if (p == me || i >= pc.len[p]) continue;
      const int64_t e = (pc.lo[p] + i) << 2;
      bool fast;
      float* tp = fused_tensor(f, cur[p], e, fast);
      if (fast)
        *reinterpret_cast<float4*>(tp) = x[p];
      else
        store4_slow<false>(f, cur[p], e, x[p]);
    }
  }
}

template <int N>
__device__ __forceinline__ void fused_twoshot_body(const FusedArgs& f, const int cta, const int ctas) {
  constexpr int U = Unroll<N>::value;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  MGW_EXPECT(a.slot_stride == 0 || a.n * 4 <= a.slot_stride);  // fp32 bucket fits its slot
  const int me = a.rank;
  const int b = cta, G = ctas;
  const int64_t nv = a.n >> 2;
  const bool last = b == G - 1;
  const int64_t tail0 = nv << 2;
  float* mine = const_cast<float*>(s_in[me]);
  __shared__ PartChunks<N> pc;  // CTA-uniform: keep it out of the registers
  if (threadIdx.x == 0) part_chunks<N>(nv, b, G, pc);
  __syncthreads();
  phase_mark(a, 0, cta);
  if (!(a.flags & kSkipPack)) {
    fused_pack_parts<N>(f, mine, pc);
    if (last) fused_pack_range(f, mine, 0, 0, tail0, a.n);  // the n % 4 tail (part N-1)
  }
  phase_mark(a, 1, cta);
  int status = MGW_DEV_OK;
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, cta);
    phase_mark(a, 2, cta);
    if (status == MGW_DEV_OK) {
      fused_reduce_range<N, U>(f, s_in, s_end, pc.lo[me], pc.lo[me] + pc.len[me], mine);
      if (last && me == N - 1) fused_reduce_tail<N>(f, s_in, s_end, tail0, a.n, mine);
    }
    phase_mark(a, 3, cta);
  }
  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase2)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.mid, parity, epoch, a.tag, a, cta);
    phase_mark(a, 4, cta);
    if (status == MGW_DEV_OK) {
      fused_scatter_parts<N>(f, s_in, me, pc);
      if (last && me != N - 1) fused_scatter_range(f, s_in[N - 1], 0, 0, tail0, a.n);
    }
    phase_mark(a, 5, cta);
  }
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(fused_twoshot, FusedArgs)

}  // namespace mgw
