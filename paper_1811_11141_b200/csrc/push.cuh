// push.cuh -- push-based group exchanges: two-shot (pack -> reduce-scatter -> all-gather
// -> unpack in one kernel) for large buckets, one-shot for mid-size ones.  Same result as
// ring_allreduce (allreduce_net.py:370-411) on the group bucket (:499-509).
//
// The pull two-shot (fused.cuh) pays a remote-read round trip in each of its phases:
// every load from a peer slot waits ~2 us for NVLink.  Here every byte crosses NVLink
// as a *store* (fire-and-forget, pipelined by the fabric) and every load is local:
//
//   phase 1  CTA b reads chunk b of every part p from the layer tensors (scaled) and
//            stores it into rank p's incoming area, row `me`             -> barrier
//   phase 2  CTA b folds chunk b of its own part from the N local incoming rows in the
//            reference order (fold start = the element's `_segments` segment), writes
//            the result to its own tensors and stores it into every peer's gather
//            area at the bucket offset                                      -> barrier
//   phase 3  CTA b copies chunk b of every peer part from its local gather area into
//            its tensors.
//
// Same bits as the pull kernels (same fp32 adds in the same order).  Incoming area =
// slot[parity] of each rank viewed as [N src][stride] (stride = one part + tail), gather
// area = a second pair of capacity-sized buffers in the IPC region.  Reuse distance 2 by
// parity, as for the slots: a peer can only store into my area of call k + 2 after its
// CTA b passed the call k + 1 barrier with my CTA b, i.e. after my call k finished.
#pragma once

#include "fused.cuh"

namespace mgw {

struct PushArgs {
  FusedArgs f;                 // f.ar.slot[r] = rank r's slot 0 (incoming area for parity 0)
  char* gather[kMaxRanks];     // rank r's gather area 0 (parity 1 follows at f.ar.slot_stride)
  int64_t stride;              // incoming row stride in elements (multiple of 4)
  uint64_t* pipe[kMaxRanks];   // pipelined two-shot (pipe.cuh): rank r's sub-chunk flags
  int subs;                    // pipelined two-shot: sub-chunks per CTA chunk
};

// incoming row stride in floats: the longest part (ceil(nv / world) + kPartAlign slots,
// part_begin rounds down) + one slot for the n % 4 tail
__host__ __device__ __forceinline__ int64_t push_stride(int64_t nv, int world) {
  return ((nv + world - 1) / world + kPartAlign + 1) * 4;
}

template <int N>
__device__ __forceinline__ void push_twoshot_body(const PushArgs& x, const int cta, const int ctas) {
  const FusedArgs& f = x.f;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];  // incoming area of every rank (this parity)
  __shared__ int64_t s_end[kMaxRanks];
  __shared__ float* s_gat[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  if (threadIdx.x < N) s_gat[threadIdx.x] = reinterpret_cast<float*>(x.gather[threadIdx.x] + (int64_t)parity * a.slot_stride);
  const int me = a.rank;
  const int b = cta, G = ctas;
  const int64_t nv = a.n >> 2;
  const bool last = b == G - 1;
  const int64_t tail0 = nv << 2;
  const int64_t stride = x.stride;
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  __shared__ PartChunks<N> pc;
  __shared__ int64_t s_part0[kMaxRanks + 1];  // first element of every part
  if (threadIdx.x == 0) part_chunks<N>(nv, b, G, pc);
  if (threadIdx.x <= N) s_part0[threadIdx.x] = part_begin(threadIdx.x, nv, N) << 2;
  __syncthreads();

  phase_mark(a, 0, cta);
  // ---- phase 1: push chunk b of every part p into rank p's incoming row `me`
  if (!(a.flags & kSkipPack)) {
    int cur[N];
#pragma unroll
    for (int p = 0; p < N; ++p)
      cur[p] = fused_row_covering(f, (pc.lo[p] + (threadIdx.x < pc.len[p] ? threadIdx.x : 0)) << 2);
    // parts in batches of at most PB loads in flight: N = 8 with all parts at once
    // overflowed the 64 registers of the (512, 2) launch bounds and spilled
    constexpr int PB = N <= 4 ? N : 4;
    for (int64_t i = threadIdx.x; i < pc.longest; i += kThreads) {
#pragma unroll
      for (int pb = 0; pb < N; pb += PB) {
        float4 v[PB];
        bool fast[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          const int p = pb + q;
          fast[q] = false;
          if (p < N && i < pc.len[p]) {
            const float* tp = fused_tensor(f, cur[p], (pc.lo[p] + i) << 2, fast[q]);
            if (fast[q]) v[q] = *reinterpret_cast<const float4*>(tp);
          }
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          const int p = pb + q;
          if (p >= N || i >= pc.len[p]) continue;
          const int64_t e = (pc.lo[p] + i) << 2;
          float* dst = const_cast<float*>(s_in[p]) + (int64_t)me * stride + (e - s_part0[p]);
          MGW_EXPECT(e >= s_part0[p] && e + 4 <= s_part0[p] + stride &&
                     (a.slot_stride == 0 || (int64_t)N * stride * 4 <= a.slot_stride));
          if (fast[q])
            *reinterpret_cast<float4*>(dst) = scaled ? fmul4(v[q], scale) : v[q];
          else
            pack4_slow<false>(f, dst - e, cur[p], e, scale);  // dst - e: the row base, indexed by e
        }
      }
    }
    if (last) {  // the n % 4 tail belongs to part N-1
      float* dst = const_cast<float*>(s_in[N - 1]) + (int64_t)me * stride - s_part0[N - 1];
      for (int64_t e = tail0 + threadIdx.x; e < a.n; e += kThreads) {
        const float y = *fused_tensor1(f, fused_row_covering(f, e), e);
        dst[e] = scaled ? __fmul_rn(y, scale) : y;
      }
    }
  }
  phase_mark(a, 1, cta);
  int status = MGW_DEV_OK;
  // ---- phase 2: fold my part's chunk b from the N local rows, write my tensors, push
  //      the result into every peer's gather area
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, cta);
    phase_mark(a, 2, cta);
    if (status == MGW_DEV_OK) {
      const float* in = s_in[me];
      const int64_t p0 = s_part0[me];
      const int64_t v0 = pc.lo[me], v1 = pc.lo[me] + pc.len[me];
      int seg = advance_segment(0, (v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0) << 2, s_end);
      int k = fused_row_covering(f, (v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0) << 2);
      for (int64_t v = v0 + threadIdx.x; v < v1; v += kThreads) {
        const int64_t e = v << 2;
        const int64_t o = e - p0;
        seg = advance_segment(seg, e, s_end);
        float4 y;
        if (e + 3 < s_end[seg]) {
          float4 xs[N];
#pragma unroll
          for (int kk = 0; kk < N; ++kk) {
            const int src = seg + kk >= N ? seg + kk - N : seg + kk;
            xs[kk] = __ldcg(reinterpret_cast<const float4*>(in + (int64_t)src * stride + o));
          }
          y = xs[0];
#pragma unroll
          for (int kk = 1; kk < N; ++kk) y = fadd4(y, xs[kk]);
        } else {  // the slot straddles a segment boundary
          float r[4];
          int s = seg;
          for (int j = 0; j < 4; ++j) {
            s = advance_segment(s, e + j, s_end);
            float acc = __ldcg(in + (int64_t)s * stride + o + j);
            for (int kk = 1; kk < N; ++kk) {
              const int src = s + kk >= N ? s + kk - N : s + kk;
              acc = __fadd_rn(acc, __ldcg(in + (int64_t)src * stride + o + j));
            }
            r[j] = acc;
          }
          y = make_float4(r[0], r[1], r[2], r[3]);
        }
#pragma unroll
        for (int q = 0; q < N; ++q)
          if (q != me) *reinterpret_cast<float4*>(s_gat[q] + e) = y;
        bool fast;
        float* tp = fused_tensor(f, k, e, fast);
        if (fast) {
          *reinterpret_cast<float4*>(tp) = y;
        } else {
          const float r[4] = {y.x, y.y, y.z, y.w};
          for (int j = 0; j < 4; ++j) *fused_tensor1(f, k, e + j) = r[j];
        }
      }
      if (last && me == N - 1) {
        for (int64_t e = tail0 + threadIdx.x; e < a.n; e += kThreads) {
          const int64_t o = e - p0;
          const int s = advance_segment(0, e, s_end);
          float acc = __ldcg(in + (int64_t)s * stride + o);
          for (int kk = 1; kk < N; ++kk) {
            const int src = s + kk >= N ? s + kk - N : s + kk;
            acc = __fadd_rn(acc, __ldcg(in + (int64_t)src * stride + o));
          }
          for (int q = 0; q < N; ++q)
            if (q != me) s_gat[q][e] = acc;
          *fused_tensor1(f, fused_row_covering(f, e), e) = acc;
        }
      }
    }
  }
  phase_mark(a, 3, cta);
  // ---- phase 3: copy chunk b of every peer part from my gather area into my tensors
  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase2)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.mid, parity, epoch, a.tag, a, cta);
    phase_mark(a, 4, cta);
    if (status == MGW_DEV_OK) {
      const float* g = s_gat[me];
      for (int p = 0; p < N; ++p)
        if (p != me) fused_scatter_range(f, g, pc.lo[p], pc.lo[p] + pc.len[p], 0, 0);
      if (last && me != N - 1) fused_scatter_range(f, g, 0, 0, tail0, a.n);
    }
    phase_mark(a, 5, cta);
  }
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(push_twoshot, PushArgs)

// Push one-shot: CTA b stores chunk b of its (scaled) bucket into row `me` of every
// rank's incoming area (x.gather[r], rows of `stride` = n rounded to 16 B), one barrier,
// then folds chunk b from the N local rows in the reference order into its tensors.
// (N-1)·M NVLink bytes out per rank, all as stores; no remote loads.
template <int N>
__device__ __forceinline__ void push_oneshot_body(const PushArgs& x, const int cta, const int ctas) {
  constexpr int U = Unroll<N>::value;
  const FusedArgs& f = x.f;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];  // unused slots (prologue computes them)
  __shared__ int64_t s_end[kMaxRanks];
  __shared__ float* s_row[kMaxRanks];       // rank r's incoming area (this parity)
  __shared__ const float* s_mine[kMaxRanks];  // my incoming rows, one per source
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  const int me = a.rank;
  const int64_t stride = x.stride;
  if (threadIdx.x < N) {
    s_row[threadIdx.x] = reinterpret_cast<float*>(x.gather[threadIdx.x] + (int64_t)parity * a.slot_stride);
    s_mine[threadIdx.x] =
        reinterpret_cast<const float*>(x.gather[me] + (int64_t)parity * a.slot_stride) + (int64_t)threadIdx.x * stride;
  }
  __syncthreads();
  const int64_t nv = a.n >> 2;
  int64_t v0, v1;
  cta_chunk(0, nv, cta, ctas, v0, v1);
  const bool last = cta == ctas - 1;
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  phase_mark(a, 0, cta);
  // ---- push chunk b of my bucket into row `me` of every rank
  if (!(a.flags & kSkipPack)) {
    constexpr int UP = 4;
    if (v0 < v1) {
      int k = fused_row_covering(f, (v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0) << 2);
      for (int64_t base = v0 + threadIdx.x; base < v1; base += (int64_t)UP * kThreads) {
        float4 v[UP];
        bool fast[UP];
        int ku[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          const int64_t vv = base + (int64_t)u * kThreads;
          fast[u] = false;
          ku[u] = k;
          if (vv < v1) {
            const float* tp = fused_tensor(f, k, vv << 2, fast[u]);
            ku[u] = k;
            if (fast[u]) v[u] = *reinterpret_cast<const float4*>(tp);
          }
        }
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          const int64_t vv = base + (int64_t)u * kThreads;
          if (vv >= v1) continue;
          const int64_t e = vv << 2;
          if (!fast[u]) {
            float r[4];
            for (int j = 0; j < 4; ++j) r[j] = *fused_tensor1(f, ku[u], e + j);
            v[u] = make_float4(r[0], r[1], r[2], r[3]);
          }
          if (scaled) v[u] = fmul4(v[u], scale);
          MGW_EXPECT(e + 4 <= stride && (a.slot_stride == 0 || (int64_t)N * stride * 4 <= a.slot_stride));
#pragma unroll
          for (int q = 0; q < N; ++q) *reinterpret_cast<float4*>(s_row[q] + (int64_t)me * stride + e) = v[u];
        }
      }
    }
    if (last) {
      for (int64_t e = (nv << 2) + threadIdx.x; e < a.n; e += kThreads) {
        float y = *fused_tensor1(f, fused_row_covering(f, e), e);
        if (scaled) y = __fmul_rn(y, scale);
        for (int q = 0; q < N; ++q) s_row[q][(int64_t)me * stride + e] = y;
      }
    }
  }
  phase_mark(a, 1, cta);
  int status = MGW_DEV_OK;
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, cta);
    phase_mark(a, 2, cta);
    if (status == MGW_DEV_OK) {
      // fold chunk b from the N local rows (they play the slots of fused_reduce_range)
      fused_reduce_range<N, U>(f, s_mine, s_end, v0, v1, nullptr);
      if (last) fused_reduce_tail<N>(f, s_mine, s_end, nv << 2, a.n, nullptr);
    }
    phase_mark(a, 3, cta);
  }
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(push_oneshot, PushArgs)

}  // namespace mgw
