// pipe.cuh -- pipelined push two-shot for large buckets: the same reduce-scatter /
// all-gather as push.cuh (same bits: ring_allreduce's fold order, allreduce_net.py:
// 370-411, on the group bucket :499-509), with the two whole-chunk barriers replaced by
// per-sub-chunk flags so the phases of consecutive sub-chunks overlap.
//
// push.cuh's phase probe (profiles/phases_n4_r02.json, 16 MiB at N = 4) spends 28 of 56 us
// in its two barriers: a CTA cannot fold before the slowest peer CTA has pushed its whole
// chunk, nor gather before the slowest peer has folded its whole part.  Here CTA b cuts its
// chunk of every part into S sub-chunks and runs a three-stage software pipeline:
//
//   iteration i:  A  push sub-chunk i of every part p to rank p's incoming row `me`,
//                    then flag "pushed (b, i)" to every peer
//                 B  wait until every peer flagged "pushed (b, i-1)"; fold sub-chunk i-1
//                    of my part from the N local rows (reference fold order), write my
//                    tensors, store the result into every peer's gather area, flag
//                    "gathered (b, i-1)" to every peer
//                 C  wait until every peer p flagged "gathered (b, i-2)"; copy sub-chunk
//                    i-2 of every peer part from my gather area into my tensors
//
// so the NVLink stores of stage A (sub-chunk i) and B (sub-chunk i-1) are in flight
// together and a late peer delays one sub-chunk, not the whole chunk.  Deadlock-free:
// within an iteration every signal precedes every wait, and the waits of iteration i need
// only signals of iterations <= i-1.  Thread t handles the same slots (t, t + 512, ...) of a
// sub-chunk in all three stages on every rank, so warp w only ever waits for warp w of its
// peers: flags are per warp, the pipeline has no CTA-wide barrier, and while one warp's
// release fence waits for its NVLink stores to land the other 15 keep issuing (a CTA-wide
// flag stalled the whole CTA for a round trip per sub-chunk stage -- 2x slower, measured).
// Flags: (epoch << 32 | collective tag) at pipe[r][kind][parity][b][warp][sub][src], reuse
// distance 2 by parity as for the barrier flags.
#pragma once

#include "push.cuh"

namespace mgw {

constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ size_t pipe_index(int kind, int parity, int cta, int warp, int sub, int src) {
  return (((((size_t)kind * 2 + parity) * kMaxBlocks + cta) * kWarps + warp) * kPipeSub + sub) * kMaxRanks + src;
}

// this warp's stage `kind` of sub-chunk `sub` is done: tell every peer (its stores first)
__device__ __forceinline__ void pipe_signal(const PushArgs& x, int kind, int parity, int cta, int sub, uint64_t word) {
  __syncwarp();  // orders the warp's data stores before the release below
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < x.f.ar.world && lane != x.f.ar.rank)
    store_release_sys(x.pipe[lane] + pipe_index(kind, parity, cta, warp, sub, x.f.ar.rank), word);
}

// wait until the same warp of every peer's CTA `cta` signalled stage `kind` of `sub`
static __device__ __noinline__ int pipe_wait(const PushArgs& x, int kind, int parity, int cta, int sub, uint32_t epoch) {
  const ArArgs& a = x.f.ar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int status = MGW_DEV_OK;
  if (lane < a.world && lane != a.rank) {
    const uint64_t* mine = x.pipe[a.rank] + pipe_index(kind, parity, cta, warp, sub, lane);
    const uint64_t start = global_ns();
    for (uint32_t spin = 0;; ++spin) {
      const uint64_t v = load_acquire_sys(mine);
      if ((uint32_t)(v >> 32) == epoch) {
        if ((uint32_t)v != a.tag) status = MGW_DEV_MISMATCH;
        break;
      }
      if ((spin & 63) == 63) {
        if (load_relaxed_sys32(a.abort_flag[a.rank]) != 0u) {
          status = MGW_DEV_PEER_ABORT;
          break;
        }
        if (global_ns() - start > a.timeout_ns) {
          status = MGW_DEV_TIMEOUT;
          break;
        }
      }
    }
  }
  // the warp agrees on the worst status (max: MISMATCH 1 < TIMEOUT 2 < PEER_ABORT 3 -- any
  // non-zero stops the warp) and orders its later reads after the acquiring lanes' loads
  status = __reduce_max_sync(0xffffffffu, status);
  if (status != MGW_DEV_OK && lane == 0) {
    atomicCAS(a.err, 0, status);
    if (status != MGW_DEV_PEER_ABORT)
      for (int r = 0; r < a.world; ++r) store_release_sys32(a.abort_flag[r], 1u);
  }
  return status;
}

template <int N>
__device__ __forceinline__ void push_pipe_body(const PushArgs& x, const int cta, const int ctas) {
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
  const int64_t nv = a.n >> 2;
  const bool last = cta == ctas - 1;
  const int64_t tail0 = nv << 2;
  const int64_t stride = x.stride;
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  const int S = x.subs;
  const bool sync = !(a.flags & kNoBarrier);
  const bool do_push = !(a.flags & kSkipPack), do_fold = !(a.flags & kSkipPhase1), do_gather = !(a.flags & kSkipPhase2);
  const uint64_t word = ((uint64_t)epoch << 32) | a.tag;
  __shared__ PartChunks<N> pc;
  __shared__ int64_t s_part0[kMaxRanks + 1];  // first element of every part
  if (threadIdx.x == 0) part_chunks<N>(nv, cta, ctas, pc);
  if (threadIdx.x <= N) s_part0[threadIdx.x] = part_begin(threadIdx.x, nv, N) << 2;
  __syncthreads();
  MGW_EXPECT(S >= 1 && S <= kPipeSub && (a.slot_stride == 0 || (int64_t)N * stride * 4 <= a.slot_stride));
  // sub-chunk j of part p: slots [s_sub[p][j], s_sub[p][j + 1]) (shared: the bounds stay out of
  // the registers); thread t always handles the slots t, t + 512, ... of a sub-chunk in every
  // stage, so warp w depends only on warp w of every peer (per-warp flags: no CTA-wide
  // barrier inside the pipeline)
  __shared__ int64_t s_sub[kMaxRanks][kPipeSub + 1];
  if (threadIdx.x < N * (S + 1)) {
    const int p = threadIdx.x / (S + 1), j = threadIdx.x % (S + 1);
    s_sub[p][j] = pc.lo[p] + pc.len[p] * j / S;
  }
  __syncthreads();
  auto sub_lo = [&](int p, int j) { return s_sub[p][j]; };
  constexpr int PB = N <= 4 ? N : 4;  // parts per batch of loads in flight

  int status = MGW_DEV_OK;
  for (int it = 0; it < S + 2 && status == MGW_DEV_OK; ++it) {
    // ---- A: push sub-chunk `it` of every part p into rank p's incoming row `me`
    if (do_push && it < S) {
#pragma unroll
      for (int pb = 0; pb < N; pb += PB) {
        int64_t longest = 0;
        int cur[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          const int p = pb + q < N ? pb + q : N - 1;
          const int64_t len = pb + q < N ? sub_lo(p, it + 1) - sub_lo(p, it) : 0;
          longest = len > longest ? len : longest;
          cur[q] = fused_row_covering(f, (sub_lo(p, it) + (threadIdx.x < len ? threadIdx.x : 0)) << 2);
        }
        for (int64_t i = threadIdx.x; i < longest; i += kThreads) {
          float4 v[PB];
          bool fast[PB];
#pragma unroll
          for (int q = 0; q < PB; ++q) {
            fast[q] = false;
            const int p = pb + q < N ? pb + q : N - 1;
            if (pb + q < N && i < sub_lo(p, it + 1) - sub_lo(p, it)) {
              const float* tp = fused_tensor(f, cur[q], (sub_lo(p, it) + i) << 2, fast[q]);
              if (fast[q]) v[q] = *reinterpret_cast<const float4*>(tp);
            }
          }
#pragma unroll
          for (int q = 0; q < PB; ++q) {
            const int p = pb + q;
            if (p >= N || i >= sub_lo(p, it + 1) - sub_lo(p, it)) continue;
            const int64_t e = (sub_lo(p, it) + i) << 2;
            float* dst = const_cast<float*>(s_in[p]) + (int64_t)me * stride + (e - s_part0[p]);
            MGW_EXPECT(e >= s_part0[p] && e + 4 <= s_part0[p] + stride);
            if (fast[q])
              *reinterpret_cast<float4*>(dst) = scaled ? fmul4(v[q], scale) : v[q];
            else
              pack4_slow<false>(f, dst - e, cur[q], e, scale);  // dst - e: the row base, indexed by e
          }
        }
      }
      if (last && it == S - 1) {  // the n % 4 tail belongs to part N-1 (threads 0..2: warp 0)
        float* dst = const_cast<float*>(s_in[N - 1]) + (int64_t)me * stride - s_part0[N - 1];
        for (int64_t e = tail0 + threadIdx.x; e < a.n; e += kThreads) {
          const float y = *fused_tensor1(f, fused_row_covering(f, e), e);
          dst[e] = scaled ? __fmul_rn(y, scale) : y;
        }
      }
      if (sync) pipe_signal(x, 0, parity, cta, it, word);
    }
    // ---- B: fold sub-chunk it-1 of my part, write my tensors and every peer's gather area
    const int jb = it - 1;
    if (do_fold && jb >= 0 && jb < S) {
      if (sync) status = pipe_wait(x, 0, parity, cta, jb, epoch);
      if (status != MGW_DEV_OK) break;
      const float* in = s_in[me];
      const int64_t p0 = s_part0[me];
      const int64_t v0 = sub_lo(me, jb), v1 = sub_lo(me, jb + 1);
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
        if (fast)
          *reinterpret_cast<float4*>(tp) = y;
        else
          store4_slow<false>(f, k, e, y);
      }
      if (last && me == N - 1 && jb == S - 1) {
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
      if (sync) pipe_signal(x, 1, parity, cta, jb, word);
    }
    // ---- C: copy sub-chunk it-2 of every peer part from my gather area into my tensors
    const int jc = it - 2;
    if (do_gather && jc >= 0) {
      if (sync) status = pipe_wait(x, 1, parity, cta, jc, epoch);
      if (status != MGW_DEV_OK) break;
      const float* g = s_gat[me];
      for (int p = 0; p < N; ++p)
        if (p != me) fused_scatter_range(f, g, sub_lo(p, jc), sub_lo(p, jc + 1), 0, 0);
      if (last && me != N - 1 && jc == S - 1) fused_scatter_range(f, g, 0, 0, tail0, a.n);
    }
  }
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(push_pipe, PushArgs)

}  // namespace mgw
