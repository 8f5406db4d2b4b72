// b16push.cuh -- push two-shot for bf16 gradients with fp32 accumulation: push.cuh's
// store-only exchange on bf16.cuh's format (same bits as the bf16 pull kernels and the
// oracle ring_allreduce_bf16: the reference ring's fold order, allreduce_net.py:370-411, in
// fp32 over exactly-upcast inputs, scaled and rounded once by the part's owner).
//
//   phase 1  CTA b copies chunk b of every part p from the layer tensors (bf16) into rank p's
//            incoming row `me`                                            -> barrier
//   phase 2  CTA b folds chunk b of its own part from the N local rows in the reference
//            order (fp32), rounds once, writes its tensors and stores the bf16 result into
//            every peer's gather area                                     -> barrier
//   phase 3  CTA b copies chunk b of every peer part from its local gather area into its
//            tensors.
//
// Every NVLink byte is a store (2 (N-1)/N x M out per rank); all loads are local.  Rows:
// slot[parity] of each rank viewed as bf16 [N src][stride], stride = one part of 16-B slots
// (8 bf16, + kPartAlign for part_begin's rounding) + the n % 8 tail; gather area = the second capacity pair of the IPC region.
#pragma once

#include "bf16.cuh"
#include "push.cuh"

namespace mgw {

__host__ __device__ __forceinline__ int64_t b16_push_stride(int64_t n, int world) {
  return ((n / kB16 + world - 1) / world + kPartAlign + 1) * kB16;  // as push_stride()
}

template <int N>
__device__ __forceinline__ void b16_push_body(const PushArgs& x, const int cta, const int ctas) {
  const FusedArgs& f = x.f;
  const ArArgs& a = f.ar;
  __shared__ const float* s_in[kMaxRanks];  // incoming area of every rank (this parity)
  __shared__ int64_t s_end[kMaxRanks];
  __shared__ uint16_t* s_gat[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  if (threadIdx.x < N)
    s_gat[threadIdx.x] = reinterpret_cast<uint16_t*>(x.gather[threadIdx.x] + (int64_t)parity * a.slot_stride);
  const int me = a.rank;
  const int64_t nv = a.n / kB16;
  const bool last = cta == ctas - 1;
  const int64_t tail0 = nv * kB16;
  const int64_t stride = x.stride;  // bf16 elements per incoming row
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  __shared__ PartChunks<N> pc;
  __shared__ int64_t s_part0[kMaxRanks + 1];  // first element of every part
  if (threadIdx.x == 0) part_chunks<N>(nv, cta, ctas, pc);
  if (threadIdx.x <= N) s_part0[threadIdx.x] = part_begin(threadIdx.x, nv, N) * kB16;
  __syncthreads();
  MGW_EXPECT(a.slot_stride == 0 || (int64_t)N * stride * 2 <= a.slot_stride);
  auto row = [&](int p) { return reinterpret_cast<uint16_t*>(const_cast<float*>(s_in[p])); };

  // ---- phase 1: copy chunk b of every part p into rank p's incoming row `me`
  if (!(a.flags & kSkipPack)) {
    int cur[N];
#pragma unroll
    for (int p = 0; p < N; ++p)
      cur[p] = fused_row_covering(f, (pc.lo[p] + (threadIdx.x < pc.len[p] ? threadIdx.x : 0)) * kB16);
    constexpr int PB = N <= 4 ? N : 4;  // parts per batch of loads in flight
    for (int64_t i = threadIdx.x; i < pc.longest; i += kThreads) {
#pragma unroll
      for (int pb = 0; pb < N; pb += PB) {
        uint4 v[PB];
        bool fast[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          const int p = pb + q;
          fast[q] = false;
          if (p < N && i < pc.len[p]) {
            const uint16_t* tp = b16_tensor(f, cur[p], (pc.lo[p] + i) * kB16, fast[q]);
            if (fast[q]) v[q] = *reinterpret_cast<const uint4*>(tp);
          }
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          const int p = pb + q;
          if (p >= N || i >= pc.len[p]) continue;
          const int64_t e = (pc.lo[p] + i) * kB16;
          uint16_t* dst = row(p) + (int64_t)me * stride + (e - s_part0[p]);
          MGW_EXPECT(e >= s_part0[p] && e + kB16 <= s_part0[p] + stride);
          if (fast[q])
            *reinterpret_cast<uint4*>(dst) = v[q];
          else
            for (int j = 0; j < kB16; ++j) dst[j] = *b16_tensor1(f, cur[p], e + j);
        }
      }
    }
    if (last) {  // the n % 8 tail belongs to part N-1
      uint16_t* dst = row(N - 1) + (int64_t)me * stride - s_part0[N - 1];
      for (int64_t e = tail0 + threadIdx.x; e < a.n; e += kThreads) dst[e] = *b16_tensor1(f, fused_row_covering(f, e), e);
    }
  }
  int status = MGW_DEV_OK;
  // ---- phase 2: fold my part's chunk b from the N local rows, write my tensors and every
  //      peer's gather area
  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, cta);
    if (status == MGW_DEV_OK) {
      const uint16_t* in = row(me);
      const int64_t p0 = s_part0[me];
      const int64_t v0 = pc.lo[me], v1 = pc.lo[me] + pc.len[me];
      int seg = advance_segment(0, (v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0) * kB16, s_end);
      int k = fused_row_covering(f, (v0 + threadIdx.x < v1 ? v0 + threadIdx.x : v0) * kB16);
      for (int64_t v = v0 + threadIdx.x; v < v1; v += kThreads) {
        const int64_t e = v * kB16;
        const int64_t o = e - p0;
        seg = advance_segment(seg, e, s_end);
        uint4 y;
        if (e + kB16 - 1 < s_end[seg]) {
          uint4 xs[N];
#pragma unroll
          for (int kk = 0; kk < N; ++kk) {
            const int src = seg + kk >= N ? seg + kk - N : seg + kk;
            xs[kk] = __ldcg(reinterpret_cast<const uint4*>(in + (int64_t)src * stride + o));
          }
          y = b16_fold8<N>(xs, scale, scaled);
        } else {  // the slot straddles a segment boundary: element by element
          uint32_t w[4] = {0u, 0u, 0u, 0u};
          int s = seg;
          for (int j = 0; j < kB16; ++j) {
            s = advance_segment(s, e + j, s_end);
            float acc = b16_to_f32(__ldcg(in + (int64_t)s * stride + o + j));
            for (int kk = 1; kk < N; ++kk) {
              const int src = s + kk >= N ? s + kk - N : s + kk;
              acc = __fadd_rn(acc, b16_to_f32(__ldcg(in + (int64_t)src * stride + o + j)));
            }
            w[j >> 1] |= (uint32_t)f32_to_b16(scaled ? __fmul_rn(acc, scale) : acc) << ((j & 1) * 16);
          }
          y = make_uint4(w[0], w[1], w[2], w[3]);
        }
#pragma unroll
        for (int q = 0; q < N; ++q)
          if (q != me) *reinterpret_cast<uint4*>(s_gat[q] + e) = y;
        bool fast;
        uint16_t* tp = b16_tensor(f, k, e, fast);
        if (fast) {
          *reinterpret_cast<uint4*>(tp) = y;
        } else {
          const uint16_t* h = reinterpret_cast<const uint16_t*>(&y);
          for (int j = 0; j < kB16; ++j) *b16_tensor1(f, k, e + j) = h[j];
        }
      }
      if (last && me == N - 1) {
        for (int64_t e = tail0 + threadIdx.x; e < a.n; e += kThreads) {
          const int64_t o = e - p0;
          const int s = advance_segment(0, e, s_end);
          float acc = b16_to_f32(__ldcg(in + (int64_t)s * stride + o));
          for (int kk = 1; kk < N; ++kk) {
            const int src = s + kk >= N ? s + kk - N : s + kk;
            acc = __fadd_rn(acc, b16_to_f32(__ldcg(in + (int64_t)src * stride + o)));
          }
          const uint16_t y = f32_to_b16(scaled ? __fmul_rn(acc, scale) : acc);
          for (int q = 0; q < N; ++q)
            if (q != me) s_gat[q][e] = y;
          *b16_tensor1(f, fused_row_covering(f, e), e) = y;
        }
      }
    }
  }
  // ---- phase 3: copy chunk b of every peer part from my gather area into my tensors
  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase2)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.mid, parity, epoch, a.tag, a, cta);
    if (status == MGW_DEV_OK) {
      const uint16_t* g = s_gat[me];
      for (int p = 0; p < N; ++p)
        if (p != me) b16_scatter_range(f, g, pc.lo[p], pc.lo[p] + pc.len[p], 0, 0);
      if (last && me != N - 1) b16_scatter_range(f, g, 0, 0, tail0, a.n);
    }
  }
  finish_call(a, ctas);
}

MGW_DEFINE_KERNELS(b16_push, PushArgs)

}  // namespace mgw
