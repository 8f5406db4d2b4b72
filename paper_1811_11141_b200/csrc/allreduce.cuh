// allreduce.cuh -- K2 one-shot and K3 two-shot all-reduce over CUDA-IPC peer memory.
//
// Fold order (bit-exact with allreduce_net.py:360-411): element e lies in segment
// s = seg(e) of `_segments(n, N)` (q, r = divmod(n, N); the first r segments hold
// q + 1 elements); the reference ring accumulates it as
//     ((x_s + x_{s+1}) + x_{s+2}) + ... + x_{s+N-1}      (ranks mod N)
// Both kernels evaluate exactly that left fold with __fadd_rn.  The *work* split is
// free: K3 partitions the bucket into N 16-B aligned parts (not the reference's
// segments), so both of its phases stream equal, aligned chunks; every 16-B slot
// still looks up its own fold start.  Slots straddling a segment boundary (at most
// N-1 of them) take a scalar path.
//
// Synchronisation: per-CTA flag barriers in every rank's IPC control area
// (st.release.sys / ld.acquire.sys), flags tagged (epoch << 32 | collective_tag) so any
// disagreement between ranks (length, kernel, grid, dtype, scale, group) is detected at
// the barrier; epochs come from a device call counter (graph-replay safe); bounded spins
// set a device error word and raise a sticky abort flag on every rank.
#pragma once

#include <cstring>

#include "common.cuh"

namespace mgw {

enum : int { kNoBarrier = 1, kSkipPhase1 = 2, kSkipPhase2 = 4, kSkipPack = 8, kPhaseMarks = 16 };

struct ArArgs {
  char* slot[kMaxRanks];       // slot-0 base of every rank (peer mapped; own at [rank])
  uint64_t* arrive[kMaxRanks]; // per-rank entry-barrier flags [2][kMaxBlocks][kMaxRanks]
  uint64_t* mid[kMaxRanks];    // per-rank mid-barrier flags   [2][kMaxBlocks][kMaxRanks]
  uint32_t* abort_flag[kMaxRanks];
  float* out[kMaxRanks];       // result buffer (a real rank uses out[rank])
  uint32_t* state;             // local [completed calls, finished CTAs]; null: no epochs
  int* err;                    // local device error word
  uint64_t* stamp;             // optional kernel span stamps [2]
  int64_t slot_stride;         // bytes from slot 0 to slot 1
  int64_t n;                   // elements
  uint64_t timeout_ns;
  int rank;
  int world;
  int flags;
  uint32_t tag;                // host: the caller's group tag; the launcher replaces it with
                               // collective_tag() -- every barrier flag and LL header carries it
};

// ---- collective tag.  The reference rejects a frame whose (iteration, group_low, segment,
// bytes) header disagrees (allreduce_net.py:340-345).  Here every barrier flag and LL
// header carries a 32-bit digest of everything the ranks must agree on: element count,
// dtype + kernel, grid (CTA b of every rank must handle the same chunk), scale, and the
// caller's group tag (head layer / iteration).  A rank whose digest differs from a peer's
// at any barrier raises MGW_DEV_MISMATCH on every rank within one flag round trip.
enum TagKind : uint32_t {
  kTagOneshot = 1, kTagTwoshot, kTagFusedOneshot, kTagFusedTwoshot, kTagLL, kTagNvls, kTagPush, kTagPushOneshot,
  kTagB16Oneshot, kTagB16Twoshot, kTagB16LL, kTagPushPipe, kTagB16Push, kTagLL128, kTagB16LL128, kTagLL128One, kTagB16LL128One
};

inline uint32_t tag_mix(uint32_t h, uint32_t k) {  // murmur3 block step
  k *= 0xcc9e2d51u;
  k = (k << 15) | (k >> 17);
  k *= 0x1b873593u;
  h ^= k;
  h = (h << 13) | (h >> 19);
  return h * 5u + 0xe6546b64u;
}

inline uint32_t collective_tag(uint32_t group_tag, int64_t n, uint32_t kind, int grid, float scale) {
  uint32_t sb;
  memcpy(&sb, &scale, sizeof(sb));
  uint32_t h = 0x6d677766u;
  h = tag_mix(h, group_tag);
  h = tag_mix(h, (uint32_t)n);
  h = tag_mix(h, (uint32_t)((uint64_t)n >> 32));
  h = tag_mix(h, kind);
  h = tag_mix(h, (uint32_t)grid);
  h = tag_mix(h, sb);
  h ^= 24u;  // murmur3 finalizer
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

// Phase marks (mgw_probe_phases): CTA 0 records %globaltimer at its phase boundaries into
// stamp[2 + k] (ncu cannot replay a multi-rank kernel, so the kernels time themselves).
__device__ __forceinline__ void phase_mark(const ArArgs& a, int k, int cta) {
  if (!(a.flags & kPhaseMarks) || a.stamp == nullptr) return;
  __syncthreads();
  if (cta == 0 && threadIdx.x == 0) a.stamp[2 + k] = global_ns();
}

// Kernel bodies take their CTA index `cta` and grid size `ctas` as arguments: the plain
// kernel passes (blockIdx.x, gridDim.x); the rank-group kernel (one cooperative launch
// holding every rank's CTAs on one device, tests and single-GPU emulation of the real
// barrier protocol) passes each rank's own index and count.
template <class Args>
struct RankGroup {
  Args args[kMaxRanks];
  int first[kMaxRanks + 1];  // CTA range of rank r: [first[r], first[r + 1])
  __device__ __forceinline__ int rank_of(int block) const {
    int r = 0;
    while (block >= first[r + 1]) ++r;
    return r;
  }
};

#define MGW_DEFINE_KERNELS(name, Args)                                                              \
  template <int N>                                                                                 \
  __global__ void __launch_bounds__(kThreads, 2) name##_kernel(const __grid_constant__ Args x) {   \
    name##_body<N>(x, blockIdx.x, gridDim.x);                                                      \
  }                                                                                                \
  template <int N>                                                                                 \
  __global__ void __launch_bounds__(kThreads, 2) name##_group(const __grid_constant__ RankGroup<Args> g) { \
    const int r = g.rank_of(blockIdx.x);                                                           \
    name##_body<N>(g.args[r], blockIdx.x - g.first[r], g.first[r + 1] - g.first[r]);               \
  }

// Loads in flight per thread ~ 8: unroll the slot loop by 8 / N.
template <int N>
struct Unroll {
  static constexpr int value = N <= 2 ? 4 : (N <= 4 ? 2 : 1);
};

// One barrier round for this CTA.  Thread t < world signals rank t and waits for
// rank t's matching CTA.
#ifndef MGW_BARRIER_RELAXED_POLL
#define MGW_BARRIER_RELAXED_POLL 0
#endif
static __device__ __noinline__ int cta_barrier(uint64_t* const* flags, int parity, uint32_t epoch, uint32_t tag,
                                               const ArArgs& a, int cta) {
  __shared__ int s_status;
  if (threadIdx.x == 0) s_status = 0;
  __syncthreads();  // also orders this CTA's earlier stores before the release below
  const int t = threadIdx.x;
  MGW_EXPECT(cta >= 0 && cta < kMaxBlocks && a.world <= kMaxRanks && a.rank < a.world);
  if (t < a.world) {
    const size_t base = ((size_t)parity * kMaxBlocks + cta) * kMaxRanks;
    store_release_sys(flags[t] + base + a.rank, ((uint64_t)epoch << 32) | tag);
    const uint64_t* mine = flags[a.rank] + base + t;
    const uint64_t start = global_ns();
    int status = MGW_DEV_OK;
    for (uint32_t spin = 0;; ++spin) {
#if MGW_BARRIER_RELAXED_POLL
      const uint64_t v = ld_relaxed_sys64(mine);
#else
      const uint64_t v = load_acquire_sys(mine);
#endif
      if ((uint32_t)(v >> 32) == epoch) {
        if ((uint32_t)v != tag) status = MGW_DEV_MISMATCH;
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
    if (status != MGW_DEV_OK) atomicCAS(&s_status, 0, status);
#if MGW_BARRIER_RELAXED_POLL
    fence_acq_rel_sys();  // one acquire fence after the relaxed polls
#endif
  }
  __syncthreads();
  const int status = s_status;
  if (status != MGW_DEV_OK && threadIdx.x == 0) {
    atomicCAS(a.err, 0, status);
    if (status != MGW_DEV_PEER_ABORT)
      for (int r = 0; r < a.world; ++r) store_release_sys32(a.abort_flag[r], 1u);
  }
  return status;
}

// Peer gate (opt-in, mgw_comm_set_gate): one warp announces "collective `epoch` is
// next on my comm stream" to every peer and waits until every peer has announced the
// same, so the bulk kernel that follows is launched only when all ranks have reached
// it.  Under a real backward pass ranks drift by tens of microseconds; without the
// gate the first rank's CTAs would sit in the entry barrier holding SM slots that the
// backward kernels need.  Door words are monotonic epochs -- no parity, no reset.
static __global__ void gate_kernel(const __grid_constant__ ArArgs a) {
  grid_dep_wait();  // a programmatic producer (the engine's fill) must finish before the
                    // exchange behind this gate reads its rows (the exchange's own wait
                    // only covers the gate)
  const int t = threadIdx.x;
  const uint32_t epoch = load_volatile32(a.state) + 1u;
  int status = MGW_DEV_OK;
  if (t < a.world) {
    uint64_t* door_t = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(a.arrive[t]) - kArriveOff + kDoorOff);
    const uint64_t* mine =
        reinterpret_cast<const uint64_t*>(reinterpret_cast<char*>(a.arrive[a.rank]) - kArriveOff + kDoorOff) + t;
    store_release_sys(door_t + a.rank, epoch);
    const uint64_t start = global_ns();
    for (uint32_t spin = 0;; ++spin) {
      if ((int32_t)((uint32_t)load_acquire_sys(mine) - epoch) >= 0) break;
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
  if (status != MGW_DEV_OK) {
    atomicCAS(a.err, 0, status);
    if (status != MGW_DEV_PEER_ABORT)
      for (int r = 0; r < a.world; ++r) store_release_sys32(a.abort_flag[r], 1u);
  }
}

inline int launch_gate(const ArArgs& a, cudaStream_t stream) {
  gate_kernel<<<1, 32, 0, stream>>>(a);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

// Last CTA out advances the call counter (epochs and slot parity come from it).
// Kernel completion publishes the counter to the next kernel on the stream.
__device__ __forceinline__ void finish_call(const ArArgs& a, int ctas) {
  stamp_exit(a.stamp);
  if (a.state == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t ticket = atomicAdd(&a.state[1], 1u);
    if (ticket == (uint32_t)ctas - 1) {
      a.state[1] = 0u;
      atomicAdd(&a.state[0], 1u);
    }
  }
}

template <int N>
__device__ __forceinline__ float fold1(const float* const* in, int s, int64_t e) {
  float x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int src = s + k >= N ? s + k - N : s + k;
    x[k] = __ldcg(in[src] + e);
  }
  float acc = x[0];
#pragma unroll
  for (int k = 1; k < N; ++k) acc = __fadd_rn(acc, x[k]);
  return acc;
}

// fold start of element e: advance a per-thread segment cursor (monotone in e)
__device__ __forceinline__ int advance_segment(int s, int64_t e, const int64_t* seg_end) {
  while (e >= seg_end[s]) ++s;
  return s;
}

// U slots of 16 B starting at vector v, stride `step` vectors: fold every slot that
// lies inside one segment; write results to dst0 (and dst1 when non-null).
template <int N, int U>
__device__ __forceinline__ void reduce_slots(const float* const* in, const int64_t* seg_end, int& seg, int64_t v,
                                             int64_t v_end, int64_t step, float* dst0, float* dst1) {
  float4 x[U][N];
  int su[U];
  bool ok[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t vv = v + u * step;
    ok[u] = false;
    su[u] = seg;
    if (vv < v_end) {
      const int64_t e = vv << 2;
      seg = advance_segment(seg, e, seg_end);
      su[u] = seg;
      ok[u] = e + 3 < seg_end[seg];
      if (ok[u]) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int src = seg + k >= N ? seg + k - N : seg + k;
          x[u][k] = __ldcg(reinterpret_cast<const float4*>(in[src] + e));
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t vv = v + u * step;
    if (vv >= v_end) continue;
    const int64_t e = vv << 2;
    if (ok[u]) {
      float4 acc = x[u][0];
#pragma unroll
      for (int k = 1; k < N; ++k) acc = fadd4(acc, x[u][k]);
      *reinterpret_cast<float4*>(dst0 + e) = acc;
      if (dst1) *reinterpret_cast<float4*>(dst1 + e) = acc;
    } else {
      int s = su[u];
      for (int j = 0; j < 4; ++j) {
        s = advance_segment(s, e + j, seg_end);
        const float y = fold1<N>(in, s, e + j);
        dst0[e + j] = y;
        if (dst1) dst1[e + j] = y;
      }
    }
  }
}

template <int N>
__device__ __forceinline__ void reduce_tail(const float* const* in, const int64_t* seg_end, int64_t e0, int64_t e1,
                                            float* dst0, float* dst1) {
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    int s = advance_segment(0, e, seg_end);
    const float y = fold1<N>(in, s, e);
    dst0[e] = y;
    if (dst1) dst1[e] = y;
  }
}

template <int N>
__device__ __forceinline__ void kernel_prologue(const ArArgs& a, uint32_t& epoch, int& parity, const float** s_in,
                                                int64_t* s_end) {
  grid_dep_wait();  // inputs written by a programmatic producer (the engine's gradient fill)
  stamp_enter(a.stamp);
  epoch = a.state != nullptr ? load_volatile32(a.state) + 1u : 0u;
  parity = (int)(epoch & 1u);
  MGW_EXPECT(a.slot_stride == 0 || a.n * 2 <= a.slot_stride);  // the bucket fits its slot (bf16 bound)
  if (threadIdx.x < N) {
    const int t = threadIdx.x;
    s_in[t] = reinterpret_cast<const float*>(a.slot[t] + (int64_t)parity * a.slot_stride);
    const int64_t q = a.n / N, r = a.n % N;
    s_end[t] = (int64_t)(t + 1) * q + (t + 1 < r ? t + 1 : r);  // end of reference segment t
  }
  __syncthreads();
}

// K2: every rank reads all N buckets and writes the whole reduced vector.
template <int N>
__global__ void __launch_bounds__(kThreads, 2) oneshot_kernel(const __grid_constant__ ArArgs a) {
  constexpr int U = Unroll<N>::value;
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  int status = MGW_DEV_OK;
  if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, blockIdx.x);
  if (status == MGW_DEV_OK && a.n > 0) {
    float* out = a.out[a.rank];
    const int64_t nv = a.n >> 2;
    const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
    const int64_t v0 = (int64_t)blockIdx.x * per;
    const int64_t v1 = v0 + per < nv ? v0 + per : nv;
    int seg = advance_segment(0, (v0 + threadIdx.x) << 2 < a.n ? (v0 + threadIdx.x) << 2 : 0, s_end);
    for (int64_t v = v0 + threadIdx.x; v < v1; v += (int64_t)U * kThreads)
      reduce_slots<N, U>(s_in, s_end, seg, v, v1, kThreads, out, nullptr);
    if (blockIdx.x == gridDim.x - 1) reduce_tail<N>(s_in, s_end, nv << 2, a.n, out, nullptr);
  }
  finish_call(a, gridDim.x);
}

// Work parts of the two-shot: rank p owns 16-B slots [part(p), part(p+1)); the n % 4 tail
// elements belong to rank N-1.  Part and per-CTA chunk boundaries fall on kPartAlign slots
// (512 B: one warp's 16-B accesses), so no warp store straddles a chunk edge -- unaligned
// chunks cost the push two-shot 7 % at 32 MiB (profiles/per_cta_n4_r02.json).  Parts only
// partition the work: the fold order follows the reference's segments (s_end), not parts.
constexpr int64_t kPartAlign = 32;
__host__ __device__ __forceinline__ int64_t part_begin(int p, int64_t nv, int world) {
  return p >= world ? nv : ((int64_t)p * nv / world) & ~(kPartAlign - 1);
}
// slots per CTA when `len` slots are split over `ctas` CTAs (a multiple of kPartAlign)
__host__ __device__ __forceinline__ int64_t chunk_per(int64_t len, int ctas) {
  const int64_t per = (len + ctas - 1) / ctas;
  return (per + kPartAlign - 1) / kPartAlign * kPartAlign;
}
// CTA b's chunk [lo, hi) of [q0, q1)
__host__ __device__ __forceinline__ void cta_chunk(int64_t q0, int64_t q1, int b, int ctas, int64_t& lo, int64_t& hi) {
  const int64_t per = chunk_per(q1 - q0, ctas);
  lo = q0 + (int64_t)b * per;
  if (lo > q1) lo = q1;
  hi = lo + per < q1 ? lo + per : q1;
}

// K3: phase 1 reduces this rank's part (fold order per slot) into its own slot (in
// place) and into out; phase 2 copies every peer's reduced part into out.
template <int N>
__global__ void __launch_bounds__(kThreads, 2) twoshot_kernel(const __grid_constant__ ArArgs a) {
  constexpr int U = Unroll<N>::value;
  constexpr int UC = N <= 2 ? 8 : (N <= 3 ? 4 : (N <= 5 ? 2 : 1));  // copy slots per peer per step
  __shared__ const float* s_in[kMaxRanks];
  __shared__ int64_t s_end[kMaxRanks];
  uint32_t epoch;
  int parity;
  kernel_prologue<N>(a, epoch, parity, s_in, s_end);
  const int me = a.rank;
  const int b = blockIdx.x, G = gridDim.x;
  const int64_t nv = a.n >> 2;
  float* out = a.out[me];
  float* own = const_cast<float*>(s_in[me]);
  float* second = out != own ? out : nullptr;
  int status = MGW_DEV_OK;

  if (!(a.flags & kSkipPhase1)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.arrive, parity, epoch, a.tag, a, blockIdx.x);
    if (status == MGW_DEV_OK && a.n > 0) {
      int64_t v0, v1;
      cta_chunk(part_begin(me, nv, N), part_begin(me + 1, nv, N), b, G, v0, v1);
      int seg = advance_segment(0, ((v0 + threadIdx.x) << 2) < a.n ? (v0 + threadIdx.x) << 2 : 0, s_end);
      for (int64_t v = v0 + threadIdx.x; v < v1; v += (int64_t)U * kThreads)
        reduce_slots<N, U>(s_in, s_end, seg, v, v1, kThreads, own, second);
      if (me == N - 1 && b == G - 1) reduce_tail<N>(s_in, s_end, nv << 2, a.n, own, second);
    }
  }

  if (status == MGW_DEV_OK && !(a.flags & kSkipPhase2)) {
    if (!(a.flags & kNoBarrier)) status = cta_barrier(a.mid, parity, epoch, a.tag, a, blockIdx.x);
    if (status == MGW_DEV_OK && a.n > 0) {
      // chunk b of every peer part; peers interleaved so N-1 streams are in flight.
      // Chunk bounds live in shared memory to keep the copy loop's registers for data.
      __shared__ int64_t s_lo[kMaxRanks], s_len[kMaxRanks];
      if (threadIdx.x > 0 && threadIdx.x < N) {
        const int k = threadIdx.x;
        const int p = me + k >= N ? me + k - N : me + k;
        int64_t c0, c1;
        cta_chunk(part_begin(p, nv, N), part_begin(p + 1, nv, N), b, G, c0, c1);
        s_lo[k] = c0;
        s_len[k] = c1 > c0 ? c1 - c0 : 0;
      }
      __syncthreads();
      int64_t longest = 0;
      for (int k = 1; k < N; ++k) longest = s_len[k] > longest ? s_len[k] : longest;
      float4* out4 = reinterpret_cast<float4*>(out);
      for (int64_t i = threadIdx.x; i < longest; i += (int64_t)UC * kThreads) {
        float4 x[UC][N];
#pragma unroll
        for (int u = 0; u < UC; ++u)
#pragma unroll
          for (int k = 1; k < N; ++k) {
            const int64_t ii = i + (int64_t)u * kThreads;
            const int p = me + k >= N ? me + k - N : me + k;
            if (ii < s_len[k]) x[u][k] = __ldcg(reinterpret_cast<const float4*>(s_in[p]) + s_lo[k] + ii);
          }
#pragma unroll
        for (int u = 0; u < UC; ++u)
#pragma unroll
          for (int k = 1; k < N; ++k) {
            const int64_t ii = i + (int64_t)u * kThreads;
            if (ii < s_len[k]) out4[s_lo[k] + ii] = x[u][k];
          }
      }
      if (me != N - 1 && b == G - 1)
        for (int64_t e = (nv << 2) + threadIdx.x; e < a.n; e += blockDim.x) out[e] = __ldcg(s_in[N - 1] + e);
    }
  }
  finish_call(a, gridDim.x);
}

inline int grid_for(int64_t vectors, int64_t per_cta, int max_ctas) {
  int64_t g = (vectors + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  if (g > max_ctas) g = max_ctas;
  return (int)g;
}

// CTAs for a collective over `vectors` 16-B slots (whole bucket for one-shot, one part
// for two-shot), or `per_cta` slots per CTA when tuned.  Default: spread a mid-size
// bucket over up to one CTA per SM (slots per CTA a multiple of 128, at most one batch of
// U slots per thread) -- engine-mode sweeps (profiles/grid_n{2,4}_r01.json) show one CTA
// per SM beats both fewer, fatter CTAs (load issue per SM) and two per SM (per-CTA flag
// traffic, shared SM issue) for 0.25-8 MB; beyond 148 full batches the grid grows to the
// CTA cap.
#ifndef MGW_LOCAL_SPREAD
#define MGW_LOCAL_SPREAD 1  // CTAs per SM the single-rank (HBM-bound) group kernel spreads over
#endif
inline int unroll_of(int world) { return world <= 2 ? 4 : (world <= 4 ? 2 : 1); }  // == Unroll<N>::value

inline int collective_grid_rt(int world, int64_t vectors, int64_t per_cta, int max_ctas) {
  if (per_cta <= 0) {
    const int64_t full = (int64_t)kThreads * unroll_of(world);
    const int64_t spread = (int64_t)kSMs * (world == 1 ? MGW_LOCAL_SPREAD : 1);
    per_cta = (vectors + spread - 1) / spread;
    per_cta = (per_cta + 127) / 128 * 128;
    per_cta = per_cta < 128 ? 128 : (per_cta > full ? full : per_cta);
  }
  return grid_for(vectors, per_cta, max_ctas);
}

template <int N>
inline int collective_grid(int64_t vectors, int64_t per_cta, int max_ctas) {
  static_assert(Unroll<N>::value == (N <= 2 ? 4 : (N <= 4 ? 2 : 1)), "unroll_of mirrors Unroll<N>");
  if (per_cta <= 0) {
    const int64_t full = (int64_t)kThreads * Unroll<N>::value;
    const int64_t spread = (int64_t)kSMs * (N == 1 ? MGW_LOCAL_SPREAD : 1);
    per_cta = (vectors + spread - 1) / spread;
    per_cta = (per_cta + 127) / 128 * 128;
    per_cta = per_cta < 128 ? 128 : (per_cta > full ? full : per_cta);
  }
  return grid_for(vectors, per_cta, max_ctas);
}

}  // namespace mgw
