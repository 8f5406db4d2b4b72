// ll128.cuh -- flag-in-line two-shot and one-shot ("LL128"): the push kernels' data movement
// with no barrier at all.  Same result as ring_allreduce (allreduce_net.py:370-411) on the group
// bucket (:499-509), bit for bit; fp32 (4 per 16-B slot, scaled at pack) and bf16 (8 per
// slot, fp32 accumulation, scaled and rounded once by the part's owner, as bf16.cuh).
//
// The push two-shot (push.cuh) pays two CTA barriers per call; each is a system-scope
// release (the CTA stalls until every NVLink store it issued is acknowledged) plus a flag
// round trip, and a phase cannot start on any data until the slowest peer CTA signalled.
// Here data and flag travel together: a 128-B line = 8 lanes x 16 B, lanes 0..6 carry 7
// 16-B slots of the bucket, lane 7 carries 8 B of payload (half of a slot shared by a pair
// of lines) and the flag (epoch << 32 | collective tag): 120 B of payload per line.
// One warp store instruction writes whole lines (a group of 8 consecutive lanes per line),
// and NVLink delivers a warp's 128-B line as one write, so a reader that sees the flag of a
// line (loaded by the same warp instruction as the other 7 lanes) sees its payload -- the
// NVLink LL128 contract of NCCL's protocol of that name.  Readers only poll local memory.
//
//   phase 1  CTA b stores its line range of every part p (scaled) into rank p's incoming
//            row `me`                                  (lines: 2 (N-1)/N x M x 16/15 out)
//   phase 2  CTA b polls its line range of its own part in the N local rows, folds in the
//            reference order (fold start = the element's `_segments` segment), writes its
//            tensors and stores result lines into every peer's gather row `me`
//   phase 3  CTA b polls its line range of every peer part in its gather rows and writes
//            its tensors.
// A CTA runs the three phases per round of 64-128 lines per part (l128_round_lines), so its
// local copies overlap the NVLink traffic of the next round.  The one-shot (ONE) pushes its
// line range of the whole bucket to every rank and folds the whole bucket locally: phases
// 1-2 only, (N-1) x M x 16/15 out, one hop.
//
// Every CTA depends only on the same CTA index of its peers (same part / line split), so
// the grid need not be co-resident across ranks.  Areas: incoming lines = slot[parity] of
// the IPC region ([N src][row_lines]), gather lines = gather[parity] ([N part][row_lines]):
// the slots every other kernel uses, with the same reuse distance 2 by parity (a pull
// kernel of call k may still be reading a peer's slot[parity k] when this rank starts
// call k + 1).  The flag's epoch tells calls apart; lines must fit one slot.
// Disagreement: CTA 0 pushes the LL header (barrier word of CTA 0) and polls check the
// source's header, so a peer in another collective fails fast as for LL.
#pragma once

#include "bf16.cuh"
#include "ll.cuh"

namespace mgw {

constexpr int kL128Lanes = 8;                          // 16-B lanes per 128-B line
constexpr int kL128Vec = kL128Lanes - 1;               // whole 16-B slots per line (lanes 0..6)
constexpr int kL128PairSlots = 2 * kL128Vec + 1;       // 16-B slots per line pair (15)
constexpr int kL128Step = kThreads / kL128Lanes;       // lines per CTA step (64 = 32 pairs)
constexpr int kL128Words = 2 * kL128Lanes;             // u64 words per line
#ifndef MGW_L128_ROUND_LINES
#define MGW_L128_ROUND_LINES 0  // A/B: a fixed round (multiple of 64 lines); 0 = by the CTA's span
#endif
static_assert(MGW_L128_ROUND_LINES % kL128Step == 0, "rounds are whole CTA steps");
// Lines per part per round for a CTA whose longest part range is `span` lines: about four
// rounds, 64 or 128 lines (same-box A/B at N = 4, profiles/ll128_rounds_r02.json:
// 16 MiB 2 x 64 -> 505 GB/s vs 478 in one round, 32 MiB 4 x 64 -> 542, 64 MiB 4 x 128 -> 578,
// 128 MiB 8 x 128 -> 585).  Every rank derives the same span, so the same rounds: a CTA's
// round r only ever waits on round r of the same CTA index elsewhere.
__device__ __forceinline__ int64_t l128_round_lines(int64_t span, bool one) {
  if (MGW_L128_ROUND_LINES > 0) return MGW_L128_ROUND_LINES;
  if (one) return 2 * kL128Step;  // the one-shot: 128 (N = 2, 4 / 8 MiB: 334 / 431 vs 313 / 410 GB/s at 64)
  return span / 4 > kL128Step ? 2 * kL128Step : kL128Step;
}

// Lines come in pairs: lanes 0..6 of the even line carry slots 0..6 of the pair, lanes
// 0..6 of the odd line slots 7..13, and lane 7 of each line carries one 8-B half of slot
// 14 next to its flag word -- 240 B of payload per 256 B (16/15 on the wire instead of
// 8/7), every tensor access still a 16-B aligned slot.  Slot of (line l, lane sub)
// relative to its part:
__host__ __device__ __forceinline__ int64_t l128_slot(int64_t l, int sub) {
  const int64_t base = (l >> 1) * kL128PairSlots;
  return sub < kL128Vec ? base + (l & 1) * kL128Vec + sub : base + 2 * kL128Vec;
}
// lines holding `slots` 16-B slots (whole pairs)
__host__ __device__ __forceinline__ int64_t l128_lines(int64_t slots) {
  return 2 * ((slots + kL128PairSlots - 1) / kL128PairSlots);
}
// CTA b's line range [l0, l1) of a part of `slots` slots: whole pairs, so a warp's groups
// 2k and 2k+1 always hold the two lines of one pair
__device__ __forceinline__ void l128_cta_lines(int64_t slots, int b, int ctas, int64_t& l0, int64_t& l1) {
  cta_chunk(0, l128_lines(slots) / 2, b, ctas, l0, l1);
  l0 *= 2;
  l1 *= 2;
}

struct L128Args {
  FusedArgs f;
  char* in[kMaxRanks];       // rank r's slot 0: incoming lines [N src][row_lines] (parity 1 at slot_stride)
  char* gat[kMaxRanks];      // rank r's gather area 0: result lines [N part][row_lines]
  uint64_t* hdr[kMaxRanks];  // header words (CTA 0's arrive flags), as LLArgs::hdr
  int64_t hdr_stride;        // words from parity 0 to parity 1 of hdr
  int64_t row_lines;         // lines per row (the longest part)
};

// 16-B slots of a bucket of n elements (4 fp32 / 8 bf16; the last one partial)
__host__ __device__ __forceinline__ int64_t l128_slots(int64_t n, bool b16) { return b16 ? (n + 7) / 8 : (n + 3) / 4; }
// lines per row: the longest part (part_begin rounds down to kPartAlign) in lines; the
// one-shot's row holds the whole bucket
__host__ __device__ __forceinline__ int64_t l128_row_lines(int64_t n, int world, bool b16, bool one = false) {
  if (one) return l128_lines(l128_slots(n, b16));
  return l128_lines((l128_slots(n, b16) + world - 1) / world + kPartAlign);
}

__device__ __forceinline__ void st_volatile_v2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void ld_volatile_v2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// Warp-collective: poll until every active group's line (this lane's 16 B at `p`) carries
// `expect` in its flag lane.  Returns a warp-uniform status.  Slow path every 16 spins: a
// flag of this epoch with another tag, or the source's header of this epoch with another
// tag (a peer in a different collective), the abort flag, the timeout.
#ifndef MGW_L128_BACKOFF_NS
#define MGW_L128_BACKOFF_NS 0  // A/B: sleep between re-polls of a line that has not arrived
#endif
__device__ __forceinline__ int l128_poll(const uint64_t* p, bool active, uint64_t expect, const uint64_t* hdr,
                                         const ArArgs& a, uint64_t& w0, uint64_t& w1) {
  const int flag_lane = (threadIdx.x & 31) | (kL128Lanes - 1);
  const uint32_t epoch = (uint32_t)(expect >> 32);
  uint64_t start = 0;
  for (uint32_t spin = 0;; ++spin) {
    if (MGW_L128_BACKOFF_NS > 0 && spin > 0) __nanosleep(MGW_L128_BACKOFF_NS);
    if (active) ld_volatile_v2(p, w0, w1);
    const uint64_t flag = __shfl_sync(0xffffffffu, w1, flag_lane);
    if (__all_sync(0xffffffffu, !active || flag == expect)) return MGW_DEV_OK;
    if ((spin & 15) == 15) {
      int st = MGW_DEV_OK;
      if (active && flag != expect && (uint32_t)(flag >> 32) == epoch) st = MGW_DEV_MISMATCH;
      if (active && st == MGW_DEV_OK) {
        const uint64_t h = ld_relaxed_sys_u64(hdr);
        if ((uint32_t)(h >> 32) == epoch && (uint32_t)h != a.tag) st = MGW_DEV_MISMATCH;
      }
      if (st == MGW_DEV_OK && load_relaxed_sys32(a.abort_flag[a.rank]) != 0u) st = MGW_DEV_PEER_ABORT;
      if (spin == 15) start = global_ns();
      if (st == MGW_DEV_OK && global_ns() - start > a.timeout_ns) st = MGW_DEV_TIMEOUT;
      const int any = __reduce_max_sync(0xffffffffu, st);  // warp-uniform: any error ends the call
      if (any != MGW_DEV_OK) return any;
    }
  }
}

// Element j of a 16-B slot held as two u64 words: fp32 (4 per slot) or bf16 (8 per slot,
// exactly upcast).
template <bool B16>
__device__ __forceinline__ float l128_get(uint64_t lo, uint64_t hi, int j) {
  if (B16) {
    const uint64_t w = j < 4 ? lo : hi;
    return __uint_as_float((uint32_t)((w >> (16 * (j & 3))) & 0xFFFFu) << 16);
  }
  const uint64_t w = j < 2 ? lo : hi;
  return __uint_as_float((uint32_t)(j & 1 ? w >> 32 : w));
}

// the reference fold of element j from the N sources' words, starting at source `seg`
// (static register indexing: the rotation is unrolled per start)
template <int N, bool B16>
__device__ __forceinline__ float l128_fold_elem(const uint64_t (&lo)[N], const uint64_t (&hi)[N], int seg, int j) {
  float out = 0.f;
#pragma unroll
  for (int s = 0; s < N; ++s) {
    if (s == seg) {
      float acc = l128_get<B16>(lo[s], hi[s], j);
#pragma unroll
      for (int kk = 1; kk < N; ++kk) {
        const int src = (s + kk) % N;
        acc = __fadd_rn(acc, l128_get<B16>(lo[src], hi[src], j));
      }
      out = acc;
    }
  }
  return out;
}

// The reduced slot at bucket element e: every element folded from its segment's start
// (one rotation for the whole slot when it lies in one segment); bf16: scaled and
// rounded once here (fp32 was scaled at pack, as the reference packs).  Padding
// elements past n come out 0.
template <int N, bool B16>
__device__ __forceinline__ void l128_fold_slot(const uint64_t (&lo)[N], const uint64_t (&hi)[N], int seg, int64_t e,
                                               int64_t n, const int64_t* s_end, float scale, bool scaled,
                                               uint64_t& olo, uint64_t& ohi) {
  constexpr int K = B16 ? 8 : 4;
  float r[K];
  if (e + K - 1 < s_end[seg]) {
#pragma unroll
    for (int j = 0; j < K; ++j) r[j] = 0.f;
#pragma unroll
    for (int s = 0; s < N; ++s) {
      if (s == seg) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          float acc = l128_get<B16>(lo[s], hi[s], j);
#pragma unroll
          for (int kk = 1; kk < N; ++kk) {
            const int src = (s + kk) % N;
            acc = __fadd_rn(acc, l128_get<B16>(lo[src], hi[src], j));
          }
          r[j] = acc;
        }
      }
    }
  } else {  // the slot straddles a segment boundary, or is the partial last slot
    int s2 = seg;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      r[j] = 0.f;
      if (e + j < n) {
        s2 = advance_segment(s2, e + j, s_end);
        r[j] = l128_fold_elem<N, B16>(lo, hi, s2, j);
      }
    }
  }
  if (B16) {
    uint64_t w[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < K; ++j)
      w[j >> 2] |= (uint64_t)f32_to_b16(scaled ? __fmul_rn(r[j], scale) : r[j]) << (16 * (j & 3));
    olo = w[0];
    ohi = w[1];
  } else {
    olo = (uint64_t)__float_as_uint(r[0]) | ((uint64_t)__float_as_uint(r[1]) << 32);
    ohi = (uint64_t)__float_as_uint(r[2]) | ((uint64_t)__float_as_uint(r[3]) << 32);
  }
}

// bucket slot v from the layer tensors (fp32: scaled; bf16: raw); zeros past n
template <bool B16>
__device__ __forceinline__ void l128_load(const FusedArgs& f, int& k, int64_t v, float scale, bool scaled,
                                          uint64_t& lo, uint64_t& hi) {
  if (B16) {
    const int64_t e = v * kB16;
    bool fast;
    const uint16_t* tp = b16_tensor(f, k, e, fast);
    if (fast) {
      const uint4 x = *reinterpret_cast<const uint4*>(tp);
      lo = (uint64_t)x.x | ((uint64_t)x.y << 32);
      hi = (uint64_t)x.z | ((uint64_t)x.w << 32);
      return;
    }
    uint64_t w[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < kB16; ++j)
      if (e + j < f.ar.n) w[j >> 2] |= (uint64_t)*b16_tensor1(f, k, e + j) << (16 * (j & 3));
    lo = w[0];
    hi = w[1];
    return;
  }
  const int64_t e = v << 2;
  bool fast;
  const float* tp = fused_tensor(f, k, e, fast);
  float r[4];
  if (fast) {
    const float4 x = *reinterpret_cast<const float4*>(tp);
    r[0] = x.x, r[1] = x.y, r[2] = x.z, r[3] = x.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = e + j < f.ar.n ? *fused_tensor1(f, k, e + j) : 0.f;
  }
  if (scaled)
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = __fmul_rn(r[j], scale);
  lo = (uint64_t)__float_as_uint(r[0]) | ((uint64_t)__float_as_uint(r[1]) << 32);
  hi = (uint64_t)__float_as_uint(r[2]) | ((uint64_t)__float_as_uint(r[3]) << 32);
}

// bucket slot v into the layer tensors (elements past n dropped)
template <bool B16>
__device__ __forceinline__ void l128_store(const FusedArgs& f, int& k, int64_t v, uint64_t lo, uint64_t hi) {
  if (B16) {
    const int64_t e = v * kB16;
    bool fast;
    uint16_t* tp = b16_tensor(f, k, e, fast);
    if (fast) {
      *reinterpret_cast<uint4*>(tp) = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
      return;
    }
#pragma unroll
    for (int j = 0; j < kB16; ++j)
      if (e + j < f.ar.n) *b16_tensor1(f, k, e + j) = (uint16_t)((j < 4 ? lo : hi) >> (16 * (j & 3)));
    return;
  }
  const int64_t e = v << 2;
  bool fast;
  float* tp = fused_tensor(f, k, e, fast);
  if (fast) {
    *reinterpret_cast<float4*>(tp) = make_float4(l128_get<false>(lo, hi, 0), l128_get<false>(lo, hi, 1),
                                                 l128_get<false>(lo, hi, 2), l128_get<false>(lo, hi, 3));
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (e + j < f.ar.n) *fused_tensor1(f, k, e + j) = l128_get<false>(lo, hi, j);
}

// ONE = the one-shot: every rank pushes its whole bucket (one line range per CTA) into
// every rank's incoming row `me` and folds its line range of the whole bucket from the N
// local rows -- one NVLink hop, (N-1) x M x 16/15 out, no gather phase.
template <int N, bool B16, bool ONE>
__device__ __forceinline__ void ll128_any_body(const L128Args& x, const int cta, const int ctas) {
  constexpr int K = B16 ? kB16 : 4;  // elements per 16-B slot
  const FusedArgs& f = x.f;
  const ArArgs& a = f.ar;
  grid_dep_wait();
  stamp_enter(a.stamp);
  __shared__ int64_t s_end[kMaxRanks];
  const uint32_t epoch = load_volatile32(a.state) + 1u;
  const int parity = (int)(epoch & 1u);
  const int me = a.rank;
  const int64_t n = a.n;
  const int64_t slots = l128_slots(n, B16);
  if (threadIdx.x < N) {
    const int t = threadIdx.x;
    const int64_t q = n / N, r = n % N;
    s_end[t] = (int64_t)(t + 1) * q + (t + 1 < r ? t + 1 : r);  // end of reference segment t
  }
  // kSkipPack / kSkipPhase1 / kSkipPhase2 run one phase per launch (emulated ranks on one
  // device, tests only: every launch polls lines that earlier launches wrote)
  const bool do_push = !(a.flags & kSkipPack), do_fold = !(a.flags & kSkipPhase1),
             do_unpack = !(a.flags & kSkipPhase2);
  if (do_push && cta == 0 && threadIdx.x < N)
    st_relaxed_sys_u64(x.hdr[threadIdx.x] + parity * x.hdr_stride + me, ((uint64_t)epoch << 32) | a.tag);
  __syncthreads();
  const uint64_t expect = ((uint64_t)epoch << 32) | a.tag;
  const int sub = threadIdx.x & (kL128Lanes - 1);  // lane within the line
  const int grp = threadIdx.x / kL128Lanes;        // line within the CTA step (pairs: 2k, 2k+1)
  const bool shared_lane = sub == kL128Vec;        // lane 7: half of the pair's slot 14 + flag
  const bool odd = grp & 1;                        // the pair's second line (high half of slot 14)
  // the words lane `sub` puts on the wire for slot words (lo, hi)
  auto wire_lo = [&](uint64_t lo, uint64_t hi) { return shared_lane ? (odd ? hi : lo) : lo; };
  auto wire_hi = [&](uint64_t hi) { return shared_lane ? expect : hi; };
  const int64_t rl = x.row_lines;
  const float scale = f.scale;
  const bool scaled = scale != 1.0f;
  const uint64_t* hdr_mine = x.hdr[me] + parity * x.hdr_stride;
  MGW_EXPECT(a.slot_stride == 0 || (int64_t)N * rl * 128 <= a.slot_stride);
  const int64_t poff = (int64_t)parity * a.slot_stride;
  auto in_of = [&](int r) { return reinterpret_cast<uint64_t*>(x.in[r] + poff); };
  auto gat_of = [&](int r) { return reinterpret_cast<uint64_t*>(x.gat[r] + poff); };
  int status = MGW_DEV_OK;

  // line range [l0, l1) of this CTA in part p (one-shot: the whole bucket), computed once
  // per CTA into shared memory (the 64-bit divisions cost ~1 us per thread if repeated)
  __shared__ int64_t s_rng[kMaxRanks][4];
  __shared__ int64_t s_span;
  if (threadIdx.x < (ONE ? 1 : N)) {
    const int p = threadIdx.x;
    const int64_t q0 = ONE ? 0 : part_begin(p, slots, N), q1 = ONE ? slots : part_begin(p + 1, slots, N);
    int64_t l0, l1;
    l128_cta_lines(q1 - q0, cta, ctas, l0, l1);
    s_rng[p][0] = q0;
    s_rng[p][1] = q1;
    s_rng[p][2] = l0;
    s_rng[p][3] = l1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t span = 0;
    for (int p = 0; p < (ONE ? 1 : N); ++p) span = s_rng[p][3] - s_rng[p][2] > span ? s_rng[p][3] - s_rng[p][2] : span;
    s_span = span;
  }
  __syncthreads();
  auto range_of = [&](int p, int64_t& q0, int64_t& q1, int64_t& l0, int64_t& l1) {
    const int r = ONE ? 0 : p;
    q0 = s_rng[r][0];
    q1 = s_rng[r][1];
    l0 = s_rng[r][2];
    l1 = s_rng[r][3];
  };
  // The CTA walks its line ranges in rounds (l128_round_lines) of lines per part, all three phases
  // per round: a CTA's local phase 3 of round r then overlaps the NVLink pushes of round
  // r + 1 (its own and other CTAs'), instead of every CTA pushing, then folding, then
  // copying in lock-step (profiles/ll128_rounds_r02.json).  Round r of a phase only waits
  // on round r of the same CTA index on the peers, so there is no cycle.
  const int64_t span = s_span;
  const int64_t round = l128_round_lines(span, ONE);
  int seg = 0, k2 = 0;
  bool k2_set = false;
  phase_mark(a, 0, cta);
  for (int64_t off = 0; off < span && status == MGW_DEV_OK; off += round) {
    // ---- phase 1: this round's lines of every part p into rank p's incoming row `me`
    //      (one-shot: this round's lines of the whole bucket into every rank's row `me`)
    if (do_push) {
#pragma unroll 1
      for (int p = 0; p < (ONE ? 1 : N); ++p) {
        int64_t q0, q1, l0, l1;
        range_of(p, q0, q1, l0, l1);
        const int64_t r0 = l0 + off, r1 = l0 + off + round < l1 ? l0 + off + round : l1;
        int k = 0;
        bool k_set = false;
        for (int64_t base = r0; base < r1; base += kL128Step) {
          const int64_t l = base + grp;
          const int64_t v = q0 + l128_slot(l, sub);
          const bool live = l < r1 && v < q1;
          uint64_t lo = 0, hi = 0;
          if (live) {
            if (!k_set) {
              k = fused_row_covering(f, v * K);
              k_set = true;
            }
            l128_load<B16>(f, k, v, scale, scaled, lo, hi);
          }
          const uint64_t w0 = wire_lo(lo, hi), w1 = wire_hi(hi);
          __syncwarp();
          if (l < r1) {
            if (ONE) {
#pragma unroll
              for (int r = 0; r < N; ++r) {
                const int q = me + 1 + r < N ? me + 1 + r : me + 1 + r - N;  // peers first, mine last
                st_volatile_v2(in_of(q) + ((int64_t)me * rl + l) * kL128Words + sub * 2, w0, w1);
              }
            } else {
              st_volatile_v2(in_of(p) + ((int64_t)me * rl + l) * kL128Words + sub * 2, w0, w1);
            }
          }
        }
      }
    }
    // ---- phase 2: fold this round's lines of my part from the N local rows; write my
    //      tensors and every peer's gather row `me`
    if (do_fold) {
      int64_t q0, q1, l0, l1;
      range_of(ONE ? 0 : me, q0, q1, l0, l1);
      const int64_t r0 = l0 + off, r1 = l0 + off + round < l1 ? l0 + off + round : l1;
      const uint64_t* in = in_of(me) + sub * 2;
      for (int64_t base = r0; base < r1 && status == MGW_DEV_OK; base += kL128Step) {
        const int64_t l = base + grp;
        const bool active = l < r1;
        const int64_t v = q0 + l128_slot(l, sub);
        uint64_t lo[N], hi[N];
#pragma unroll
        for (int s = 0; s < N; ++s) {
          lo[s] = hi[s] = 0;
          if (active) ld_volatile_v2(in + ((int64_t)s * rl + l) * kL128Words, lo[s], hi[s]);
        }
#pragma unroll
        for (int s = 0; s < N; ++s) {
          const uint64_t flag = __shfl_sync(0xffffffffu, hi[s], (threadIdx.x & 31) | (kL128Lanes - 1));
          if (!__all_sync(0xffffffffu, !active || flag == expect)) {
            const int st =
                l128_poll(in + ((int64_t)s * rl + l) * kL128Words, active, expect, hdr_mine + s, a, lo[s], hi[s]);
            if (st != MGW_DEV_OK) status = st;
          }
        }
        if (status != MGW_DEV_OK) break;
        // lane 7: rebuild slot 14 from its own half and the partner line's (lane ^ 8)
#pragma unroll
        for (int s = 0; s < N; ++s) {
          const uint64_t other = __shfl_xor_sync(0xffffffffu, lo[s], kL128Lanes);
          if (shared_lane) {
            hi[s] = odd ? lo[s] : other;
            lo[s] = odd ? other : lo[s];
          }
        }
        const bool live = active && v < q1;
        uint64_t ylo = 0, yhi = 0;
        if (live) {
          const int64_t e = v * K;
          seg = advance_segment(seg, e, s_end);
          l128_fold_slot<N, B16>(lo, hi, seg, e, n, s_end, scale, scaled, ylo, yhi);
          if (!k2_set) {
            k2 = fused_row_covering(f, e);
            k2_set = true;
          }
          if (!(shared_lane && odd)) l128_store<B16>(f, k2, v, ylo, yhi);  // slot 14: the even line's lane
        }
        if (ONE) continue;  // the one-shot has every part: no result lines
        const uint64_t w0 = wire_lo(ylo, yhi), w1 = wire_hi(yhi);
        __syncwarp();
#pragma unroll
        for (int q = 0; q < N; ++q)
          if (q != me && active) st_volatile_v2(gat_of(q) + ((int64_t)me * rl + l) * kL128Words + sub * 2, w0, w1);
      }
    }
    // ---- phase 3: this round's lines of every peer part from my gather rows into my tensors
    if (do_unpack && !ONE) {
#pragma unroll 1
      for (int p = 0; p < N && status == MGW_DEV_OK; ++p) {
        if (p == me) continue;
        int64_t q0, q1, l0, l1;
        range_of(p, q0, q1, l0, l1);
        const int64_t r0 = l0 + off, r1 = l0 + off + round < l1 ? l0 + off + round : l1;
        const uint64_t* g = gat_of(me) + (int64_t)p * rl * kL128Words + sub * 2;
        int k = 0;
        bool k_set = false;
        for (int64_t base = r0; base < r1; base += kL128Step) {
          const int64_t l = base + grp;
          const bool active = l < r1;
          uint64_t w0 = 0, w1 = 0;
          const int st = l128_poll(g + l * kL128Words, active, expect, hdr_mine + p, a, w0, w1);
          if (st != MGW_DEV_OK) {
            status = st;
            break;
          }
          const int64_t v = q0 + l128_slot(l, sub);
          const uint64_t other = __shfl_xor_sync(0xffffffffu, w0, kL128Lanes);  // slot 14's other half
          if (shared_lane) w1 = other;  // the even line's lane 7 writes slot 14: (own half, odd half)
          if (active && v < q1 && !(shared_lane && odd)) {
            if (!k_set) {
              k = fused_row_covering(f, v * K);
              k_set = true;
            }
            l128_store<B16>(f, k, v, w0, w1);
          }
        }
      }
    }
  }
  if (status != MGW_DEV_OK && (threadIdx.x & 31) == 0) ll_report(a, status);
  phase_mark(a, 1, cta);
  finish_call(a, ctas);
}

template <int N>
__device__ __forceinline__ void ll128_body(const L128Args& x, const int cta, const int ctas) {
  ll128_any_body<N, false, false>(x, cta, ctas);
}
template <int N>
__device__ __forceinline__ void b16_ll128_body(const L128Args& x, const int cta, const int ctas) {
  ll128_any_body<N, true, false>(x, cta, ctas);
}
template <int N>
__device__ __forceinline__ void ll128_one_body(const L128Args& x, const int cta, const int ctas) {
  ll128_any_body<N, false, true>(x, cta, ctas);
}
template <int N>
__device__ __forceinline__ void b16_ll128_one_body(const L128Args& x, const int cta, const int ctas) {
  ll128_any_body<N, true, true>(x, cta, ctas);
}

MGW_DEFINE_KERNELS(ll128, L128Args)
MGW_DEFINE_KERNELS(b16_ll128, L128Args)
MGW_DEFINE_KERNELS(ll128_one, L128Args)
MGW_DEFINE_KERNELS(b16_ll128_one, L128Args)

}  // namespace mgw
