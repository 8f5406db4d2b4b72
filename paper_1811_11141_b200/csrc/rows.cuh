// rows.cuh -- K1 pack(+scale), K4 unpack, and the fill / check helpers.
//
// A merge group's bucket is the concatenation of its layer gradients, layer `high`
// first (allreduce_net.py:499-509).  Two kernels move it:
//
// * rows_kernel (every op, any alignment): the bucket is cut into one balanced tile per
//   CTA (at most one resident wave, no tail wave); every thread owns fixed 16-B slots of
//   its tile and keeps the layer row holding its current slot in registers (rows are
//   sorted by bucket offset, so the cursor is monotone per thread and a descriptor is
//   read only when a slot crosses into the next row).  A slot inside one row at a 16-B
//   aligned tensor address moves as one 128-bit access; slots that straddle two rows or
//   sit at a misaligned tensor address fall back to four scalar accesses.
// * bulk_rows_kernel (pack with scale 1, unpack; buckets >= kBulkMinBytes): TMA bulk
//   copies.  Per CTA tile, one elected thread streams every row segment whose tensor and
//   bucket addresses share 16-B alignment through a 4-stage shared-memory ring
//   (cp.async.bulk global->shared on an mbarrier, then shared->global as a bulk group),
//   keeping 64 KB per CTA in flight without holding them in registers; the other warps
//   copy the ragged row edges and misaligned rows with scalar accesses meanwhile.
//
// Descriptor rows travel inside the kernel parameters (__grid_constant__, read
// through the constant cache) when a group has <= kInlineRows layers, so the first
// load of a tiny pack is not a dependent global load; larger groups read a device
// table.
#pragma once

#include "common.cuh"

namespace mgw {

enum class RowOp { kPack, kUnpack, kFill, kCheck };

struct RowsParam {
  Row inline_rows[kInlineRows];
  const Row* rows;  // device table, used when n_rows > kInlineRows
  int n_rows;
  int use_inline;
  float* bucket;
  int64_t total;  // bucket elements
  int64_t tile;   // bucket elements per CTA step (multiple of 4 * kThreads)
  float scale;
  const float* values;      // kFill / kCheck: one value per row
  const uint32_t* calls;    // comm pack: slot parity = (completed calls + 1) & 1
  int64_t slot_stride_elems;
  unsigned long long* mismatches;  // kCheck
  uint64_t* stamp;
};

__device__ __forceinline__ Row row_at(const RowsParam& p, int k) {
  return p.use_inline ? p.inline_rows[k] : p.rows[k];
}

__device__ __forceinline__ int row_covering(const RowsParam& p, int64_t e) {
  int lo = 0, hi = p.n_rows;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const Row r = row_at(p, mid);
    if (r.offset + r.count > e)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

template <RowOp kOp, bool kScale>
__device__ __forceinline__ void scalar_op(float* t, float* b, float scale, float value, unsigned long long& bad) {
  if constexpr (kOp == RowOp::kPack) {
    *b = kScale ? __fmul_rn(*t, scale) : *t;
  } else if constexpr (kOp == RowOp::kUnpack) {
    *t = *b;
  } else if constexpr (kOp == RowOp::kFill) {
    *t = value;
  } else {
    bad += (*t != value);
  }
}

constexpr int kRowsUnroll = 4;  // 16-B slots per thread per step

template <RowOp kOp, bool kScale>
__global__ void __launch_bounds__(kThreads, 2) rows_kernel(const __grid_constant__ RowsParam p) {
  grid_dep_wait();
  stamp_enter(p.stamp);
  float* bucket = p.bucket;
  if (p.calls != nullptr) bucket += (int64_t)((load_volatile32(p.calls) + 1u) & 1u) * p.slot_stride_elems;
  const float scale = p.scale;
  unsigned long long bad = 0;
  const int64_t tile = p.tile;
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < p.total; t0 += (int64_t)gridDim.x * tile) {
    const int64_t t1 = t0 + tile < p.total ? t0 + tile : p.total;
    int k = row_covering(p, t0 + 4 * threadIdx.x < t1 ? t0 + 4 * threadIdx.x : t0);
    Row cur = row_at(p, k < p.n_rows ? k : p.n_rows - 1);  // this thread's current row
    for (int64_t base = t0 + 4 * threadIdx.x; base < t1; base += 4 * kThreads * kRowsUnroll) {
      float* tp[kRowsUnroll];
      float value[kRowsUnroll];
      bool fast[kRowsUnroll];
      int ku[kRowsUnroll];
#pragma unroll
      for (int u = 0; u < kRowsUnroll; ++u) {
        const int64_t e = base + (int64_t)u * 4 * kThreads;
        fast[u] = false;
        tp[u] = nullptr;
        value[u] = 0.f;
        ku[u] = k;
        if (e < t1) {
          while (e >= cur.offset + cur.count) cur = row_at(p, ++k);
          ku[u] = k;
          tp[u] = cur.ptr + (e - cur.offset);
          if constexpr (kOp == RowOp::kFill || kOp == RowOp::kCheck) value[u] = p.values[k];
          fast[u] = e + 4 <= t1 && e + 4 <= cur.offset + cur.count && (reinterpret_cast<uintptr_t>(tp[u]) & 15) == 0;
        }
      }
      if constexpr (kOp == RowOp::kPack || kOp == RowOp::kUnpack || kOp == RowOp::kCheck) {
        float4 v[kRowsUnroll];
#pragma unroll
        for (int u = 0; u < kRowsUnroll; ++u) {
          if (fast[u]) {
            const int64_t e = base + (int64_t)u * 4 * kThreads;
            v[u] = (kOp == RowOp::kUnpack) ? *reinterpret_cast<const float4*>(bucket + e)
                                           : *reinterpret_cast<const float4*>(tp[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < kRowsUnroll; ++u) {
          if (!fast[u]) continue;
          const int64_t e = base + (int64_t)u * 4 * kThreads;
          if constexpr (kOp == RowOp::kPack) {
            *reinterpret_cast<float4*>(bucket + e) = kScale ? fmul4(v[u], scale) : v[u];
          } else if constexpr (kOp == RowOp::kUnpack) {
            *reinterpret_cast<float4*>(tp[u]) = v[u];
          } else {
            bad += (v[u].x != value[u]) + (v[u].y != value[u]) + (v[u].z != value[u]) + (v[u].w != value[u]);
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < kRowsUnroll; ++u)
          if (fast[u]) *reinterpret_cast<float4*>(tp[u]) = make_float4(value[u], value[u], value[u], value[u]);
      }
      // slow path: element by element, each finding its own row (unrolled so the per-u
      // arrays stay in registers)
#pragma unroll
      for (int u = 0; u < kRowsUnroll; ++u) {
        const int64_t e = base + (int64_t)u * 4 * kThreads;
        if (fast[u] || e >= t1) continue;
        int kk = ku[u];
        for (int j = 0; j < 4 && e + j < t1; ++j) {
          Row r = row_at(p, kk);
          while (e + j >= r.offset + r.count) r = row_at(p, ++kk);  // rows tile the bucket in order
          scalar_op<kOp, kScale>(r.ptr + (e + j - r.offset), bucket + e + j, scale, kOp == RowOp::kFill || kOp == RowOp::kCheck ? p.values[kk] : 0.f, bad);
        }
      }
    }
  }
  if constexpr (kOp == RowOp::kCheck) {
    if (bad) atomicAdd(p.mismatches, bad);
  }
  stamp_exit(p.stamp);
}

// Tile and grid for a bucket of `total` elements: at most one resident wave (512-thread
// CTAs at <= 64 registers -> 2 per SM) and exactly one tile per CTA, balanced to 16 B --
// ncu r01 showed fixed 64 KB tiles leaving 5.3 tiles per CTA (a 14 % tail) -- and at
// least one full step (one 16-B slot per thread) per CTA.
inline int rows_grid(int64_t total, int64_t* tile_out) {
  constexpr int64_t kStep = 4 * kThreads;
  const int64_t cap = (int64_t)kSMs * 2;
  int64_t grid = (total + kStep - 1) / kStep;
  grid = grid < 1 ? 1 : (grid > cap ? cap : grid);
  int64_t tile = (total + grid - 1) / grid;
  tile = (tile + 3) / 4 * 4;
  *tile_out = tile;
  return (int)((total + tile - 1) / tile);
}

// ------------------------------------------------------------------ TMA bulk path

constexpr int kBulkThreads = 128;            // warp 0: the TMA stream; warps 1-3: ragged edges
constexpr int kBulkStages = 4;
constexpr uint32_t kBulkChunk = 16384;       // bytes per stage
constexpr int64_t kBulkMinBytes = 1 << 20;   // smaller buckets: rows_kernel (latency, not bytes)
constexpr int kBulkCtasPerSM = 3;            // 3 x 64 KB of stages per SM

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(smem)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(smem)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// One row segment of a tile: bucket elements [a, b) of row `r`, split into a head (until
// the bucket address is 16-B aligned), a bulk middle (when the tensor address is then
// 16-B aligned too) and a tail; a misaligned row is all "head".
struct SegSplit {
  int64_t a, mid0, mid1, b;
};

__device__ __forceinline__ SegSplit split_segment(const Row& r, int64_t a, int64_t b) {
  SegSplit s{a, a, a, b};
  const int64_t head_end = (a + 3) / 4 * 4 < b ? (a + 3) / 4 * 4 : b;
  const float* t = r.ptr + (head_end - r.offset);
  if ((reinterpret_cast<uintptr_t>(t) & 15) != 0) {  // phases differ: the whole segment is scalar
    s.mid0 = s.mid1 = b;
    return s;
  }
  s.mid0 = head_end;
  s.mid1 = head_end + (b - head_end) / 4 * 4;
  return s;
}

template <bool kPack>
__global__ void __launch_bounds__(kBulkThreads) bulk_rows_kernel(const __grid_constant__ RowsParam p) {
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t full[kBulkStages];
  grid_dep_wait();
  stamp_enter(p.stamp);
  float* bucket = p.bucket;
  if (p.calls != nullptr) bucket += (int64_t)((load_volatile32(p.calls) + 1u) & 1u) * p.slot_stride_elems;
  const int64_t t0 = (int64_t)blockIdx.x * p.tile;
  const int64_t t1 = t0 + p.tile < p.total ? t0 + p.tile : p.total;
  if (threadIdx.x == 0)
    for (int i = 0; i < kBulkStages; ++i) mbar_init(&full[i]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (t0 < t1) {
    const int k_first = row_covering(p, t0);
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) {
        // warp 0, one thread: stream every aligned middle through the stage ring; chunk c
        // uses stage c % S; its load is issued S - 1 chunks ahead of its store
        struct Chunk {
          const float* src;
          float* dst;
          uint32_t bytes;
        };
        Chunk ring[kBulkStages];
        int k = k_first;
        int64_t pos = t0;  // next bucket element to consider
        int64_t c_next = 0, c_store = 0;
        auto next_chunk = [&](Chunk& out) -> bool {
          while (pos < t1 && k < p.n_rows) {
            const Row r = row_at(p, k);
            const int64_t a = pos > r.offset ? pos : r.offset;
            const int64_t b = r.offset + r.count < t1 ? r.offset + r.count : t1;
            if (a >= b) {
              ++k;
              continue;
            }
            const SegSplit sg = split_segment(r, a, b);
            int64_t m0 = a < sg.mid0 ? sg.mid0 : a;
            if (m0 < sg.mid1) {
              const int64_t m1 = m0 + (int64_t)(kBulkChunk / 4) < sg.mid1 ? m0 + (int64_t)(kBulkChunk / 4) : sg.mid1;
              float* tens = const_cast<float*>(r.ptr) + (m0 - r.offset);
              out.src = kPack ? tens : bucket + m0;
              out.dst = kPack ? bucket + m0 : tens;
              out.bytes = (uint32_t)((m1 - m0) * 4);
              pos = m1;
              if (pos >= b) ++k;
              return true;
            }
            pos = b;
            ++k;
          }
          return false;
        };
        // prologue: S - 1 loads in flight
        for (; c_next < kBulkStages - 1; ++c_next) {
          Chunk& ch = ring[c_next % kBulkStages];
          if (!next_chunk(ch)) break;
          mbar_expect_tx(&full[c_next % kBulkStages], ch.bytes);
          bulk_load(stage + (c_next % kBulkStages) * kBulkChunk, ch.src, ch.bytes, &full[c_next % kBulkStages]);
        }
        bool more = c_next == kBulkStages - 1;
        for (; c_store < c_next; ++c_store) {
          const int st = (int)(c_store % kBulkStages);
          mbar_wait(&full[st], (uint32_t)((c_store / kBulkStages) & 1));
          bulk_store(ring[st].dst, stage + st * kBulkChunk, ring[st].bytes);
          // refill: chunk c_next takes the stage of chunk c_store - 1, whose store must have
          // finished reading it -- at most the store just issued may still be reading
          if (more) {
            Chunk& ch = ring[c_next % kBulkStages];
            if (next_chunk(ch)) {
              bulk_wait_read_1();
              mbar_expect_tx(&full[c_next % kBulkStages], ch.bytes);
              bulk_load(stage + (c_next % kBulkStages) * kBulkChunk, ch.src, ch.bytes, &full[c_next % kBulkStages]);
              ++c_next;
            } else {
              more = false;
            }
          }
        }
        bulk_wait_all();
      }
    } else {
      // warps 1-3: the scalar parts (row heads / tails, misaligned rows)
      const int tid = threadIdx.x - 32, nt = kBulkThreads - 32;
      for (int k = k_first; k < p.n_rows; ++k) {
        const Row r = row_at(p, k);
        if (r.offset >= t1) break;
        const int64_t a = t0 > r.offset ? t0 : r.offset;
        const int64_t b = r.offset + r.count < t1 ? r.offset + r.count : t1;
        if (a >= b) continue;
        const SegSplit sg = split_segment(r, a, b);
        for (int64_t e = a + tid; e < sg.mid0; e += nt) {
          float* t = const_cast<float*>(r.ptr) + (e - r.offset);
          if (kPack) bucket[e] = *t; else *t = bucket[e];
        }
        for (int64_t e = sg.mid1 + tid; e < b; e += nt) {
          float* t = const_cast<float*>(r.ptr) + (e - r.offset);
          if (kPack) bucket[e] = *t; else *t = bucket[e];
        }
      }
    }
  }
  stamp_exit(p.stamp);
}

inline int bulk_rows_grid(int64_t total, int64_t* tile_out) {
  const int64_t cap = (int64_t)kSMs * kBulkCtasPerSM;
  const int64_t per_chunk = kBulkChunk / 4;
  int64_t grid = (total + per_chunk - 1) / per_chunk;
  grid = grid < 1 ? 1 : (grid > cap ? cap : grid);
  int64_t tile = (total + grid - 1) / grid;
  tile = (tile + 3) / 4 * 4;
  *tile_out = tile;
  return (int)((total + tile - 1) / tile);
}

}  // namespace mgw
