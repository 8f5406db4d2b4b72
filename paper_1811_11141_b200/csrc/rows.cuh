// rows.cuh -- K1 pack(+scale), K4 unpack, and the fill / check helpers.
//
// A merge group's bucket is the concatenation of its layer gradients, layer `high`
// first (allreduce_net.py:499-509).  The kernels walk the *bucket* in 8-64 KB tiles,
// one tile per CTA step; every thread owns fixed 16-B slots of the tile and finds the
// layer row holding each slot by a forward scan (rows are sorted by bucket offset, so
// the scan is monotone per thread).  A slot that lies inside one row at a 16-B aligned
// tensor address moves as one 128-bit access; slots that straddle two rows or sit at a
// misaligned tensor address fall back to four scalar accesses.  All 512 threads stay
// busy whatever the mix of row sizes (BERT has 124 tensors <= 3,072 elements).
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
          Row r = row_at(p, k);
          while (e >= r.offset + r.count) r = row_at(p, ++k);
          ku[u] = k;
          tp[u] = r.ptr + (e - r.offset);
          if constexpr (kOp == RowOp::kFill || kOp == RowOp::kCheck) value[u] = p.values[k];
          fast[u] = e + 4 <= t1 && e + 4 <= r.offset + r.count && (reinterpret_cast<uintptr_t>(tp[u]) & 15) == 0;
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

// Tile and grid for a bucket of `total` elements.  At most one resident wave: 512-thread
// CTAs at <= 64 registers (spill-free with the unrolled slow path) -> 2 per SM (a grid
// beyond the resident wave leaves a tail, ncu r01).  A mid-sized group (a 9.4 MB ResNet
// layer) is spread over the whole wave with smaller tiles instead of parking on 144
// CTAs of 64 KB: more SMs, more bytes in flight.
inline int rows_grid(int64_t total, int64_t* tile_out) {
  constexpr int64_t kStep = 4 * kThreads;  // one 16-B slot per thread
  const int64_t cap = (int64_t)kSMs * 2;
  int64_t tile = (total + cap - 1) / cap;
  tile = (tile + kStep - 1) / kStep * kStep;
  tile = tile < kStep ? kStep : (tile > kTile ? kTile : tile);
  *tile_out = tile;
  const int64_t tiles = (total + tile - 1) / tile;
  return (int)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap));
}

// Launch one row operation over a bucket of `total` elements.  `host_rows` must
// mirror `dev_rows` (same rows); rows must tile [0, total) contiguously in order.
}  // namespace mgw
