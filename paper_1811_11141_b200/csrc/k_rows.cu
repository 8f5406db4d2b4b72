// k_rows.cu -- host launchers of the rows.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "rows.cuh"

namespace mgw {

// rows path: 0 = auto (TMA bulk for large aligned pack / unpack), 1 = LDG kernel only,
// 2 = bulk wherever allowed (mgw_set_option(MGW_OPT_ROWS_PATH, ...), for A/B runs)
static int g_rows_path = 0;

int set_rows_path(int v) {
  if (v < 0 || v > 2) return set_error(MGW_EINVAL, "rows path must be 0, 1 or 2");
  g_rows_path = v;
  return MGW_OK;
}

// TMA bulk copies need 16-B aligned bucket and tensor addresses: take the bulk path when
// the bucket is large and at least 15/16 of its bytes sit in phase-aligned rows.
static bool use_bulk(const Row* host_rows, int n_rows, const float* bucket, int64_t total, float scale) {
  if (g_rows_path == 1 || scale != 1.0f || host_rows == nullptr) return false;
  if ((reinterpret_cast<uintptr_t>(bucket) & 15) != 0) return false;
  if (g_rows_path == 0 && total * 4 < kBulkMinBytes) return false;
  int64_t aligned = 0;
  for (int k = 0; k < n_rows; ++k) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(host_rows[k].ptr) - (uintptr_t)host_rows[k].offset * 4;
    if ((base & 15) == 0) aligned += host_rows[k].count;
  }
  return aligned * 16 >= total * 15;
}

template <bool kPack>
static int launch_bulk_rows(RowsParam& p, cudaStream_t stream) {
  static bool configured = false;
  const int smem = kBulkStages * (int)kBulkChunk;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(bulk_rows_kernel<kPack>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_error(MGW_ECUDA, "bulk rows smem: %s", cudaGetErrorString(e));
    configured = true;
  }
  const int grid = bulk_rows_grid(p.total, &p.tile);
  bulk_rows_kernel<kPack><<<grid, kBulkThreads, smem, stream>>>(p);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

template <RowOp kOp>
int launch_rows(const Row* host_rows, const Row* dev_rows, int n_rows, float* bucket, int64_t total, float scale,
                const float* values, const uint32_t* calls, int64_t slot_stride_elems,
                unsigned long long* mismatches, cudaStream_t stream, uint64_t* stamp,
                cudaEvent_t pdl_event) {
  if (total <= 0 || n_rows <= 0) return MGW_OK;
  RowsParam p;
  p.use_inline = n_rows <= kInlineRows && host_rows != nullptr;
  if (p.use_inline)
    for (int k = 0; k < n_rows; ++k) p.inline_rows[k] = host_rows[k];
  p.rows = dev_rows;
  p.n_rows = n_rows;
  p.bucket = bucket;
  p.total = total;
  p.scale = scale;
  p.values = values;
  p.calls = calls;
  p.slot_stride_elems = slot_stride_elems;
  p.mismatches = mismatches;
  p.stamp = stamp;
  if (!p.use_inline && dev_rows == nullptr) return set_error(MGW_EINVAL, "row table missing");
  if constexpr (kOp == RowOp::kPack || kOp == RowOp::kUnpack) {
    if (pdl_event == nullptr && use_bulk(host_rows, n_rows, bucket, total, kOp == RowOp::kPack ? scale : 1.0f))
      return launch_bulk_rows<kOp == RowOp::kPack>(p, stream);
  }
  const int grid = rows_grid(total, &p.tile);
  if (pdl_event != nullptr) {
    // record `pdl_event` as a programmatic event that fires once every block has started:
    // the consumer (the group's exchange) launches early and waits in grid_dep_wait()
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticEvent;
    attr[0].val.programmaticEvent.event = pdl_event;
    attr[0].val.programmaticEvent.flags = 0;
    attr[0].val.programmaticEvent.triggerAtBlockStart = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = (kOp == RowOp::kPack && scale != 1.0f) ? cudaLaunchKernelEx(&cfg, rows_kernel<kOp, true>, p)
                                                            : cudaLaunchKernelEx(&cfg, rows_kernel<kOp, false>, p);
    if (e != cudaSuccess) return set_error(MGW_ECUDA, "programmatic launch: %s", cudaGetErrorString(e));
    return MGW_OK;
  }
  if (kOp == RowOp::kPack && scale != 1.0f)
    rows_kernel<kOp, true><<<grid, kThreads, 0, stream>>>(p);
  else
    rows_kernel<kOp, false><<<grid, kThreads, 0, stream>>>(p);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

}  // namespace mgw

namespace mgw {
template int launch_rows<RowOp::kPack>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                       const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                       cudaEvent_t);
template int launch_rows<RowOp::kUnpack>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                         const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                         cudaEvent_t);
template int launch_rows<RowOp::kFill>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                       const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                       cudaEvent_t);
template int launch_rows<RowOp::kCheck>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                        const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                        cudaEvent_t);
MGW_DEFINE_VIOLATIONS(rows)

}  // namespace mgw
