// k_rows.cu -- host launchers of the rows.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "rows.cuh"

namespace mgw {

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
}  // namespace mgw
