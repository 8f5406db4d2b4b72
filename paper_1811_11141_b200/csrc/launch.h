// launch.h -- host launchers of every kernel family.  Each family lives in its own
// translation unit (k_*.cu) so the sm_100a build compiles them in parallel; the C ABI
// (mgwfbp_b200.cu) only sees these declarations and the argument structs.
#pragma once

#include "allreduce.cuh"
#include "fused.cuh"
#include "ll.cuh"
#include "nvls.cuh"
#include "push.cuh"
#include "rows.cuh"

namespace mgw {

int launch_allreduce(const ArArgs& a, int algo, int max_ctas, cudaStream_t stream, const int64_t* per_cta = nullptr);
int launch_fused(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream, const int64_t* per_cta = nullptr);
int launch_push(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta);
int launch_push1(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta);
int launch_ll(const LLArgs& l, int max_ctas, cudaStream_t stream);
int launch_ll_b16(const LLArgs& l, int max_ctas, cudaStream_t stream);
int launch_b16(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream);
int launch_nvls(const NvlsArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta);

template <RowOp kOp>
int launch_rows(const Row* host_rows, const Row* dev_rows, int n_rows, float* bucket, int64_t total, float scale,
                const float* values, const uint32_t* calls, int64_t slot_stride_elems,
                unsigned long long* mismatches, cudaStream_t stream, uint64_t* stamp = nullptr,
                cudaEvent_t pdl_event = nullptr);
extern template int launch_rows<RowOp::kPack>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                              const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                              cudaEvent_t);
extern template int launch_rows<RowOp::kUnpack>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                                const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                                cudaEvent_t);
extern template int launch_rows<RowOp::kFill>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                              const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                              cudaEvent_t);
extern template int launch_rows<RowOp::kCheck>(const Row*, const Row*, int, float*, int64_t, float, const float*,
                                               const uint32_t*, int64_t, unsigned long long*, cudaStream_t, uint64_t*,
                                               cudaEvent_t);

}  // namespace mgw
