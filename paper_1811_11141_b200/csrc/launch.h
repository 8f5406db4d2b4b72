// launch.h -- host launchers of every kernel family.  Each family lives in its own
// translation unit (k_*.cu) so the sm_100a build compiles them in parallel; the C ABI
// (mgwfbp_b200.cu) only sees these declarations and the argument structs.
#pragma once

#include "allreduce.cuh"
#include "fused.cuh"
#include "ll.cuh"
#include "nvls.cuh"
#include "pipe.cuh"
#include "b16push.cuh"
#include "ll128.cuh"
#include "rows.cuh"

namespace mgw {

int launch_allreduce(const ArArgs& a, int algo, int max_ctas, cudaStream_t stream, const int64_t* per_cta = nullptr);
int launch_fused(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream, const int64_t* per_cta = nullptr);
int launch_push(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta);
int launch_push1(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta);
int launch_push_pipe(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta);
int launch_ll(const LLArgs& l, int max_ctas, cudaStream_t stream);
int launch_ll_b16(const LLArgs& l, int max_ctas, cudaStream_t stream);
int launch_b16(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream);
int launch_b16_push(const PushArgs& x, int max_ctas, cudaStream_t stream);
int launch_ll128(const L128Args& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta, bool b16, bool one);
int launch_nvls(const NvlsArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta);

// plan_*: the grid a launch uses for these arguments and settings; stamps the collective
// tag into the arguments (the plain launchers above plan, then launch).
int plan_fused(FusedArgs& f, int algo, int max_ctas, const int64_t* per_cta);
int plan_push(PushArgs& x, int max_ctas, const int64_t* per_cta);
int plan_push1(PushArgs& x, int max_ctas, const int64_t* per_cta);
int plan_push_pipe(PushArgs& x, int max_ctas, const int64_t* per_cta);
int plan_ll(LLArgs& l, int max_ctas);
int plan_ll_b16(LLArgs& l, int max_ctas);
int plan_b16(FusedArgs& f, int algo, int max_ctas);
int plan_b16_push(PushArgs& x, int max_ctas);
int plan_ll128(L128Args& x, int max_ctas, const int64_t* per_cta, bool b16, bool one);

// Rank-group launches: every rank's planned CTAs in ONE cooperative launch on one device
// (co-residency guaranteed, so ranks that wait on one another always run together).
int launch_fused_group(const RankGroup<FusedArgs>& g, int world, int algo, cudaStream_t stream);
int launch_push_group(const RankGroup<PushArgs>& g, int world, int kind /* 0 two-shot, 1 one-shot, 2 pipe */,
                      cudaStream_t stream);
int launch_ll_group(const RankGroup<LLArgs>& g, int world, cudaStream_t stream);
int launch_b16_group(const RankGroup<FusedArgs>& g, int world, int algo, cudaStream_t stream);
int launch_ll_b16_group(const RankGroup<LLArgs>& g, int world, cudaStream_t stream);
int launch_b16_push_group(const RankGroup<PushArgs>& g, int world, cudaStream_t stream);
int launch_ll128_group(const RankGroup<L128Args>& g, int world, cudaStream_t stream, bool b16, bool one);

template <class Args>
inline int launch_cooperative(void (*kernel)(const RankGroup<Args>), const RankGroup<Args>& g, cudaStream_t stream) {
  const int blocks = g.first[kMaxRanks];
  if (blocks <= 0) return MGW_OK;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, g);
  if (e != cudaSuccess)
    return set_error(MGW_ECUDA, "cooperative rank-group launch of %d CTAs: %s", blocks, cudaGetErrorString(e));
  return MGW_OK;
}

int set_rows_path(int v);
int set_pipe_sub_slots(int64_t v);  // pipelined two-shot: slots per sub-chunk per part

// checked build: per translation unit violation counters (MGW_EXPECT in common.cuh)
int violations_allreduce(unsigned long long* out, bool reset);
int violations_bf16(unsigned long long* out, bool reset);
int violations_fused(unsigned long long* out, bool reset);
int violations_ll(unsigned long long* out, bool reset);
int violations_ll128(unsigned long long* out, bool reset);
int violations_nvls(unsigned long long* out, bool reset);
int violations_push(unsigned long long* out, bool reset);
int violations_rows(unsigned long long* out, bool reset);  // 0 auto, 1 LDG rows_kernel only, 2 TMA bulk wherever allowed

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
