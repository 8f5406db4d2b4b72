// k_fused.cu -- host launchers of the fused.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "fused.cuh"

namespace mgw {

int plan_fused(FusedArgs& f, int algo, int max_ctas, const int64_t* per_cta) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  const int w = f.ar.world;
  const int64_t nv = f.ar.n >> 2;
  const bool one = algo == MGW_ALGO_ONESHOT;
  const int grid = one ? collective_grid_rt(w, nv, per_cta ? per_cta[0] : 0, max_ctas)
                       : collective_grid_rt(w, nv / (w > 0 ? w : 1), per_cta ? per_cta[1] : 0, max_ctas);
  f.ar.tag = collective_tag(f.ar.tag, f.ar.n, one ? kTagFusedOneshot : kTagFusedTwoshot, grid, f.scale);
  return grid;
}

template <int N>
static int launch_fused_n(const FusedArgs& f, int algo, int grid, cudaStream_t stream) {
  if (N == 1 && algo != MGW_ALGO_ONESHOT)  // one rank: the one-input fold is the one-shot
    return set_error(MGW_EINVAL, "a single rank runs the one-shot group kernel only");
  if constexpr (N == 1) {
    fused_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  } else {
    if (algo == MGW_ALGO_ONESHOT)
      fused_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
    else
      fused_twoshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_fused(const FusedArgs& f0, int algo, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  FusedArgs f = f0;
  const int grid = plan_fused(f, algo, max_ctas, per_cta);
  switch (f.ar.world) {
    case 1: return launch_fused_n<1>(f, algo, grid, stream);
    case 2: return launch_fused_n<2>(f, algo, grid, stream);
    case 3: return launch_fused_n<3>(f, algo, grid, stream);
    case 4: return launch_fused_n<4>(f, algo, grid, stream);
    case 5: return launch_fused_n<5>(f, algo, grid, stream);
    case 6: return launch_fused_n<6>(f, algo, grid, stream);
    case 7: return launch_fused_n<7>(f, algo, grid, stream);
    case 8: return launch_fused_n<8>(f, algo, grid, stream);
    default: return set_error(MGW_EINVAL, "world %d outside 1..%d", f.ar.world, kMaxRanks);
  }
}

template <int N>
static int group_fused_n(const RankGroup<FusedArgs>& g, int algo, cudaStream_t stream) {
  return algo == MGW_ALGO_ONESHOT ? launch_cooperative(fused_oneshot_group<N>, g, stream)
                                  : launch_cooperative(fused_twoshot_group<N>, g, stream);
}

int launch_fused_group(const RankGroup<FusedArgs>& g, int world, int algo, cudaStream_t stream) {
  switch (world) {
    case 2: return group_fused_n<2>(g, algo, stream);
    case 3: return group_fused_n<3>(g, algo, stream);
    case 4: return group_fused_n<4>(g, algo, stream);
    case 5: return group_fused_n<5>(g, algo, stream);
    case 6: return group_fused_n<6>(g, algo, stream);
    case 7: return group_fused_n<7>(g, algo, stream);
    case 8: return group_fused_n<8>(g, algo, stream);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

MGW_DEFINE_VIOLATIONS(fused)

}  // namespace mgw
