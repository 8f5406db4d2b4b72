// k_fused.cu -- host launchers of the fused.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "fused.cuh"

namespace mgw {

template <int N>
int launch_fused_n(const FusedArgs& f0, int algo, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  const int64_t nv = f0.ar.n >> 2;
  FusedArgs f = f0;
  if (algo == MGW_ALGO_ONESHOT) {
    const int grid = collective_grid<N>(nv, per_cta ? per_cta[0] : 0, max_ctas);
    f.ar.tag = collective_tag(f0.ar.tag, f0.ar.n, kTagFusedOneshot, grid, f0.scale);
    fused_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  } else {
    const int grid = collective_grid<N>(nv / N, per_cta ? per_cta[1] : 0, max_ctas);
    f.ar.tag = collective_tag(f0.ar.tag, f0.ar.n, kTagFusedTwoshot, grid, f0.scale);
    fused_twoshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_fused(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream,
                        const int64_t* per_cta) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  switch (f.ar.world) {
    case 1: return launch_fused_n<1>(f, algo, max_ctas, stream, per_cta);
    case 2: return launch_fused_n<2>(f, algo, max_ctas, stream, per_cta);
    case 3: return launch_fused_n<3>(f, algo, max_ctas, stream, per_cta);
    case 4: return launch_fused_n<4>(f, algo, max_ctas, stream, per_cta);
    case 5: return launch_fused_n<5>(f, algo, max_ctas, stream, per_cta);
    case 6: return launch_fused_n<6>(f, algo, max_ctas, stream, per_cta);
    case 7: return launch_fused_n<7>(f, algo, max_ctas, stream, per_cta);
    case 8: return launch_fused_n<8>(f, algo, max_ctas, stream, per_cta);
    default: return set_error(MGW_EINVAL, "world %d outside 1..%d", f.ar.world, kMaxRanks);
  }
}

}  // namespace mgw
