// k_allreduce.cu -- host launchers of the allreduce.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "allreduce.cuh"

namespace mgw {

template <int N>
int launch_allreduce_n(const ArArgs& a0, int algo, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  const int64_t nv = a0.n >> 2;
  ArArgs a = a0;
  if (algo == MGW_ALGO_ONESHOT) {
    const int grid = collective_grid<N>(nv, per_cta ? per_cta[0] : 0, max_ctas);
    a.tag = collective_tag(a0.tag, a0.n, kTagOneshot, grid, 1.f);
    oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(a);
  } else {
    const int grid = collective_grid<N>(nv / N, per_cta ? per_cta[1] : 0, max_ctas);
    a.tag = collective_tag(a0.tag, a0.n, kTagTwoshot, grid, 1.f);
    twoshot_kernel<N><<<grid, kThreads, 0, stream>>>(a);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_allreduce(const ArArgs& a, int algo, int max_ctas, cudaStream_t stream,
                            const int64_t* per_cta) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;  // one barrier flag slot per CTA
  switch (a.world) {
    case 1: return launch_allreduce_n<1>(a, algo, max_ctas, stream, per_cta);
    case 2: return launch_allreduce_n<2>(a, algo, max_ctas, stream, per_cta);
    case 3: return launch_allreduce_n<3>(a, algo, max_ctas, stream, per_cta);
    case 4: return launch_allreduce_n<4>(a, algo, max_ctas, stream, per_cta);
    case 5: return launch_allreduce_n<5>(a, algo, max_ctas, stream, per_cta);
    case 6: return launch_allreduce_n<6>(a, algo, max_ctas, stream, per_cta);
    case 7: return launch_allreduce_n<7>(a, algo, max_ctas, stream, per_cta);
    case 8: return launch_allreduce_n<8>(a, algo, max_ctas, stream, per_cta);
    default: return set_error(MGW_EINVAL, "world %d outside 1..%d", a.world, kMaxRanks);
  }
}

MGW_DEFINE_VIOLATIONS(allreduce)

}  // namespace mgw
