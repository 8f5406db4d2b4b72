// k_ll.cu -- host launchers of the ll.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "ll.cuh"

namespace mgw {

int plan_ll(LLArgs& l, int max_ctas) {
  const int64_t pairs = (l.f.ar.n + 1) >> 1;
  const int grid = grid_for(pairs, kThreads, max_ctas < kSMs ? max_ctas : kSMs);
  l.f.ar.tag = collective_tag(l.f.ar.tag, l.f.ar.n, kTagLL, grid, l.f.scale);
  return grid;
}

template <int N>
static int launch_ll_n(const LLArgs& l, int grid, cudaStream_t stream) {
  ll_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(l);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_ll(const LLArgs& l0, int max_ctas, cudaStream_t stream) {
  if (l0.f.ar.n > kLLMaxElems) return set_error(MGW_EINVAL, "LL path takes at most %lld elements", (long long)kLLMaxElems);
  LLArgs l = l0;
  const int grid = plan_ll(l, max_ctas);
  switch (l.f.ar.world) {
    case 2: return launch_ll_n<2>(l, grid, stream);
    case 3: return launch_ll_n<3>(l, grid, stream);
    case 4: return launch_ll_n<4>(l, grid, stream);
    case 5: return launch_ll_n<5>(l, grid, stream);
    case 6: return launch_ll_n<6>(l, grid, stream);
    case 7: return launch_ll_n<7>(l, grid, stream);
    case 8: return launch_ll_n<8>(l, grid, stream);
    default: return set_error(MGW_EINVAL, "LL path needs 2..%d ranks, got %d", kMaxRanks, l.f.ar.world);
  }
}

int launch_ll_group(const RankGroup<LLArgs>& g, int world, cudaStream_t stream) {
  switch (world) {
    case 2: return launch_cooperative(ll_oneshot_group<2>, g, stream);
    case 3: return launch_cooperative(ll_oneshot_group<3>, g, stream);
    case 4: return launch_cooperative(ll_oneshot_group<4>, g, stream);
    case 5: return launch_cooperative(ll_oneshot_group<5>, g, stream);
    case 6: return launch_cooperative(ll_oneshot_group<6>, g, stream);
    case 7: return launch_cooperative(ll_oneshot_group<7>, g, stream);
    case 8: return launch_cooperative(ll_oneshot_group<8>, g, stream);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

MGW_DEFINE_VIOLATIONS(ll)

}  // namespace mgw
