// k_ll.cu -- host launchers of the ll.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "ll.cuh"

namespace mgw {

template <int N>
int launch_ll_n(const LLArgs& l0, int max_ctas, cudaStream_t stream) {
  const int64_t pairs = (l0.f.ar.n + 1) >> 1;
  LLArgs l = l0;
  const int grid = grid_for(pairs, kThreads, max_ctas < kSMs ? max_ctas : kSMs);
  l.f.ar.tag = collective_tag(l0.f.ar.tag, l0.f.ar.n, kTagLL, grid, l0.f.scale);
  ll_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(l);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_ll(const LLArgs& l, int max_ctas, cudaStream_t stream) {
  if (l.f.ar.n > kLLMaxElems) return set_error(MGW_EINVAL, "LL path takes at most %lld elements", (long long)kLLMaxElems);
  switch (l.f.ar.world) {
    case 2: return launch_ll_n<2>(l, max_ctas, stream);
    case 3: return launch_ll_n<3>(l, max_ctas, stream);
    case 4: return launch_ll_n<4>(l, max_ctas, stream);
    case 5: return launch_ll_n<5>(l, max_ctas, stream);
    case 6: return launch_ll_n<6>(l, max_ctas, stream);
    case 7: return launch_ll_n<7>(l, max_ctas, stream);
    case 8: return launch_ll_n<8>(l, max_ctas, stream);
    default: return set_error(MGW_EINVAL, "LL path needs 2..%d ranks, got %d", kMaxRanks, l.f.ar.world);
  }
}

}  // namespace mgw
