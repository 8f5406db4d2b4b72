// k_bf16.cu -- host launchers of the bf16.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "bf16.cuh"

namespace mgw {

int launch_ll_b16(const LLArgs& l0, int max_ctas, cudaStream_t stream) {
  LLArgs l = l0;
  if (l.f.ar.n > 2 * kLLMaxElems)
    return set_error(MGW_EINVAL, "bf16 LL path takes at most %lld elements", (long long)(2 * kLLMaxElems));
  const int64_t quads = (l.f.ar.n + 3) >> 2;
  const int grid = grid_for(quads, kThreads, max_ctas < kSMs ? max_ctas : kSMs);
  l.f.ar.tag = collective_tag(l0.f.ar.tag, l0.f.ar.n, kTagB16LL, grid, l0.f.scale);
  switch (l.f.ar.world) {
    case 2: ll_b16_kernel<2><<<grid, kThreads, 0, stream>>>(l); break;
    case 3: ll_b16_kernel<3><<<grid, kThreads, 0, stream>>>(l); break;
    case 4: ll_b16_kernel<4><<<grid, kThreads, 0, stream>>>(l); break;
    case 5: ll_b16_kernel<5><<<grid, kThreads, 0, stream>>>(l); break;
    case 6: ll_b16_kernel<6><<<grid, kThreads, 0, stream>>>(l); break;
    case 7: ll_b16_kernel<7><<<grid, kThreads, 0, stream>>>(l); break;
    case 8: ll_b16_kernel<8><<<grid, kThreads, 0, stream>>>(l); break;
    default: return set_error(MGW_EINVAL, "LL path needs 2..%d ranks, got %d", kMaxRanks, l.f.ar.world);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

template <int N>
int launch_b16_n(const FusedArgs& f0, int algo, int max_ctas, cudaStream_t stream) {
  const int64_t nv = f0.ar.n / kB16;
  FusedArgs f = f0;
  if (algo == MGW_ALGO_ONESHOT) {
    const int grid = collective_grid<N>(nv, 0, max_ctas);
    f.ar.tag = collective_tag(f0.ar.tag, f0.ar.n, kTagB16Oneshot, grid, f0.scale);
    b16_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  } else {
    const int grid = collective_grid<N>(nv / N, 0, max_ctas);
    f.ar.tag = collective_tag(f0.ar.tag, f0.ar.n, kTagB16Twoshot, grid, f0.scale);
    b16_twoshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_b16(const FusedArgs& f, int algo, int max_ctas, cudaStream_t stream) {
  if (algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT)
    return set_error(MGW_EINVAL, "bf16 buckets support one-shot and two-shot only (algorithm %d)", algo);
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  switch (f.ar.world) {
    case 1: return launch_b16_n<1>(f, algo, max_ctas, stream);
    case 2: return launch_b16_n<2>(f, algo, max_ctas, stream);
    case 3: return launch_b16_n<3>(f, algo, max_ctas, stream);
    case 4: return launch_b16_n<4>(f, algo, max_ctas, stream);
    case 5: return launch_b16_n<5>(f, algo, max_ctas, stream);
    case 6: return launch_b16_n<6>(f, algo, max_ctas, stream);
    case 7: return launch_b16_n<7>(f, algo, max_ctas, stream);
    case 8: return launch_b16_n<8>(f, algo, max_ctas, stream);
    default: return set_error(MGW_EINVAL, "world %d outside 1..%d", f.ar.world, kMaxRanks);
  }
}

}  // namespace mgw
