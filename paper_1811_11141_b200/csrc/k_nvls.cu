// k_nvls.cu -- host launchers of the nvls.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "nvls.cuh"

namespace mgw {

int launch_nvls(const NvlsArgs& x0, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  NvlsArgs x = x0;
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  const int64_t nv = x.f.ar.n >> 2;
  const int64_t per = per_cta && per_cta[1] > 0 ? per_cta[1] : (int64_t)kThreads * 4;
  const int grid = grid_for(nv / (x.f.ar.world > 0 ? x.f.ar.world : 1), per, max_ctas);
  x.f.ar.tag = collective_tag(x0.f.ar.tag, x0.f.ar.n, kTagNvls, grid, x0.f.scale);
  switch (x.f.ar.world) {
    case 2: nvls_kernel<2><<<grid, kThreads, 0, stream>>>(x); break;
    case 3: nvls_kernel<3><<<grid, kThreads, 0, stream>>>(x); break;
    case 4: nvls_kernel<4><<<grid, kThreads, 0, stream>>>(x); break;
    case 5: nvls_kernel<5><<<grid, kThreads, 0, stream>>>(x); break;
    case 6: nvls_kernel<6><<<grid, kThreads, 0, stream>>>(x); break;
    case 7: nvls_kernel<7><<<grid, kThreads, 0, stream>>>(x); break;
    case 8: nvls_kernel<8><<<grid, kThreads, 0, stream>>>(x); break;
    default: return set_error(MGW_EINVAL, "NVLS needs 2..%d ranks, got %d", kMaxRanks, x.f.ar.world);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

MGW_DEFINE_VIOLATIONS(nvls)

}  // namespace mgw
