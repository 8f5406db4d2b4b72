// k_push.cu -- host launchers of the push.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "push.cuh"

namespace mgw {

template <int N>
int launch_push1_n(const PushArgs& x0, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  PushArgs x = x0;
  const int grid = collective_grid<N>(x0.f.ar.n >> 2, per_cta ? per_cta[0] : 0, max_ctas);
  x.f.ar.tag = collective_tag(x0.f.ar.tag, x0.f.ar.n, kTagPushOneshot, grid, x0.f.scale);
  push_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_push1(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  switch (x.f.ar.world) {
    case 2: return launch_push1_n<2>(x, max_ctas, stream, per_cta);
    case 3: return launch_push1_n<3>(x, max_ctas, stream, per_cta);
    case 4: return launch_push1_n<4>(x, max_ctas, stream, per_cta);
    case 5: return launch_push1_n<5>(x, max_ctas, stream, per_cta);
    case 6: return launch_push1_n<6>(x, max_ctas, stream, per_cta);
    case 7: return launch_push1_n<7>(x, max_ctas, stream, per_cta);
    case 8: return launch_push1_n<8>(x, max_ctas, stream, per_cta);
    default: return set_error(MGW_EINVAL, "push one-shot needs 2..%d ranks, got %d", kMaxRanks, x.f.ar.world);
  }
}

int launch_push(const PushArgs& x0, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  PushArgs x = x0;
  const int64_t nv = x.f.ar.n >> 2;
  int64_t per = per_cta ? per_cta[1] : 0;
  if (per <= 0) {
    // large buckets stream better in long per-CTA chunks: 2048-4096 slots (32-64 KB per
    // part) per CTA, spread over one CTA per SM (profiles/grid_pushtune_n4_r01.json:
    // 32 MB 105 -> 98 us, 64 MB 195 -> 180 us at N = 4)
    const int64_t part = nv / (x.f.ar.world > 0 ? x.f.ar.world : 1);
    per = (part + kSMs - 1) / kSMs;
    per = (per + 127) / 128 * 128;
    per = per < 2048 ? 2048 : (per > 4096 ? 4096 : per);
  }
  const int grid = grid_for(nv / (x0.f.ar.world > 0 ? x0.f.ar.world : 1), per, max_ctas);
  x.f.ar.tag = collective_tag(x0.f.ar.tag, x0.f.ar.n, kTagPush, grid, x0.f.scale);
  switch (x.f.ar.world) {
    case 2: push_twoshot_kernel<2><<<grid, kThreads, 0, stream>>>(x); break;
    case 3: push_twoshot_kernel<3><<<grid, kThreads, 0, stream>>>(x); break;
    case 4: push_twoshot_kernel<4><<<grid, kThreads, 0, stream>>>(x); break;
    case 5: push_twoshot_kernel<5><<<grid, kThreads, 0, stream>>>(x); break;
    case 6: push_twoshot_kernel<6><<<grid, kThreads, 0, stream>>>(x); break;
    case 7: push_twoshot_kernel<7><<<grid, kThreads, 0, stream>>>(x); break;
    case 8: push_twoshot_kernel<8><<<grid, kThreads, 0, stream>>>(x); break;
    default: return set_error(MGW_EINVAL, "push two-shot needs 2..%d ranks, got %d", kMaxRanks, x.f.ar.world);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

}  // namespace mgw
