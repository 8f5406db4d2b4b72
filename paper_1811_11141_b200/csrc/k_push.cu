// k_push.cu -- host launchers of the push.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "push.cuh"

namespace mgw {

int plan_push1(PushArgs& x, int max_ctas, const int64_t* per_cta) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  const int grid = collective_grid_rt(x.f.ar.world, x.f.ar.n >> 2, per_cta ? per_cta[0] : 0, max_ctas);
  x.f.ar.tag = collective_tag(x.f.ar.tag, x.f.ar.n, kTagPushOneshot, grid, x.f.scale);
  return grid;
}

int plan_push(PushArgs& x, int max_ctas, const int64_t* per_cta) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  const int w = x.f.ar.world > 0 ? x.f.ar.world : 1;
  const int64_t nv = x.f.ar.n >> 2;
  int64_t per = per_cta ? per_cta[1] : 0;
  if (per <= 0) {
    // large buckets stream better in long per-CTA chunks: 2048-4096 slots (32-64 KB per
    // part) per CTA, spread over one CTA per SM (profiles/grid_pushtune_n4_r01.json:
    // 32 MB 105 -> 98 us, 64 MB 195 -> 180 us at N = 4)
    per = (nv / w + kSMs - 1) / kSMs;
    per = (per + 127) / 128 * 128;
    per = per < 2048 ? 2048 : (per > 4096 ? 4096 : per);
  }
  const int grid = grid_for(nv / w, per, max_ctas);
  x.f.ar.tag = collective_tag(x.f.ar.tag, x.f.ar.n, kTagPush, grid, x.f.scale);
  return grid;
}

template <int N>
static int launch_push_n(const PushArgs& x, bool one, int grid, cudaStream_t stream) {
  if (one)
    push_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  else
    push_twoshot_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

static int launch_push_any(const PushArgs& x0, bool one, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  PushArgs x = x0;
  const int grid = one ? plan_push1(x, max_ctas, per_cta) : plan_push(x, max_ctas, per_cta);
  switch (x.f.ar.world) {
    case 2: return launch_push_n<2>(x, one, grid, stream);
    case 3: return launch_push_n<3>(x, one, grid, stream);
    case 4: return launch_push_n<4>(x, one, grid, stream);
    case 5: return launch_push_n<5>(x, one, grid, stream);
    case 6: return launch_push_n<6>(x, one, grid, stream);
    case 7: return launch_push_n<7>(x, one, grid, stream);
    case 8: return launch_push_n<8>(x, one, grid, stream);
    default:
      return set_error(MGW_EINVAL, "push %s needs 2..%d ranks, got %d", one ? "one-shot" : "two-shot", kMaxRanks,
                       x.f.ar.world);
  }
}

int launch_push1(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  return launch_push_any(x, true, max_ctas, stream, per_cta);
}

int launch_push(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  return launch_push_any(x, false, max_ctas, stream, per_cta);
}

template <int N>
static int group_push_n(const RankGroup<PushArgs>& g, bool one, cudaStream_t stream) {
  return one ? launch_cooperative(push_oneshot_group<N>, g, stream) : launch_cooperative(push_twoshot_group<N>, g, stream);
}

int launch_push_group(const RankGroup<PushArgs>& g, int world, bool one, cudaStream_t stream) {
  switch (world) {
    case 2: return group_push_n<2>(g, one, stream);
    case 3: return group_push_n<3>(g, one, stream);
    case 4: return group_push_n<4>(g, one, stream);
    case 5: return group_push_n<5>(g, one, stream);
    case 6: return group_push_n<6>(g, one, stream);
    case 7: return group_push_n<7>(g, one, stream);
    case 8: return group_push_n<8>(g, one, stream);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

MGW_DEFINE_VIOLATIONS(push)

}  // namespace mgw
