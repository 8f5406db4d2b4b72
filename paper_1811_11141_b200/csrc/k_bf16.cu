// k_bf16.cu -- host launchers of the bf16.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "b16push.cuh"

namespace mgw {

int plan_ll_b16(LLArgs& l, int max_ctas) {
  const int64_t quads = (l.f.ar.n + 3) >> 2;
  const int grid = grid_for(quads, kThreads, max_ctas < kSMs ? max_ctas : kSMs);
  l.f.ar.tag = collective_tag(l.f.ar.tag, l.f.ar.n, kTagB16LL, grid, l.f.scale);
  return grid;
}

int launch_ll_b16(const LLArgs& l0, int max_ctas, cudaStream_t stream) {
  if (l0.f.ar.n > 2 * kLLMaxElems)
    return set_error(MGW_EINVAL, "bf16 LL path takes at most %lld elements", (long long)(2 * kLLMaxElems));
  LLArgs l = l0;
  const int grid = plan_ll_b16(l, max_ctas);
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

int plan_b16(FusedArgs& f, int algo, int max_ctas) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  const int w = f.ar.world > 0 ? f.ar.world : 1;
  const int64_t nv = f.ar.n / kB16;
  const bool one = algo == MGW_ALGO_ONESHOT;
  const int grid = one ? collective_grid_rt(w, nv, 0, max_ctas) : collective_grid_rt(w, nv / w, 0, max_ctas);
  f.ar.tag = collective_tag(f.ar.tag, f.ar.n, one ? kTagB16Oneshot : kTagB16Twoshot, grid, f.scale);
  return grid;
}

template <int N>
static int launch_b16_n(const FusedArgs& f, int algo, int grid, cudaStream_t stream) {
  if (algo == MGW_ALGO_ONESHOT)
    b16_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  else
    b16_twoshot_kernel<N><<<grid, kThreads, 0, stream>>>(f);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_b16(const FusedArgs& f0, int algo, int max_ctas, cudaStream_t stream) {
  if (algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT)
    return set_error(MGW_EINVAL, "bf16 buckets support one-shot and two-shot only (algorithm %d)", algo);
  FusedArgs f = f0;
  const int grid = plan_b16(f, algo, max_ctas);
  switch (f.ar.world) {
    case 1: return launch_b16_n<1>(f, algo, grid, stream);
    case 2: return launch_b16_n<2>(f, algo, grid, stream);
    case 3: return launch_b16_n<3>(f, algo, grid, stream);
    case 4: return launch_b16_n<4>(f, algo, grid, stream);
    case 5: return launch_b16_n<5>(f, algo, grid, stream);
    case 6: return launch_b16_n<6>(f, algo, grid, stream);
    case 7: return launch_b16_n<7>(f, algo, grid, stream);
    case 8: return launch_b16_n<8>(f, algo, grid, stream);
    default: return set_error(MGW_EINVAL, "world %d outside 1..%d", f.ar.world, kMaxRanks);
  }
}

template <int N>
static int group_b16_n(const RankGroup<FusedArgs>& g, int algo, cudaStream_t stream) {
  return algo == MGW_ALGO_ONESHOT ? launch_cooperative(b16_oneshot_group<N>, g, stream)
                                  : launch_cooperative(b16_twoshot_group<N>, g, stream);
}

int launch_b16_group(const RankGroup<FusedArgs>& g, int world, int algo, cudaStream_t stream) {
  switch (world) {
    case 2: return group_b16_n<2>(g, algo, stream);
    case 3: return group_b16_n<3>(g, algo, stream);
    case 4: return group_b16_n<4>(g, algo, stream);
    case 5: return group_b16_n<5>(g, algo, stream);
    case 6: return group_b16_n<6>(g, algo, stream);
    case 7: return group_b16_n<7>(g, algo, stream);
    case 8: return group_b16_n<8>(g, algo, stream);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

// bf16 push two-shot: the push two-shot's grid rule in bf16 16-B slots
int plan_b16_push(PushArgs& x, int max_ctas) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  const int w = x.f.ar.world > 0 ? x.f.ar.world : 1;
  const int64_t nv = x.f.ar.n / kB16;
  int64_t per = (nv / w + kSMs - 1) / kSMs;
  per = (per + 127) / 128 * 128;
  per = per < 2048 ? 2048 : (per > 4096 ? 4096 : per);
  const int grid = grid_for(nv / w, per, max_ctas);
  x.f.ar.tag = collective_tag(x.f.ar.tag, x.f.ar.n, kTagB16Push, grid, x.f.scale);
  return grid;
}

int launch_b16_push(const PushArgs& x0, int max_ctas, cudaStream_t stream) {
  PushArgs x = x0;
  const int grid = plan_b16_push(x, max_ctas);
  switch (x.f.ar.world) {
    case 2: b16_push_kernel<2><<<grid, kThreads, 0, stream>>>(x); break;
    case 3: b16_push_kernel<3><<<grid, kThreads, 0, stream>>>(x); break;
    case 4: b16_push_kernel<4><<<grid, kThreads, 0, stream>>>(x); break;
    case 5: b16_push_kernel<5><<<grid, kThreads, 0, stream>>>(x); break;
    case 6: b16_push_kernel<6><<<grid, kThreads, 0, stream>>>(x); break;
    case 7: b16_push_kernel<7><<<grid, kThreads, 0, stream>>>(x); break;
    case 8: b16_push_kernel<8><<<grid, kThreads, 0, stream>>>(x); break;
    default: return set_error(MGW_EINVAL, "bf16 push two-shot needs 2..%d ranks, got %d", kMaxRanks, x.f.ar.world);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_b16_push_group(const RankGroup<PushArgs>& g, int world, cudaStream_t stream) {
  switch (world) {
    case 2: return launch_cooperative(b16_push_group<2>, g, stream);
    case 3: return launch_cooperative(b16_push_group<3>, g, stream);
    case 4: return launch_cooperative(b16_push_group<4>, g, stream);
    case 5: return launch_cooperative(b16_push_group<5>, g, stream);
    case 6: return launch_cooperative(b16_push_group<6>, g, stream);
    case 7: return launch_cooperative(b16_push_group<7>, g, stream);
    case 8: return launch_cooperative(b16_push_group<8>, g, stream);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

int launch_ll_b16_group(const RankGroup<LLArgs>& g, int world, cudaStream_t stream) {
  switch (world) {
    case 2: return launch_cooperative(ll_b16_group<2>, g, stream);
    case 3: return launch_cooperative(ll_b16_group<3>, g, stream);
    case 4: return launch_cooperative(ll_b16_group<4>, g, stream);
    case 5: return launch_cooperative(ll_b16_group<5>, g, stream);
    case 6: return launch_cooperative(ll_b16_group<6>, g, stream);
    case 7: return launch_cooperative(ll_b16_group<7>, g, stream);
    case 8: return launch_cooperative(ll_b16_group<8>, g, stream);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

MGW_DEFINE_VIOLATIONS(bf16)

}  // namespace mgw
