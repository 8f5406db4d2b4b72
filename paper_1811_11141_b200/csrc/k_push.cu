// k_push.cu -- host launchers of the push.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "pipe.cuh"

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

// the pipelined two-shot: the push two-shot's grid, S sub-chunks of >= one slot per thread
// per part (at most kPipeSub) -- S follows from n and the grid, so every rank agrees
static int64_t g_pipe_sub_slots = kThreads;  // slots per sub-chunk per part (mgw_set_option)

int set_pipe_sub_slots(int64_t v) {
  if (v < 32 || v > (1 << 20)) return set_error(MGW_EINVAL, "pipe sub-chunk slots must lie in 32..2^20");
  g_pipe_sub_slots = v;
  return MGW_OK;
}

int plan_push_pipe(PushArgs& x, int max_ctas, const int64_t* per_cta) {
  const uint32_t user_tag = x.f.ar.tag;
  const int grid = plan_push(x, max_ctas, per_cta);
  const int w = x.f.ar.world > 0 ? x.f.ar.world : 1;
  const int64_t chunk = ((x.f.ar.n >> 2) / w + grid - 1) / grid;  // slots per CTA per part
  int64_t subs = chunk / g_pipe_sub_slots;
  x.subs = (int)(subs < 1 ? 1 : (subs > kPipeSub ? kPipeSub : subs));
  x.f.ar.tag = collective_tag(user_tag, x.f.ar.n, kTagPushPipe, grid * 16 + x.subs, x.f.scale);
  return grid;
}

// kind: 0 two-shot, 1 one-shot, 2 pipelined two-shot
template <int N>
static int launch_push_n(const PushArgs& x, int kind, int grid, cudaStream_t stream) {
  if (kind == 1)
    push_oneshot_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  else if (kind == 2)
    push_pipe_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  else
    push_twoshot_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

static int launch_push_any(const PushArgs& x0, int kind, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  PushArgs x = x0;
  const int grid = kind == 1 ? plan_push1(x, max_ctas, per_cta)
                             : (kind == 2 ? plan_push_pipe(x, max_ctas, per_cta) : plan_push(x, max_ctas, per_cta));
  switch (x.f.ar.world) {
    case 2: return launch_push_n<2>(x, kind, grid, stream);
    case 3: return launch_push_n<3>(x, kind, grid, stream);
    case 4: return launch_push_n<4>(x, kind, grid, stream);
    case 5: return launch_push_n<5>(x, kind, grid, stream);
    case 6: return launch_push_n<6>(x, kind, grid, stream);
    case 7: return launch_push_n<7>(x, kind, grid, stream);
    case 8: return launch_push_n<8>(x, kind, grid, stream);
    default: return set_error(MGW_EINVAL, "push exchanges need 2..%d ranks, got %d", kMaxRanks, x.f.ar.world);
  }
}

int launch_push1(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  return launch_push_any(x, 1, max_ctas, stream, per_cta);
}

int launch_push(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  return launch_push_any(x, 0, max_ctas, stream, per_cta);
}

int launch_push_pipe(const PushArgs& x, int max_ctas, cudaStream_t stream, const int64_t* per_cta) {
  return launch_push_any(x, 2, max_ctas, stream, per_cta);
}

template <int N>
static int group_push_n(const RankGroup<PushArgs>& g, int kind, cudaStream_t stream) {
  if (kind == 1) return launch_cooperative(push_oneshot_group<N>, g, stream);
  if (kind == 2) return launch_cooperative(push_pipe_group<N>, g, stream);
  return launch_cooperative(push_twoshot_group<N>, g, stream);
}

int launch_push_group(const RankGroup<PushArgs>& g, int world, int kind, cudaStream_t stream) {
  switch (world) {
    case 2: return group_push_n<2>(g, kind, stream);
    case 3: return group_push_n<3>(g, kind, stream);
    case 4: return group_push_n<4>(g, kind, stream);
    case 5: return group_push_n<5>(g, kind, stream);
    case 6: return group_push_n<6>(g, kind, stream);
    case 7: return group_push_n<7>(g, kind, stream);
    case 8: return group_push_n<8>(g, kind, stream);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

MGW_DEFINE_VIOLATIONS(push)

}  // namespace mgw
