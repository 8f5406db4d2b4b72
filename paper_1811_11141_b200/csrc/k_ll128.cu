// k_ll128.cu -- host launchers of the ll128.cuh kernels (own translation unit: the kernel
// families compile in parallel, see __graft_entry__.build).
#include "launch.h"
#include "ll128.cuh"

namespace mgw {

// lines per CTA: at least one full CTA step (64 lines = 7.5 KB of payload per part), grid
// up to the CTA cap.  Two-shot: lines of one part; one-shot: lines of the whole bucket.
int plan_ll128(L128Args& x, int max_ctas, const int64_t* per_cta, bool b16, bool one) {
  max_ctas = max_ctas < kMaxBlocks ? max_ctas : kMaxBlocks;
  const int w = x.f.ar.world > 0 ? x.f.ar.world : 1;
  const int64_t slots = l128_slots(x.f.ar.n, b16);
  const int64_t lines = l128_lines(one ? slots : slots / w);
  const int64_t per = per_cta && per_cta[1] > 0 ? (per_cta[1] + kL128Vec - 1) / kL128Vec : kL128Step;
  const int grid = grid_for(lines, per, max_ctas);
  x.row_lines = l128_row_lines(x.f.ar.n, w, b16, one);
  const uint32_t kind = one ? (b16 ? kTagB16LL128One : kTagLL128One) : (b16 ? kTagB16LL128 : kTagLL128);
  x.f.ar.tag = collective_tag(x.f.ar.tag, x.f.ar.n, kind, grid, x.f.scale);
  return grid;
}

template <int N>
static int launch_ll128_n(const L128Args& x, int grid, cudaStream_t stream, bool b16, bool one) {
  if (one) {
    if (b16)
      b16_ll128_one_kernel<N><<<grid, kThreads, 0, stream>>>(x);
    else
      ll128_one_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  } else {
    if (b16)
      b16_ll128_kernel<N><<<grid, kThreads, 0, stream>>>(x);
    else
      ll128_kernel<N><<<grid, kThreads, 0, stream>>>(x);
  }
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int launch_ll128(const L128Args& x0, int max_ctas, cudaStream_t stream, const int64_t* per_cta, bool b16, bool one) {
  L128Args x = x0;
  const int grid = plan_ll128(x, max_ctas, per_cta, b16, one);
  switch (x.f.ar.world) {
    case 2: return launch_ll128_n<2>(x, grid, stream, b16, one);
    case 3: return launch_ll128_n<3>(x, grid, stream, b16, one);
    case 4: return launch_ll128_n<4>(x, grid, stream, b16, one);
    case 5: return launch_ll128_n<5>(x, grid, stream, b16, one);
    case 6: return launch_ll128_n<6>(x, grid, stream, b16, one);
    case 7: return launch_ll128_n<7>(x, grid, stream, b16, one);
    case 8: return launch_ll128_n<8>(x, grid, stream, b16, one);
    default: return set_error(MGW_EINVAL, "LL128 path needs 2..%d ranks, got %d", kMaxRanks, x.f.ar.world);
  }
}

template <int N>
static int launch_ll128_group_n(const RankGroup<L128Args>& g, cudaStream_t stream, bool b16, bool one) {
  if (one) return b16 ? launch_cooperative(b16_ll128_one_group<N>, g, stream) : launch_cooperative(ll128_one_group<N>, g, stream);
  return b16 ? launch_cooperative(b16_ll128_group<N>, g, stream) : launch_cooperative(ll128_group<N>, g, stream);
}

int launch_ll128_group(const RankGroup<L128Args>& g, int world, cudaStream_t stream, bool b16, bool one) {
  switch (world) {
    case 2: return launch_ll128_group_n<2>(g, stream, b16, one);
    case 3: return launch_ll128_group_n<3>(g, stream, b16, one);
    case 4: return launch_ll128_group_n<4>(g, stream, b16, one);
    case 5: return launch_ll128_group_n<5>(g, stream, b16, one);
    case 6: return launch_ll128_group_n<6>(g, stream, b16, one);
    case 7: return launch_ll128_group_n<7>(g, stream, b16, one);
    case 8: return launch_ll128_group_n<8>(g, stream, b16, one);
    default: return set_error(MGW_EINVAL, "rank group of %d outside 2..%d", world, kMaxRanks);
  }
}

MGW_DEFINE_VIOLATIONS(ll128)

}  // namespace mgw
