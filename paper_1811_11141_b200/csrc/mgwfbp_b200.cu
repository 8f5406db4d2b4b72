// mgwfbp_b200.cu -- C ABI of the MG-WFBP merged-gradient data path (sm_100a).
//
//   K1 pack+scale   gather a merge group's layer gradients into one contiguous
//                   bucket (layer `high` at offset 0; allreduce_net.py:495-509)  rows.cuh
//   K2 one-shot     every rank pulls all N peer buckets over NVLink (CUDA IPC)
//                   and folds them in the reference ring's per-element order    allreduce.cuh
//   K3 two-shot     reduce-scatter of an aligned 1/N part, then all-gather of
//                   the peers' reduced parts, same per-element fold order        allreduce.cuh
//   K4 unpack       scatter the reduced bucket back to the layer tensors         rows.cuh
//   K5 spin         simulated backward on the compute stream (%globaltimer)      below
//
// Host side: the communicator (IPC buckets, flags, peer mappings), descriptor
// tables, the Algorithm-2 schedule engine (streams, events, CUDA graph) and the
// timing helpers.  Every entry point returns MGW_* status codes.

#include "mgwfbp_b200.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_bf16.h>

#include "allreduce.cuh"
#include "bf16.cuh"
#include "launch.h"
#include "common.cuh"
#include "fused.cuh"
#include "ll.cuh"
#include "nvls.cuh"
#include "push.cuh"
#include "rows.cuh"

using namespace mgw;

namespace {

// ============================================================ K5: spin kernels

__global__ void spin_relative_kernel(int64_t ns) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = global_ns();
  while ((int64_t)(global_ns() - t0) < ns) __nanosleep(128);
}

__global__ void stamps_reset_kernel(uint64_t* stamps, int pairs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += gridDim.x * blockDim.x) {
    stamps[2 * i] = ~0ull;
    stamps[2 * i + 1] = 0ull;
  }
}

__global__ void clock_mark_kernel(uint64_t* clock) {
  if (threadIdx.x == 0) *clock = global_ns();
}

// advances the device call counter by one (timing of the gate alone, kind 6)
__global__ void finish_kernel(uint32_t* state) {
  if (threadIdx.x == 0) state[0] += 1u;
}

// bf16 gradient "production" of the engine (MGW_SCHED_BF16): row k of the group gets
// values[k] (the reference pattern rank + 1 + layer % 5, exact in bf16)
__global__ void fill_b16_kernel(const Row* rows, int n_rows, const float* values, uint64_t* stamp) {
  stamp_enter(stamp);
  for (int k = 0; k < n_rows; ++k) {
    uint16_t* p = reinterpret_cast<uint16_t*>(rows[k].ptr);
    const uint16_t v = __bfloat16_as_ushort(__float2bfloat16_rn(values[k]));
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows[k].count; e += (int64_t)gridDim.x * blockDim.x)
      p[e] = v;
  }
  stamp_exit(stamp);
}

__global__ void spin_until_kernel(const uint64_t* clock, int64_t deadline_ns) {
  if (threadIdx.x != 0) return;
  const uint64_t until = *reinterpret_cast<const volatile uint64_t*>(clock) + (uint64_t)deadline_ns;
  while (global_ns() < until) __nanosleep(128);
}

}  // namespace

// =================================================================== C ABI

// Descriptor table handle: device rows plus a host mirror (the host copy feeds the
// kernels' inline parameters).  Rows tile [0, extent) contiguously in order.
struct mgw_table_t {
  Row* dev = nullptr;
  std::vector<Row> host;
  int64_t extent = 0;
};

struct mgw_comm {
  int rank = 0;
  int world = 1;
  int device = 0;
  int64_t capacity = 0;    // bytes per slot as requested
  int64_t slot_bytes = 0;  // rounded to 256 B
  char* region = nullptr;  // own IPC region
  char* peer[kMaxRanks] = {};
  bool peers_open = false;
  uint32_t* state = nullptr;  // [calls, finished]
  int* err = nullptr;
  float* result = nullptr;
  uint64_t timeout_ns = 30ull * 1000000000ull;
  int64_t oneshot_max_bytes = 1 << 20;  // set per world in mgw_comm_create
  int64_t ll_max_bytes = 256 << 10;  // AUTO's LL ceiling (the area holds kLLElems per source)
  int max_ctas = 2 * kSMs;  // one resident wave (a 512 cap helped N=4 / 128 MB but not N=2 / 102 MB)
  int64_t vec_per_cta[2] = {0, 0};      // tuning: 16-B slots per CTA (one-shot, two-shot); 0 = default
  // NVLS (opt-in): multicast object bound to a per-rank bucket
  CUmemGenericAllocationHandle nvls_mc = 0, nvls_mem = 0;
  CUdeviceptr nvls_uc = 0, nvls_mcva = 0;
  size_t nvls_bytes = 0;
  bool nvls_mc_valid = false, nvls_bound = false;
  int64_t nvls_min_bytes = 0;  // AUTO picks NVLS at >= this size when set (0 = never)
  bool gate = false;           // launch gate_kernel ahead of every collective (mgw_comm_set_gate)
  uint32_t group_tag = 0;      // caller's group tag, folded into every collective's tag
  bool local_group = false;    // in-process rank group on one device (mgw_comm_create_local)
};

constexpr int kSchedStamps = 8;  // per group: [pack][all-reduce / fused][unpack][fill] x [start, end]

struct mgw_sched {
  mgw_comm* comm = nullptr;
  int world = 1;
  std::vector<Row> rows;
  Row* d_rows = nullptr;
  std::vector<mgw_group> groups;
  float* d_fill = nullptr;
  float* local_bucket = nullptr;  // single-rank bucket
  uint64_t* d_clock = nullptr;
  uint64_t* d_stamps = nullptr;   // per group: pack, all-reduce / fused, unpack, fill spans (4 x [start, end])
  std::vector<uint64_t> h_stamps;
  float scale = 1.f;
  uint32_t flags = 0;
  std::vector<float*> host_src, host_dst;
  // dependency events (fork/join) and the three timing events of an iteration
  cudaEvent_t dep_fork = nullptr, dep_join = nullptr, dep_compute = nullptr;
  std::vector<cudaEvent_t> dep_ready;
  cudaEvent_t t_start = nullptr, t_compute = nullptr, t_end = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaGraph_t graph = nullptr;
  int launches = 0;
  bool capturing = false;
};

namespace {

ArArgs make_args(const mgw_comm* c, int64_t n) {
  ArArgs a;
  memset(&a, 0, sizeof(a));
  for (int s = 0; s < c->world; ++s) {
    char* base = c->peer[s];
    a.slot[s] = base + kSlotOff;
    a.arrive[s] = reinterpret_cast<uint64_t*>(base + kArriveOff);
    a.mid[s] = reinterpret_cast<uint64_t*>(base + kMidOff);
    a.abort_flag[s] = reinterpret_cast<uint32_t*>(base + kAbortOff);
  }
  a.out[c->rank] = c->result;
  a.state = c->state;
  a.err = c->err;
  a.slot_stride = c->slot_bytes;
  a.n = n;
  a.timeout_ns = c->timeout_ns;
  a.rank = c->rank;
  a.world = c->world;
  a.tag = c->group_tag;
  return a;
}

// One rank per device (IPC): wait for the device.  In-process rank group: the caller has
// synchronised its own stream -- a device-wide sync would wait on peers' kernels that wait
// on this rank's next collective.
int sync_for_query(const mgw_comm* c) {
  MGW_CUDA(cudaSetDevice(c->device));
  if (!c->local_group) MGW_CUDA(cudaDeviceSynchronize());
  return MGW_OK;
}

int comm_launch_allreduce(const mgw_comm* c, const ArArgs& a, int algo, cudaStream_t stream) {
  return launch_allreduce(a, algo, c->max_ctas, stream, c->vec_per_cta);
}

// ------------------------------------------------------------- NVLS plumbing
// Driver entry points through the runtime (no link-time dependency on libcuda).
struct DriverFns {
  PFN_cuMulticastCreate mc_create = nullptr;
  PFN_cuMulticastAddDevice mc_add = nullptr;
  PFN_cuMulticastBindMem mc_bind = nullptr;
  PFN_cuMulticastUnbind mc_unbind = nullptr;
  PFN_cuMulticastGetGranularity mc_gran = nullptr;
  PFN_cuMemCreate mem_create = nullptr;
  PFN_cuMemRelease mem_release = nullptr;
  PFN_cuMemAddressReserve addr_reserve = nullptr;
  PFN_cuMemAddressFree addr_free = nullptr;
  PFN_cuMemMap mem_map = nullptr;
  PFN_cuMemUnmap mem_unmap = nullptr;
  PFN_cuMemSetAccess set_access = nullptr;
  PFN_cuMemExportToShareableHandle export_handle = nullptr;
  PFN_cuMemImportFromShareableHandle import_handle = nullptr;
  PFN_cuDeviceGetAttribute get_attr = nullptr;
  bool ok = false;
};

const DriverFns& driver() {
  static DriverFns fns = [] {
    DriverFns d;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess;
    };
    d.ok = get("cuMulticastCreate", (void**)&d.mc_create) && get("cuMulticastAddDevice", (void**)&d.mc_add) &&
           get("cuMulticastBindMem", (void**)&d.mc_bind) && get("cuMulticastUnbind", (void**)&d.mc_unbind) &&
           get("cuMulticastGetGranularity", (void**)&d.mc_gran) && get("cuMemCreate", (void**)&d.mem_create) &&
           get("cuMemRelease", (void**)&d.mem_release) && get("cuMemAddressReserve", (void**)&d.addr_reserve) &&
           get("cuMemAddressFree", (void**)&d.addr_free) && get("cuMemMap", (void**)&d.mem_map) &&
           get("cuMemUnmap", (void**)&d.mem_unmap) && get("cuMemSetAccess", (void**)&d.set_access) &&
           get("cuMemExportToShareableHandle", (void**)&d.export_handle) &&
           get("cuMemImportFromShareableHandle", (void**)&d.import_handle) &&
           get("cuDeviceGetAttribute", (void**)&d.get_attr);
    return d;
  }();
  return fns;
}

#define MGW_CU(call)                                                                                \
  do {                                                                                              \
    CUresult r_ = (call);                                                                           \
    if (r_ != CUDA_SUCCESS) return set_error(MGW_ECUDA, "%s failed: CUresult %d", #call, (int)r_); \
  } while (0)

size_t nvls_granularity(int world) {
  CUmulticastObjectProp p = {};
  p.numDevices = (unsigned)world;
  p.size = 2ull << 20;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  if (driver().mc_gran(&g, &p, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0) g = 2ull << 20;
  return g;
}

int pick_algo(const mgw_comm* c, int64_t n, int algo) {
  if (algo != MGW_ALGO_AUTO) return algo;
  return n * 4 <= c->oneshot_max_bytes ? MGW_ALGO_ONESHOT : MGW_ALGO_TWOSHOT;
}

// fused group exchange: LL push for small buckets, else pull one-shot / two-shot;
// NVLS only when enabled (not bit-exact with the reference order)
constexpr int64_t kLL128MinBytes = 1ll << 20;  // AUTO: LL128 from here (before LL's ceiling)
inline int64_t ll128_max_bytes(const mgw_comm* c) {
  return c->world == 2 ? (128ll << 20) : (c->world <= 4 ? (64ll << 20) : (16ll << 20));
}
// AUTO's LL128 choice for a bucket of `bytes` (fp32 or bf16 alike), 0 = neither: the
// one-shot (one hop, (N-1) x M x 16/15 out) for mid-size buckets, the two-shot (in rounds)
// above, the push two-shot beyond (profiles/ll128_rounds_r02.json, graph-timed bus
// GB/s, N=4: 1 MiB one-shot 140 vs two-shot 134, 2 MiB two-shot 235 vs 195, 16 MiB 505 vs
// push 431, 64 MiB 578 vs 557, 128 MiB 585 vs the wide push 590; N=2: one-shot to 16 MiB,
// two-shot to 128 MiB).  N > 4: unmeasured here, so only the two-shot, to 16 MiB.
inline int ll128_pick(const mgw_comm* c, int64_t bytes) {
  if (c->world == 2 && bytes >= (512ll << 10) && bytes <= (16ll << 20)) return MGW_ALGO_LL128_ONESHOT;
  if (c->world > 2 && c->world <= 4 && bytes >= (256ll << 10) && bytes <= kLL128MinBytes) return MGW_ALGO_LL128_ONESHOT;
  if (bytes >= kLL128MinBytes && bytes <= ll128_max_bytes(c)) return MGW_ALGO_LL128;
  return 0;
}

int pick_fused_algo(const mgw_comm* c, int64_t n, int algo) {
  if (algo != MGW_ALGO_AUTO) return algo;
  if (c->nvls_bound && c->nvls_min_bytes > 0 && n * 4 >= c->nvls_min_bytes && (size_t)n * 4 <= c->nvls_bytes)
    return MGW_ALGO_NVLS;
  // engine-mode sweeps (profiles/grid_{push,large,push1}_n*_r01.json): at N = 2 the push
  // one-shot wins up to 16 MB and the push two-shot above; at N >= 3 the push one-shot up
  // to 512 KB, the pull one-shot to 8 MB / (N - 1), the pull two-shot to 8 MB and the
  // push two-shot above (546 vs 509 GB/s bus at N = 4, 128 MB)
  // Beyond ~1 GB the push two-shot falls behind the pull two-shot again (synthetic
  // 1000-layer SyncEASGD bucket, 6.75 GB: 42.4 vs 20.8 ms at N = 4; VGG-16's 553 MB still
  // favours push, profiles/profiles_n4_r01_final.json).
  const int64_t bytes = n * 4;
  // the flag-in-line two-shot (ll128.cuh) from 1 MiB: no barriers, 2 (N-1)/N x M x 16/15 out
  // (profiles/ll128_sweep_n{2,4}_r02.json, graph-timed at N = 4: 1 MiB 11.8 vs 15.4 us,
  // 4 MiB 18.2 vs 27.9, 16 MiB 56.3 vs 58.5; level with the push two-shot at 32 MiB,
  // which stays above 16 MiB; at N = 2 it wins to 32 MiB, and from 1 MiB over the LL one-shot)
  if (c->world > 1) {
    const int l128 = ll128_pick(c, bytes);
    if (l128) return l128;
  }
  if (c->world > 1 && n * 4 <= c->ll_max_bytes && n <= kLLElems) return MGW_ALGO_LL;
  const bool push_ok = bytes <= (1ll << 30);
  if (c->world == 2)
    return bytes <= (16ll << 20) ? MGW_ALGO_PUSH_ONESHOT : (push_ok ? MGW_ALGO_PUSH : MGW_ALGO_TWOSHOT);
  if (bytes <= (512ll << 10)) return MGW_ALGO_PUSH_ONESHOT;
  if (bytes <= c->oneshot_max_bytes) return MGW_ALGO_ONESHOT;
  return bytes >= (8ll << 20) && push_ok ? MGW_ALGO_PUSH : MGW_ALGO_TWOSHOT;
}

// The kernel a fused fp32 group exchange of n elements actually runs: the AUTO choice,
// then the fallbacks when the push areas cannot hold the incoming rows.
constexpr int64_t kB16PushMinBytes = 8ll << 20;  // bf16 AUTO: push two-shot at >= 8 MB (as fp32 at N >= 3)

int resolve_fused_algo(const mgw_comm* c, int64_t n, int algo) {
  int chosen = pick_fused_algo(c, n, algo);
  if (chosen == MGW_ALGO_LL128_ONESHOT &&
      (c->world == 1 || c->world * l128_row_lines(n, c->world, false, true) * 128 > c->slot_bytes))
    chosen = MGW_ALGO_LL128;  // one rank, or the whole-bucket lines do not fit one slot
  if (chosen == MGW_ALGO_LL128 && (c->world == 1 || c->world * l128_row_lines(n, c->world, false) * 128 > c->slot_bytes))
    chosen = MGW_ALGO_PUSH;  // one rank, or the lines do not fit one slot
  if (chosen == MGW_ALGO_PUSH_ONESHOT && c->world * round_up(n, 16) * 4 > c->slot_bytes) chosen = MGW_ALGO_ONESHOT;
  if ((chosen == MGW_ALGO_PUSH || chosen == MGW_ALGO_PUSH_PIPE) &&
      c->world * push_stride(n / 4, c->world) * 4 > c->slot_bytes)
    chosen = MGW_ALGO_TWOSHOT;
  return chosen;
}

// bf16 group exchange: LL for small buckets, else pull one-shot / two-shot
int resolve_b16_algo(const mgw_comm* c, int64_t n, int algo) {
  if (algo == MGW_ALGO_AUTO) {
    // bf16 crossovers as fp32 in bytes (profiles/ll128_bf16_sweep_n{2,4}_r02.json): LL128
    // one-/two-shot (ll128_pick), LL below, push two-shot above
    const int l128 = c->world > 1 ? ll128_pick(c, n * 2) : 0;
    if (l128)
      algo = l128;
    else if (c->world > 1 && n * 2 <= c->ll_max_bytes && n <= 2 * kLLElems)
      algo = MGW_ALGO_LL;
    else if (n * 2 <= c->oneshot_max_bytes)
      algo = MGW_ALGO_ONESHOT;
    else  // large bf16 buckets: the store-only push two-shot (b16push.cuh), as for fp32
      algo = c->world > 1 && n * 2 >= kB16PushMinBytes ? MGW_ALGO_PUSH : MGW_ALGO_TWOSHOT;
  }
  if (algo == MGW_ALGO_LL && c->world == 1) algo = MGW_ALGO_ONESHOT;
  if (algo == MGW_ALGO_LL128_ONESHOT &&
      (c->world == 1 || c->world * l128_row_lines(n, c->world, true, true) * 128 > c->slot_bytes))
    algo = MGW_ALGO_LL128;
  if (algo == MGW_ALGO_LL128 && (c->world == 1 || c->world * l128_row_lines(n, c->world, true) * 128 > c->slot_bytes))
    algo = MGW_ALGO_PUSH;  // one rank, or the lines do not fit one slot
  if (algo == MGW_ALGO_PUSH && (c->world == 1 || c->world * b16_push_stride(n, c->world) * 2 > c->slot_bytes))
    algo = MGW_ALGO_TWOSHOT;  // one rank, or the incoming rows do not fit the slot
  return algo;
}

int comm_allreduce(mgw_comm* c, int64_t n, int algo, cudaStream_t stream, uint64_t* stamp = nullptr,
                   int64_t group_tag = -1) {
  if (n < 0 || n * 4 > c->slot_bytes)
    return set_error(MGW_EINVAL, "bucket of %lld elements exceeds slot capacity %lld B", (long long)n,
                     (long long)c->slot_bytes);
  if (c->world == 1) {
    if (n > 0) MGW_CUDA(cudaMemcpyAsync(c->result, c->region + kSlotOff, n * 4, cudaMemcpyDeviceToDevice, stream));
    return MGW_OK;
  }
  if (!c->peers_open) return set_error(MGW_EINVAL, "peers not opened (call mgw_comm_open_peers)");
  ArArgs a = make_args(c, n);
  if (group_tag >= 0) a.tag = (uint32_t)group_tag;
  if (c->gate) {
    int rc = launch_gate(a, stream);
    if (rc) return rc;
  }
  a.stamp = stamp;
  return comm_launch_allreduce(c, a, pick_algo(c, n, algo), stream);
}

int comm_pack(mgw_comm* c, const Row* host_rows, const Row* dev_rows, int n_rows, int64_t n, float scale,
              cudaStream_t stream, uint64_t* stamp = nullptr) {
  if (n * 4 > c->slot_bytes)
    return set_error(MGW_EINVAL, "bucket of %lld elements exceeds slot capacity %lld B", (long long)n,
                     (long long)c->slot_bytes);
  float* slot0 = reinterpret_cast<float*>(c->region + kSlotOff);
  const uint32_t* calls = c->world > 1 ? c->state : nullptr;
  return launch_rows<RowOp::kPack>(host_rows, dev_rows, n_rows, slot0, n, scale, nullptr, calls, c->slot_bytes / 4,
                                   nullptr, stream, stamp);
}

// CTA cap of the push two-shot over IPC: buckets >= g_wide_min_bytes take kMaxBlocks CTAs
// (a second, partial wave) -- the 4096-slot chunks keep streaming while the first wave's
// CTAs sit in their barriers (profiles/cta_cap_n{2,4}_r02.json: 128 MiB at N = 4 546 -> 592
// bus GB/s, 256 MiB 559 -> 609; neutral at <= 64 MiB).  Forward progress: CTAs dispatch in
// index order, so the lowest unfinished CTA index is resident on every rank.  Not for the
// cooperative single-device groups (every CTA must be co-resident there).
int64_t g_wide_min_bytes = 112ll << 20;  // mgw_set_option(MGW_OPT_WIDE_MIN_BYTES); 0 = off

static int push_cap(const mgw_comm* c, int64_t bytes) {
  if (g_wide_min_bytes > 0 && bytes >= g_wide_min_bytes && !c->local_group)
    return c->max_ctas > kMaxBlocks ? c->max_ctas : kMaxBlocks;
  return c->max_ctas;
}

// pack -> all-reduce -> unpack of one group in a single kernel (fused.cuh)
int comm_allreduce_fused(mgw_comm* c, const Row* host_rows, const Row* dev_rows, int n_rows, int64_t n, float scale,
                         int algo, cudaStream_t stream, uint64_t* stamp = nullptr, int extra_flags = 0,
                         int64_t group_tag = -1) {
  if (n < 0 || n * 4 > c->slot_bytes)
    return set_error(MGW_EINVAL, "bucket of %lld elements exceeds slot capacity %lld B", (long long)n,
                     (long long)c->slot_bytes);
  if (c->world > 1 && !c->peers_open) return set_error(MGW_EINVAL, "peers not opened (call mgw_comm_open_peers)");
  if (n == 0 || n_rows == 0) return MGW_OK;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  f.ar = make_args(c, n);
  if (group_tag >= 0) f.ar.tag = (uint32_t)group_tag;
  if (c->world > 1 && c->gate) {
    int rc = launch_gate(f.ar, stream);
    if (rc) return rc;
  }
  f.ar.stamp = stamp;
  f.ar.flags |= extra_flags;
  f.use_inline = n_rows <= kInlineRows && host_rows != nullptr;
  if (f.use_inline)
    for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = host_rows[k];
  f.rows = dev_rows;
  f.n_rows = n_rows;
  f.scale = scale;
  const int chosen = resolve_fused_algo(c, n, algo);
  if (chosen == MGW_ALGO_NVLS) {
    if (!c->nvls_bound) return set_error(MGW_EINVAL, "NVLS not set up on this communicator");
    if ((size_t)n * 4 > c->nvls_bytes)
      return set_error(MGW_EINVAL, "bucket of %lld B exceeds the NVLS buffer (%zu B)", (long long)(n * 4), c->nvls_bytes);
    NvlsArgs x;
    memset(&x, 0, sizeof(x));
    x.f = f;
    x.uc = reinterpret_cast<float*>(c->nvls_uc);
    x.mc = reinterpret_cast<float*>(c->nvls_mcva);
    return launch_nvls(x, c->max_ctas, stream, c->vec_per_cta);
  }
  if (chosen == MGW_ALGO_LL) {
    LLArgs l;
    memset(&l, 0, sizeof(l));
    l.f = f;
    for (int s = 0; s < c->world; ++s) {
      l.ll[s] = reinterpret_cast<uint64_t*>(c->peer[s] + kLLOff);
      l.hdr[s] = reinterpret_cast<uint64_t*>(c->peer[s] + kArriveOff);  // CTA 0's arrive flags
    }
    l.hdr_stride = (int64_t)kMaxBlocks * kMaxRanks;
    return launch_ll(l, c->max_ctas, stream);
  }
  if (chosen == MGW_ALGO_LL128 || chosen == MGW_ALGO_LL128_ONESHOT) {
    L128Args x;
    memset(&x, 0, sizeof(x));
    x.f = f;
    for (int s = 0; s < c->world; ++s) {
      x.in[s] = c->peer[s] + kSlotOff;
      x.gat[s] = c->peer[s] + kSlotOff + 2 * c->slot_bytes;
      x.hdr[s] = reinterpret_cast<uint64_t*>(c->peer[s] + kArriveOff);
    }
    x.hdr_stride = (int64_t)kMaxBlocks * kMaxRanks;
    return launch_ll128(x, c->max_ctas, stream, c->vec_per_cta, false, chosen == MGW_ALGO_LL128_ONESHOT);
  }
  if (chosen == MGW_ALGO_PUSH_ONESHOT || chosen == MGW_ALGO_PUSH || chosen == MGW_ALGO_PUSH_PIPE) {
    // incoming rows: one 64-B aligned row per source (one-shot), or one part + tail per
    // source (two-shot, push_stride()); resolve_fused_algo checked that they fit the slot
    const bool one = chosen == MGW_ALGO_PUSH_ONESHOT;
    PushArgs x;
    memset(&x, 0, sizeof(x));
    x.f = f;
    x.stride = one ? round_up(n, 16) : push_stride(n / 4, c->world);
    for (int s = 0; s < c->world; ++s) {
      x.gather[s] = c->peer[s] + kSlotOff + 2 * c->slot_bytes;
      x.pipe[s] = reinterpret_cast<uint64_t*>(c->peer[s] + kPipeOff);
    }
    if (chosen == MGW_ALGO_PUSH_PIPE) return launch_push_pipe(x, c->max_ctas, stream, c->vec_per_cta);
    return one ? launch_push1(x, c->max_ctas, stream, c->vec_per_cta)
               : launch_push(x, push_cap(c, n * 4), stream, c->vec_per_cta);
  }
  return launch_fused(f, chosen, c->max_ctas, stream, c->vec_per_cta);
}

// Single rank: the group's fused kernel with N = 1 -- pack into the local bucket, the
// one-input fold, write back -- one launch per group like the multi-rank path.  Every
// thread re-reads only the bucket slots it packed itself, so no barrier is needed.
int64_t g_local_min_slots = 128;  // mgw_set_option(MGW_OPT_LOCAL_MIN_SLOTS)

int local_fused(float* bucket, const Row* host_rows, const Row* dev_rows, int n_rows, int64_t n, float scale,
                cudaStream_t stream, uint64_t* stamp = nullptr, int extra_flags = 0) {
  if (n == 0 || n_rows == 0) return MGW_OK;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  f.ar.slot[0] = reinterpret_cast<char*>(bucket);
  f.ar.n = n;
  f.ar.world = 1;
  f.ar.flags = kNoBarrier | extra_flags;
  f.ar.stamp = stamp;
  f.use_inline = n_rows <= kInlineRows && host_rows != nullptr;
  if (f.use_inline)
    for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = host_rows[k];
  f.rows = dev_rows;
  f.n_rows = n_rows;
  f.scale = scale;
  // slots per CTA: the group spread over one CTA per SM, but at least g_local_min_slots per
  // CTA (fewer, fuller CTAs for small groups: less CTA start skew in a ~2 us kernel)
  const int64_t nv = n >> 2;
  int64_t per = (nv + kSMs - 1) / kSMs;
  per = (per + 127) / 128 * 128;
  const int64_t full = (int64_t)kThreads * 4;
  per = per < g_local_min_slots ? g_local_min_slots : (per > full ? full : per);
  const int64_t per_cta[2] = {per, 0};
  return launch_fused(f, MGW_ALGO_ONESHOT, 2 * kSMs, stream, per_cta);
}

// Single rank, bf16 gradients: the bf16 group kernel with N = 1 (pack -> one-input fold
// in fp32 -> bf16 write-back), the engine's stand-in like local_fused.
int local_fused_b16(uint16_t* bucket, const Row* host_rows, const Row* dev_rows, int n_rows, int64_t n, float scale,
                    cudaStream_t stream, uint64_t* stamp = nullptr) {
  if (n == 0 || n_rows == 0) return MGW_OK;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  f.ar.slot[0] = reinterpret_cast<char*>(bucket);
  f.ar.n = n;
  f.ar.world = 1;
  f.ar.flags = kNoBarrier;
  f.ar.stamp = stamp;
  f.use_inline = n_rows <= kInlineRows && host_rows != nullptr;
  if (f.use_inline)
    for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = host_rows[k];
  f.rows = dev_rows;
  f.n_rows = n_rows;
  f.scale = scale;
  return launch_b16(f, MGW_ALGO_ONESHOT, 2 * kSMs, stream);
}

// bf16 group exchange with fp32 accumulation (bf16.cuh): one-shot / two-shot only
int comm_allreduce_fused_bf16(mgw_comm* c, const Row* host_rows, const Row* dev_rows, int n_rows, int64_t n,
                              float scale, int algo, cudaStream_t stream, uint64_t* stamp = nullptr,
                              int64_t group_tag = -1) {
  if (n < 0 || n * 2 > c->slot_bytes)
    return set_error(MGW_EINVAL, "bf16 bucket of %lld elements exceeds slot capacity %lld B", (long long)n,
                     (long long)c->slot_bytes);
  if (c->world > 1 && !c->peers_open) return set_error(MGW_EINVAL, "peers not opened (call mgw_comm_open_peers)");
  if (n == 0 || n_rows == 0) return MGW_OK;
  if (c->world == 1 && scale == 1.0f) return MGW_OK;  // nothing to exchange or scale
  algo = resolve_b16_algo(c, n, algo);
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  f.ar = make_args(c, n);
  if (group_tag >= 0) f.ar.tag = (uint32_t)group_tag;
  if (c->world > 1 && c->gate) {
    int rc = launch_gate(f.ar, stream);
    if (rc) return rc;
  }
  f.ar.stamp = stamp;
  if (c->world == 1) f.ar.flags = kNoBarrier;
  f.use_inline = n_rows <= kInlineRows && host_rows != nullptr;
  if (f.use_inline)
    for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = host_rows[k];
  f.rows = dev_rows;
  f.n_rows = n_rows;
  f.scale = scale;
  if (algo == MGW_ALGO_LL) {
    LLArgs l;
    memset(&l, 0, sizeof(l));
    l.f = f;
    for (int s = 0; s < c->world; ++s) {
      l.ll[s] = reinterpret_cast<uint64_t*>(c->peer[s] + kLLOff);
      l.hdr[s] = reinterpret_cast<uint64_t*>(c->peer[s] + kArriveOff);  // CTA 0's arrive flags
    }
    l.hdr_stride = (int64_t)kMaxBlocks * kMaxRanks;
    return launch_ll_b16(l, c->max_ctas, stream);
  }
  if (algo == MGW_ALGO_LL128 || algo == MGW_ALGO_LL128_ONESHOT) {
    L128Args x;
    memset(&x, 0, sizeof(x));
    x.f = f;
    for (int s = 0; s < c->world; ++s) {
      x.in[s] = c->peer[s] + kSlotOff;
      x.gat[s] = c->peer[s] + kSlotOff + 2 * c->slot_bytes;
      x.hdr[s] = reinterpret_cast<uint64_t*>(c->peer[s] + kArriveOff);
    }
    x.hdr_stride = (int64_t)kMaxBlocks * kMaxRanks;
    return launch_ll128(x, c->max_ctas, stream, c->vec_per_cta, true, algo == MGW_ALGO_LL128_ONESHOT);
  }
  if (algo == MGW_ALGO_PUSH) {
    PushArgs x;
    memset(&x, 0, sizeof(x));
    x.f = f;
    x.stride = b16_push_stride(n, c->world);
    for (int s = 0; s < c->world; ++s) x.gather[s] = c->peer[s] + kSlotOff + 2 * c->slot_bytes;
    return launch_b16_push(x, push_cap(c, n * 2), stream);
  }
  return launch_b16(f, algo, c->max_ctas, stream);
}

const mgw_table_t* as_table(const void* t) { return static_cast<const mgw_table_t*>(t); }

int check_table(const void* t, int n, int64_t elems) {
  if (!t) return set_error(MGW_EINVAL, "table is null");
  const mgw_table_t* tb = as_table(t);
  if (n != (int)tb->host.size()) return set_error(MGW_EINVAL, "table has %d rows, %d given", (int)tb->host.size(), n);
  if (elems >= 0 && elems != tb->extent)
    return set_error(MGW_EINVAL, "bucket of %lld elements does not match the table extent %lld", (long long)elems,
                     (long long)tb->extent);
  return MGW_OK;
}

}  // namespace

extern "C" {

const char* mgw_version(void) { return "mgwfbp_b200 0.2.0 (sm_100a)"; }

int mgw_last_error(char* buf, size_t len) {
  const std::string& msg = last_error_slot();
  if (buf && len) {
    strncpy(buf, msg.c_str(), len - 1);
    buf[len - 1] = '\0';
  }
  return (int)msg.size();
}

int mgw_device_count(int* out) {
  if (!out) return set_error(MGW_EINVAL, "out is null");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return set_error(MGW_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *out = n;
  return MGW_OK;
}

int mgw_spin_ns(int64_t ns, void* stream) {
  if (ns < 0) return set_error(MGW_EINVAL, "spin time must be >= 0, got %lld", (long long)ns);
  spin_relative_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ns);
  MGW_CHECK_LAUNCH();
  return MGW_OK;
}

int mgw_desc_upload(const mgw_tensor_desc* rows, int n, void** table) {
  if (!table || n < 1 || !rows) return set_error(MGW_EINVAL, "bad descriptor table arguments");
  int64_t expect = 0;
  for (int i = 0; i < n; ++i) {
    if (rows[i].count < 0 || !rows[i].ptr) return set_error(MGW_EINVAL, "row %d: negative count or null pointer", i);
    if (rows[i].offset != expect)
      return set_error(MGW_EINVAL, "row %d: rows must tile the bucket contiguously (offset %lld, expected %lld)", i,
                       (long long)rows[i].offset, (long long)expect);
    expect += rows[i].count;
  }
  mgw_table_t* t = new mgw_table_t();
  t->host.assign(reinterpret_cast<const Row*>(rows), reinterpret_cast<const Row*>(rows) + n);
  t->extent = expect;
  cudaError_t e = cudaMalloc(&t->dev, sizeof(Row) * (size_t)n);
  if (e == cudaSuccess) e = cudaMemcpy(t->dev, rows, sizeof(Row) * (size_t)n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (t->dev) cudaFree(t->dev);
    delete t;
    return set_error(MGW_ECUDA, "descriptor upload: %s", cudaGetErrorString(e));
  }
  *table = t;
  return MGW_OK;
}

int mgw_desc_free(void* table) {
  if (table) {
    mgw_table_t* t = static_cast<mgw_table_t*>(table);
    if (t->dev) cudaFree(t->dev);
    delete t;
  }
  return MGW_OK;
}

int mgw_pack(const void* table, int n, float* bucket, int64_t bucket_elems, float scale, void* stream) {
  if (!bucket) return set_error(MGW_EINVAL, "bucket is null");
  int rc = check_table(table, n, bucket_elems);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  return launch_rows<RowOp::kPack>(t->host.data(), t->dev, n, bucket, bucket_elems, scale, nullptr, nullptr, 0, nullptr,
                                   static_cast<cudaStream_t>(stream));
}

int mgw_unpack(const void* table, int n, const float* bucket, int64_t bucket_elems, void* stream) {
  if (!bucket) return set_error(MGW_EINVAL, "bucket is null");
  int rc = check_table(table, n, bucket_elems);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  return launch_rows<RowOp::kUnpack>(t->host.data(), t->dev, n, const_cast<float*>(bucket), bucket_elems, 1.f, nullptr,
                                     nullptr, 0, nullptr, static_cast<cudaStream_t>(stream));
}

int mgw_fill_const(const void* table, int n, const float* values_dev, void* stream) {
  if (!values_dev) return set_error(MGW_EINVAL, "values are null");
  int rc = check_table(table, n, -1);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  return launch_rows<RowOp::kFill>(t->host.data(), t->dev, n, nullptr, t->extent, 1.f, values_dev, nullptr, 0, nullptr,
                                   static_cast<cudaStream_t>(stream));
}

int mgw_check_const(const void* table, int n, const float* values_dev, int64_t* mismatches, void* stream) {
  if (!values_dev || !mismatches) return set_error(MGW_EINVAL, "bad check arguments");
  int rc = check_table(table, n, -1);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // stream-ordered scratch: no cudaFree (an implicit device-wide sync would stall an
  // in-process rank group whose peers are mid-collective)
  unsigned long long* d_bad = nullptr;
  MGW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(unsigned long long), s));
  cudaError_t e = cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) {
    cudaFreeAsync(d_bad, s);
    return set_error(MGW_ECUDA, "check: %s", cudaGetErrorString(e));
  }
  rc = launch_rows<RowOp::kCheck>(t->host.data(), t->dev, n, nullptr, t->extent, 1.f, values_dev, nullptr, 0, d_bad, s);
  unsigned long long bad = 0;
  if (rc == MGW_OK) {
    e = cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "check: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(d_bad, s);
  *mismatches = (int64_t)bad;
  return rc;
}

int mgw_comm_create(int rank, int world, int device, int64_t capacity_bytes, mgw_comm** out, uint8_t* ipc_handle_out) {
  if (!out) return set_error(MGW_EINVAL, "out is null");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks) return set_error(MGW_EINVAL, "world must lie in 1..%d, got %d", kMaxRanks, world);
  if (rank < 0 || rank >= world) return set_error(MGW_EINVAL, "rank must lie in [0, %d), got %d", world, rank);
  if (capacity_bytes < 0) return set_error(MGW_EINVAL, "capacity must be >= 0");
  MGW_CUDA(cudaSetDevice(device));
  mgw_comm* c = new mgw_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->capacity = capacity_bytes;
  // + one 16-B slot per rank of slack: the push two-shot's incoming rows are part-rounded
  c->slot_bytes = round_up(std::max<int64_t>(capacity_bytes, 256) + 2 * kMaxRanks * 16, 256);
  // one-shot pulls (N-1) M per rank, two-shot 2 (N-1)/N M in two phases: measured
  // crossover on B200 ~ 8 MB / (N - 1) (profiles/ar_sweep_n*_r01_*.json)
  c->oneshot_max_bytes = world > 1 ? (8ll << 20) / (world - 1) : (1ll << 20);
  // LL beats every barrier-based exchange up to 1 MB at N = 2 and 512 KB at N <= 4
  // (engine-mode sweeps, profiles/grid_ll_n{2,4}_r01.json); its 2x wire bytes grow with N
  c->ll_max_bytes = world == 2 ? (1ll << 20) : (world <= 4 ? (512ll << 10) : (256ll << 10));
  // [control | LL | slot 0 | slot 1 | gather 0 | gather 1] (gather: push two-shot)
  const size_t region_bytes = kSlotOff + 4 * (size_t)c->slot_bytes;
  cudaError_t e = cudaMalloc(&c->region, region_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->region, 0, kSlotOff);  // flags, headers, LL area
  if (e == cudaSuccess) e = cudaMalloc(&c->state, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(c->state, 0, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&c->result, (size_t)c->slot_bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && ipc_handle_out) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, c->region);
    if (e == cudaSuccess) memcpy(ipc_handle_out, &h, MGW_IPC_HANDLE_BYTES);
  }
  if (e != cudaSuccess) {
    mgw_comm_destroy(c);
    return set_error(MGW_ECUDA, "communicator setup on device %d: %s", device, cudaGetErrorString(e));
  }
  c->peer[rank] = c->region;
  if (world == 1) c->peers_open = true;
  *out = c;
  return MGW_OK;
}

int mgw_comm_open_peers(mgw_comm* c, const uint8_t* handles) {
  if (!c) return set_error(MGW_EINVAL, "comm is null");
  if (c->world == 1) return MGW_OK;
  if (!handles) return set_error(MGW_EINVAL, "handles is null");
  MGW_CUDA(cudaSetDevice(c->device));
  for (int s = 0; s < c->world; ++s) {
    if (s == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + (size_t)s * MGW_IPC_HANDLE_BYTES, MGW_IPC_HANDLE_BYTES);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return set_error(MGW_EPROTO, "rank %d: cannot map rank %d's bucket: %s", c->rank, s, cudaGetErrorString(e));
    c->peer[s] = static_cast<char*>(p);
  }
  c->peers_open = true;
  return MGW_OK;
}

int mgw_comm_destroy(mgw_comm* c) {
  if (!c) return MGW_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (driver().ok) {
    const DriverFns& d = driver();
    if (c->nvls_mcva) {
      d.mem_unmap(c->nvls_mcva, c->nvls_bytes);
      d.addr_free(c->nvls_mcva, c->nvls_bytes);
    }
    if (c->nvls_uc) {
      d.mem_unmap(c->nvls_uc, c->nvls_bytes);
      d.addr_free(c->nvls_uc, c->nvls_bytes);
    }
    if (c->nvls_bound) d.mc_unbind(c->nvls_mc, (CUdevice)c->device, 0, c->nvls_bytes);
    if (c->nvls_mem) d.mem_release(c->nvls_mem);
    if (c->nvls_mc_valid) d.mem_release(c->nvls_mc);
  }
  if (!c->local_group)
    for (int s = 0; s < kMaxRanks; ++s)
      if (s != c->rank && c->peer[s]) cudaIpcCloseMemHandle(c->peer[s]);
  if (c->region) cudaFree(c->region);
  if (c->state) cudaFree(c->state);
  if (c->err) cudaFree(c->err);
  if (c->result) cudaFree(c->result);
  delete c;
  return MGW_OK;
}

int mgw_comm_set_timeout_ms(mgw_comm* c, int64_t ms) {
  if (!c || ms <= 0) return set_error(MGW_EINVAL, "bad timeout");
  c->timeout_ns = (uint64_t)ms * 1000000ull;
  return MGW_OK;
}

int mgw_comm_set_oneshot_max(mgw_comm* c, int64_t bytes) {
  if (!c || bytes < 0) return set_error(MGW_EINVAL, "bad one-shot threshold");
  c->oneshot_max_bytes = bytes;
  return MGW_OK;
}

int mgw_comm_set_ll_max(mgw_comm* c, int64_t bytes) {
  if (!c || bytes < 0 || bytes > kLLElems * 4) return set_error(MGW_EINVAL, "LL threshold must lie in 0..%lld B", (long long)(kLLElems * 4));
  c->ll_max_bytes = bytes;
  return MGW_OK;
}

int mgw_comm_set_tuning(mgw_comm* c, int key, int64_t value) {
  if (!c || key < 0 || key > 1 || value < 0) return set_error(MGW_EINVAL, "bad tuning key/value");
  c->vec_per_cta[key] = value;
  return MGW_OK;
}

int mgw_comm_set_max_ctas(mgw_comm* c, int ctas) {
  if (!c || ctas < 1 || ctas > kMaxBlocks) return set_error(MGW_EINVAL, "CTA cap must lie in 1..%d", kMaxBlocks);
  c->max_ctas = ctas;
  return MGW_OK;
}

int mgw_comm_set_gate(mgw_comm* c, int enable) {
  if (!c) return set_error(MGW_EINVAL, "communicator is null");
  c->gate = enable != 0;
  return MGW_OK;
}

int mgw_comm_set_group_tag(mgw_comm* c, uint32_t tag) {
  if (!c) return set_error(MGW_EINVAL, "communicator is null");
  c->group_tag = tag;
  return MGW_OK;
}

int mgw_comm_pick_algo(mgw_comm* c, int64_t n_elem, int element_bytes, int* algo) {
  if (!c || !algo || n_elem < 0 || (element_bytes != 2 && element_bytes != 4))
    return set_error(MGW_EINVAL, "bad algorithm query");
  *algo = element_bytes == 2 ? resolve_b16_algo(c, n_elem, MGW_ALGO_AUTO) : resolve_fused_algo(c, n_elem, MGW_ALGO_AUTO);
  return MGW_OK;
}

int mgw_comm_clear_error(mgw_comm* c) {
  if (!c) return set_error(MGW_EINVAL, "communicator is null");
  if (int rc = sync_for_query(c)) return rc;
  const uint32_t zero = 0;
  MGW_CUDA(cudaMemcpy(c->err, &zero, sizeof(zero), cudaMemcpyHostToDevice));
  MGW_CUDA(cudaMemcpy(c->region + kAbortOff, &zero, sizeof(zero), cudaMemcpyHostToDevice));
  return MGW_OK;
}

// Every rank of an in-process group (mgw_comm_create_local) runs its fused group exchange
// in ONE cooperative launch: each rank's arguments, algorithm, grid and tag come from its
// own communicator exactly as mgw_allreduce_fused[_bf16] would build them, so the real
// barrier / LL / push protocol (and any disagreement between the ranks) plays out between
// co-resident CTAs.  n_elem[r] < 0: rank r is absent (launches no CTAs).
int mgw_group_allreduce_fused(mgw_comm* const* comms, void* const* tables, const int64_t* n_elem, const float* scale,
                              int world, int algo, int element_bytes, void* stream) {
  if (!comms || !tables || !n_elem || !scale || world < 2 || world > kMaxRanks)
    return set_error(MGW_EINVAL, "bad rank-group arguments");
  if (element_bytes != 4 && element_bytes != 2) return set_error(MGW_EINVAL, "element_bytes must be 4 or 2");
  const bool b16 = element_bytes == 2;
  int chosen = -1;
  for (int r = 0; r < world; ++r) {
    const mgw_comm* c = comms[r];
    if (!c || !c->local_group || c->rank != r || c->world != world)
      return set_error(MGW_EINVAL, "rank %d: not rank %d of an in-process group of %d", r, r, world);
    if (n_elem[r] < 0) continue;
    if (n_elem[r] == 0 || (int64_t)n_elem[r] * element_bytes > c->slot_bytes)
      return set_error(MGW_EINVAL, "rank %d: bucket of %lld elements outside (0, slot]", r, (long long)n_elem[r]);
    const mgw_table_t* t = as_table(tables[r]);
    if (int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n_elem[r])) return rc;
    const int a = b16 ? resolve_b16_algo(c, n_elem[r], algo) : resolve_fused_algo(c, n_elem[r], algo);
    if (chosen >= 0 && a != chosen)
      return set_error(MGW_EINVAL, "a rank-group launch runs one kernel: ranks resolved algorithms %d and %d", chosen, a);
    chosen = a;
  }
  if (chosen < 0) return MGW_OK;
  if (chosen == MGW_ALGO_NVLS) return set_error(MGW_EINVAL, "NVLS has no rank-group launch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool ll = chosen == MGW_ALGO_LL, l128 = chosen == MGW_ALGO_LL128 || chosen == MGW_ALGO_LL128_ONESHOT,
             l128_one = chosen == MGW_ALGO_LL128_ONESHOT,
             push = chosen == MGW_ALGO_PUSH || chosen == MGW_ALGO_PUSH_ONESHOT || chosen == MGW_ALGO_PUSH_PIPE;
  // the argument blocks are large (8 ranks x ~1.5 KB): build them on the heap
  std::unique_ptr<RankGroup<FusedArgs>> gf(new RankGroup<FusedArgs>());
  std::unique_ptr<RankGroup<PushArgs>> gp(new RankGroup<PushArgs>());
  std::unique_ptr<RankGroup<LLArgs>> gl(new RankGroup<LLArgs>());
  std::unique_ptr<RankGroup<L128Args>> g8(new RankGroup<L128Args>());
  memset(g8.get(), 0, sizeof(*g8));
  memset(gf.get(), 0, sizeof(*gf));
  memset(gp.get(), 0, sizeof(*gp));
  memset(gl.get(), 0, sizeof(*gl));
  int first = 0;
  for (int r = 0; r < world; ++r) {
    gf->first[r] = gp->first[r] = gl->first[r] = g8->first[r] = first;
    if (n_elem[r] < 0) continue;
    const mgw_comm* c = comms[r];
    const mgw_table_t* t = as_table(tables[r]);
    const int64_t n = n_elem[r];
    FusedArgs f;
    memset(&f, 0, sizeof(f));
    f.ar = make_args(c, n);
    const int n_rows = (int)t->host.size();
    f.use_inline = n_rows <= kInlineRows;
    if (f.use_inline)
      for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = t->host[k];
    f.rows = t->dev;
    f.n_rows = n_rows;
    f.scale = scale[r];
    int grid = 0;
    if (ll) {
      LLArgs& l = gl->args[r];
      l.f = f;
      for (int q = 0; q < world; ++q) {
        l.ll[q] = reinterpret_cast<uint64_t*>(c->peer[q] + kLLOff);
        l.hdr[q] = reinterpret_cast<uint64_t*>(c->peer[q] + kArriveOff);
      }
      l.hdr_stride = (int64_t)kMaxBlocks * kMaxRanks;
      if (n > (b16 ? 2 : 1) * kLLElems) return set_error(MGW_EINVAL, "LL bucket of %lld elements too large", (long long)n);
      grid = b16 ? plan_ll_b16(l, c->max_ctas) : plan_ll(l, c->max_ctas);
    } else if (l128) {
      L128Args& x = g8->args[r];
      x.f = f;
      for (int q = 0; q < world; ++q) {
        x.in[q] = c->peer[q] + kSlotOff;
        x.gat[q] = c->peer[q] + kSlotOff + 2 * c->slot_bytes;
        x.hdr[q] = reinterpret_cast<uint64_t*>(c->peer[q] + kArriveOff);
      }
      x.hdr_stride = (int64_t)kMaxBlocks * kMaxRanks;
      grid = plan_ll128(x, c->max_ctas, c->vec_per_cta, b16, l128_one);
    } else if (push && b16) {
      PushArgs& x = gp->args[r];
      x.f = f;
      x.stride = b16_push_stride(n, world);
      for (int q = 0; q < world; ++q) x.gather[q] = c->peer[q] + kSlotOff + 2 * c->slot_bytes;
      grid = plan_b16_push(x, c->max_ctas);
    } else if (push) {
      const bool one = chosen == MGW_ALGO_PUSH_ONESHOT;
      PushArgs& x = gp->args[r];
      x.f = f;
      x.stride = one ? round_up(n, 16) : push_stride(n / 4, world);
      for (int q = 0; q < world; ++q) {
        x.gather[q] = c->peer[q] + kSlotOff + 2 * c->slot_bytes;
        x.pipe[q] = reinterpret_cast<uint64_t*>(c->peer[q] + kPipeOff);
      }
      grid = one ? plan_push1(x, c->max_ctas, c->vec_per_cta)
                 : (chosen == MGW_ALGO_PUSH_PIPE ? plan_push_pipe(x, c->max_ctas, c->vec_per_cta)
                                                 : plan_push(x, c->max_ctas, c->vec_per_cta));
    } else {
      gf->args[r] = f;
      grid = b16 ? plan_b16(gf->args[r], chosen, c->max_ctas) : plan_fused(gf->args[r], chosen, c->max_ctas, c->vec_per_cta);
    }
    first += grid;
  }
  for (int r = world; r <= kMaxRanks; ++r) gf->first[r] = gp->first[r] = gl->first[r] = g8->first[r] = first;
  if (first > 2 * kSMs)
    return set_error(MGW_EINVAL, "rank group needs %d co-resident CTAs (> %d): lower the CTA caps", first, 2 * kSMs);
  if (ll) return b16 ? launch_ll_b16_group(*gl, world, s) : launch_ll_group(*gl, world, s);
  if (l128) return launch_ll128_group(*g8, world, s, b16, l128_one);
  if (push && b16) return launch_b16_push_group(*gp, world, s);
  if (push)
    return launch_push_group(*gp, world, chosen == MGW_ALGO_PUSH_ONESHOT ? 1 : (chosen == MGW_ALGO_PUSH_PIPE ? 2 : 0), s);
  return b16 ? launch_b16_group(*gf, world, chosen, s) : launch_fused_group(*gf, world, chosen, s);
}

int mgw_set_option(int key, int64_t value) {
  switch (key) {
    case MGW_OPT_ROWS_PATH: return set_rows_path((int)value);
    case MGW_OPT_PIPE_SUB_SLOTS: return set_pipe_sub_slots(value);
    case MGW_OPT_LOCAL_MIN_SLOTS:
      if (value < 128 || value > kThreads * 4 || value % 128) return set_error(MGW_EINVAL, "local min slots: 128..2048, x128");
      g_local_min_slots = value;
      return MGW_OK;
    case MGW_OPT_WIDE_MIN_BYTES:
      if (value < 0) return set_error(MGW_EINVAL, "wide min bytes must be >= 0");
      g_wide_min_bytes = value;
      return MGW_OK;
    default: return set_error(MGW_EINVAL, "unknown option %d", key);
  }
}

int mgw_checked_violations(int reset, uint64_t* total, int* checked) {
  if (!total || !checked) return set_error(MGW_EINVAL, "bad arguments");
#ifdef MGW_CHECKED
  *checked = 1;
#else
  *checked = 0;
#endif
  unsigned long long sum = 0;
  int (*getters[])(unsigned long long*, bool) = {violations_allreduce, violations_bf16, violations_fused,
                                                 violations_ll,        violations_ll128, violations_nvls,
                                                 violations_push,      violations_rows};
  for (auto get : getters) {
    unsigned long long v = 0;
    if (get(&v, reset != 0) != MGW_OK) return set_error(MGW_ECUDA, "reading the checked-build violation counters");
    sum += v;
  }
  *total = sum;
  return MGW_OK;
}

int mgw_debug_collective_tag(uint32_t group_tag, int64_t n_elem, int kind, int grid, float scale, uint32_t* out) {
  if (!out) return set_error(MGW_EINVAL, "out is null");
  *out = collective_tag(group_tag, n_elem, (uint32_t)kind, grid, scale);
  return MGW_OK;
}

int mgw_comm_create_local(int world, int device, int64_t capacity_bytes, mgw_comm** comms) {
  if (!comms || world < 1 || world > kMaxRanks) return set_error(MGW_EINVAL, "bad local group arguments");
  for (int r = 0; r < world; ++r) comms[r] = nullptr;
  for (int r = 0; r < world; ++r) {
    int rc = mgw_comm_create(r, world, device, capacity_bytes, &comms[r], nullptr);
    if (rc) {
      for (int q = 0; q < r; ++q) mgw_comm_destroy(comms[q]);
      for (int q = 0; q < world; ++q) comms[q] = nullptr;
      return rc;
    }
  }
  for (int r = 0; r < world; ++r) {
    mgw_comm* c = comms[r];
    for (int s = 0; s < world; ++s) c->peer[s] = comms[s]->region;
    c->peers_open = true;
    c->local_group = true;
    // every rank's grid must be co-resident on the one device: 2 CTAs of 512 threads per SM
    c->max_ctas = std::max(1, 2 * kSMs / world);
  }
  return MGW_OK;
}

int mgw_comm_input(mgw_comm* c, float** slot) {
  if (!c || !slot) return set_error(MGW_EINVAL, "bad arguments");
  uint32_t calls = 0;
  if (c->world > 1) {
    MGW_CUDA(cudaSetDevice(c->device));
    MGW_CUDA(cudaDeviceSynchronize());
    MGW_CUDA(cudaMemcpy(&calls, c->state, sizeof(calls), cudaMemcpyDeviceToHost));
  }
  const int64_t parity = c->world > 1 ? (int64_t)((calls + 1u) & 1u) : 0;
  *slot = reinterpret_cast<float*>(c->region + kSlotOff + parity * c->slot_bytes);
  return MGW_OK;
}

int mgw_comm_result(mgw_comm* c, float** result) {
  if (!c || !result) return set_error(MGW_EINVAL, "bad arguments");
  *result = c->result;
  return MGW_OK;
}

int mgw_comm_pack(mgw_comm* c, const void* table, int n, int64_t n_elem, float scale, void* stream) {
  if (!c) return set_error(MGW_EINVAL, "comm is null");
  int rc = check_table(table, n, n_elem);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  return comm_pack(c, t->host.data(), t->dev, n, n_elem, scale, static_cast<cudaStream_t>(stream));
}

int mgw_allreduce(mgw_comm* c, int64_t n_elem, int algo, void* stream) {
  if (!c) return set_error(MGW_EINVAL, "comm is null");
  if (algo < MGW_ALGO_AUTO || algo > MGW_ALGO_TWOSHOT) return set_error(MGW_EINVAL, "unknown algorithm %d", algo);
  return comm_allreduce(c, n_elem, algo, static_cast<cudaStream_t>(stream));
}

int mgw_allreduce_fused(mgw_comm* c, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                        void* stream) {
  if (!c) return set_error(MGW_EINVAL, "comm is null");
  if (algo < MGW_ALGO_AUTO || algo > MGW_ALGO_LL128_ONESHOT) return set_error(MGW_EINVAL, "unknown algorithm %d", algo);
  int rc = check_table(table, n_rows, n_elem);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  if (c->world == 1) {
    // nothing to exchange: the reduced value is the (scaled) local gradient
    if (scale == 1.0f) return MGW_OK;
    if (n_elem * 4 > c->slot_bytes)
      return set_error(MGW_EINVAL, "bucket of %lld elements exceeds slot capacity %lld B", (long long)n_elem,
                       (long long)c->slot_bytes);
    return local_fused(reinterpret_cast<float*>(c->region + kSlotOff), t->host.data(), t->dev, n_rows, n_elem, scale,
                       static_cast<cudaStream_t>(stream));
  }
  return comm_allreduce_fused(c, t->host.data(), t->dev, n_rows, n_elem, scale, algo, static_cast<cudaStream_t>(stream));
}

int mgw_allreduce_fused_bf16(mgw_comm* c, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                             void* stream) {
  if (!c) return set_error(MGW_EINVAL, "comm is null");
  if (algo != MGW_ALGO_AUTO && algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT && algo != MGW_ALGO_LL &&
      algo != MGW_ALGO_PUSH && algo != MGW_ALGO_LL128 && algo != MGW_ALGO_LL128_ONESHOT)
    return set_error(MGW_EINVAL, "bf16 buckets support AUTO, LL, one-shot, two-shot, push two-shot and LL128 (got %d)",
                     algo);
  int rc = check_table(table, n_rows, n_elem);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  return comm_allreduce_fused_bf16(c, t->host.data(), t->dev, n_rows, n_elem, scale, algo,
                                   static_cast<cudaStream_t>(stream));
}

int mgw_probe_phases(mgw_comm* c, const void* table, int n_rows, int64_t n_elem, int algo, int reps, uint64_t* out,
                     void* stream) {
  if (!c || !out || reps < 1) return set_error(MGW_EINVAL, "bad phase-probe arguments");
  int rc = check_table(table, n_rows, n_elem);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<uint64_t> h((size_t)reps * 8, 0);
  for (int r = 0; r < reps; ++r) h[(size_t)r * 8] = ~0ull;  // first-CTA entry is a min
  uint64_t* d = nullptr;
  MGW_CUDA(cudaMalloc(&d, h.size() * sizeof(uint64_t)));
  cudaError_t e = cudaMemcpyAsync(d, h.data(), h.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s);
  for (int r = 0; r < reps && rc == MGW_OK && e == cudaSuccess; ++r)
    rc = c->world == 1  // the single-rank group kernel (pack -> one-input fold -> write-back)
             ? local_fused(reinterpret_cast<float*>(c->region + kSlotOff), t->host.data(), t->dev, n_rows, n_elem, 1.f,
                           s, d + (size_t)r * 8, kPhaseMarks)
             : comm_allreduce_fused(c, t->host.data(), t->dev, n_rows, n_elem, 1.f, algo, s, d + (size_t)r * 8,
                                    kPhaseMarks);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d);
  if (rc) return rc;
  if (e != cudaSuccess) return set_error(MGW_ECUDA, "phase probe: %s", cudaGetErrorString(e));
  memcpy(out, h.data(), h.size() * sizeof(uint64_t));
  return MGW_OK;
}

int mgw_nvls_supported(int device, int* ok) {
  if (!ok) return set_error(MGW_EINVAL, "ok is null");
  *ok = 0;
  if (!driver().ok) return MGW_OK;
  int v = 0;
  if (driver().get_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)device) == CUDA_SUCCESS) *ok = v;
  return MGW_OK;
}

// rank 0: create the multicast object for `bytes` (rounded up) and export a POSIX fd
int mgw_nvls_create(mgw_comm* c, int64_t bytes, int* fd_out) {
  if (!c || !fd_out || bytes <= 0 || c->world < 2) return set_error(MGW_EINVAL, "bad NVLS arguments");
  if (!driver().ok) return set_error(MGW_ECUDA, "driver multicast entry points unavailable");
  MGW_CUDA(cudaSetDevice(c->device));
  const size_t g = nvls_granularity(c->world);
  c->nvls_bytes = (size_t)round_up(bytes, (int64_t)g);
  CUmulticastObjectProp p = {};
  p.numDevices = (unsigned)c->world;
  p.size = c->nvls_bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  MGW_CU(driver().mc_create(&c->nvls_mc, &p));
  c->nvls_mc_valid = true;
  int fd = -1;
  MGW_CU(driver().export_handle(&fd, c->nvls_mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  *fd_out = fd;
  return MGW_OK;
}

// ranks != 0: import the multicast object from the fd rank 0 exported
int mgw_nvls_import(mgw_comm* c, int fd, int64_t bytes) {
  if (!c || fd < 0 || bytes <= 0) return set_error(MGW_EINVAL, "bad NVLS arguments");
  if (!driver().ok) return set_error(MGW_ECUDA, "driver multicast entry points unavailable");
  MGW_CUDA(cudaSetDevice(c->device));
  c->nvls_bytes = (size_t)round_up(bytes, (int64_t)nvls_granularity(c->world));
  MGW_CU(driver().import_handle(&c->nvls_mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  c->nvls_mc_valid = true;
  return MGW_OK;
}

// every rank adds its device; all ranks must finish this before any binds memory
int mgw_nvls_add_device(mgw_comm* c) {
  if (!c || !c->nvls_mc_valid) return set_error(MGW_EINVAL, "no multicast object");
  MGW_CU(driver().mc_add(c->nvls_mc, (CUdevice)c->device));
  return MGW_OK;
}

// every rank: allocate its copy, bind it to the multicast object, map unicast + multicast
int mgw_nvls_bind(mgw_comm* c) {
  if (!c || !c->nvls_mc_valid) return set_error(MGW_EINVAL, "no multicast object");
  const DriverFns& d = driver();
  MGW_CUDA(cudaSetDevice(c->device));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = c->device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // as the multicast object's
  MGW_CU(d.mem_create(&c->nvls_mem, c->nvls_bytes, &prop, 0));
  MGW_CU(d.mc_bind(c->nvls_mc, 0, c->nvls_mem, 0, c->nvls_bytes, 0));
  c->nvls_bound = true;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const size_t g = nvls_granularity(c->world);
  MGW_CU(d.addr_reserve(&c->nvls_uc, c->nvls_bytes, g, 0, 0));
  MGW_CU(d.mem_map(c->nvls_uc, c->nvls_bytes, 0, c->nvls_mem, 0));
  MGW_CU(d.set_access(c->nvls_uc, c->nvls_bytes, &acc, 1));
  MGW_CU(d.addr_reserve(&c->nvls_mcva, c->nvls_bytes, g, 0, 0));
  MGW_CU(d.mem_map(c->nvls_mcva, c->nvls_bytes, 0, c->nvls_mc, 0));
  MGW_CU(d.set_access(c->nvls_mcva, c->nvls_bytes, &acc, 1));
  MGW_CUDA(cudaMemset(reinterpret_cast<void*>(c->nvls_uc), 0, c->nvls_bytes));
  MGW_CUDA(cudaDeviceSynchronize());
  return MGW_OK;
}

int mgw_comm_set_nvls_min(mgw_comm* c, int64_t bytes) {
  if (!c || bytes < 0) return set_error(MGW_EINVAL, "bad NVLS threshold");
  c->nvls_min_bytes = bytes;
  return MGW_OK;
}

int mgw_event_create(void** event) {
  if (!event) return set_error(MGW_EINVAL, "event is null");
  cudaEvent_t e = nullptr;
  MGW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  *event = e;
  return MGW_OK;
}

int mgw_event_destroy(void* event) {
  if (event) MGW_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
  return MGW_OK;
}

// One call per ready merge group (autograd hook path): the comm stream waits for
// everything enqueued so far on the compute stream, then runs the fused exchange.
int mgw_group_launch(mgw_comm* c, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                     void* compute_stream, void* comm_stream, void* event) {
  if (!event) return set_error(MGW_EINVAL, "event is null");
  cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
  cudaStream_t ms = static_cast<cudaStream_t>(comm_stream);
  MGW_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), cs));
  MGW_CUDA(cudaStreamWaitEvent(ms, static_cast<cudaEvent_t>(event), 0));
  return mgw_allreduce_fused(c, table, n_rows, n_elem, scale, algo, ms);
}

int mgw_group_launch_bf16(mgw_comm* c, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                          void* compute_stream, void* comm_stream, void* event) {
  if (!event) return set_error(MGW_EINVAL, "event is null");
  cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
  cudaStream_t ms = static_cast<cudaStream_t>(comm_stream);
  MGW_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), cs));
  MGW_CUDA(cudaStreamWaitEvent(ms, static_cast<cudaEvent_t>(event), 0));
  return mgw_allreduce_fused_bf16(c, table, n_rows, n_elem, scale, algo, ms);
}

int mgw_comm_error(mgw_comm* c, int* code) {
  if (!c || !code) return set_error(MGW_EINVAL, "bad arguments");
  if (int rc = sync_for_query(c)) return rc;
  MGW_CUDA(cudaMemcpy(code, c->err, sizeof(int), cudaMemcpyDeviceToHost));
  return MGW_OK;
}

int mgw_comm_calls(mgw_comm* c, int64_t* calls) {
  if (!c || !calls) return set_error(MGW_EINVAL, "bad arguments");
  uint32_t v = 0;
  if (int rc = sync_for_query(c)) return rc;
  MGW_CUDA(cudaMemcpy(&v, c->state, sizeof(v), cudaMemcpyDeviceToHost));
  *calls = v;
  return MGW_OK;
}

int mgw_allreduce_emulated(float* const* ins, float* const* outs, int world, int64_t n, int algo, void* stream) {
  if (!ins || !outs || world < 1 || world > kMaxRanks || n < 0)
    return set_error(MGW_EINVAL, "bad emulated all-reduce arguments");
  if (algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT)
    return set_error(MGW_EINVAL, "emulated all-reduce needs an explicit algorithm");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ArArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < world; ++r) {
    a.slot[r] = reinterpret_cast<char*>(ins[r]);
    a.out[r] = outs[r];
    if (algo == MGW_ALGO_ONESHOT)
      for (int q = 0; q < world; ++q)
        if (outs[r] == ins[q]) return set_error(MGW_EINVAL, "one-shot output may not alias an input");
  }
  a.n = n;
  a.world = world;
  if (n == 0) return MGW_OK;
  if (algo == MGW_ALGO_ONESHOT) {
    for (int r = 0; r < world; ++r) {
      a.rank = r;
      a.flags = kNoBarrier;
      int rc = launch_allreduce(a, algo, 2 * kSMs, s);
      if (rc) return rc;
    }
    return MGW_OK;
  }
  for (int phase = 0; phase < 2; ++phase) {
    for (int r = 0; r < world; ++r) {
      a.rank = r;
      a.flags = kNoBarrier | (phase == 0 ? kSkipPhase2 : kSkipPhase1);
      int rc = launch_allreduce(a, algo, 2 * kSMs, s);
      if (rc) return rc;
    }
  }
  return MGW_OK;
}

// Emulated ranks on one device: every rank packs its own layer tensors into its
// slot, then the fused kernel (no barriers) folds and writes back, phase by phase.
// emulated push exchanges: incoming rows and gather areas allocated here (test path)
static int push_emulated(void* const* tables, int world, int64_t n, float scale, cudaStream_t s, bool oneshot,
                         bool pipe = false) {
  if (world < 2) return set_error(MGW_EINVAL, "push exchanges need >= 2 ranks");
  const int64_t stride = oneshot ? round_up(n, 16) : push_stride(n / 4, world);
  char* mem = nullptr;
  const size_t in_bytes = (size_t)round_up((int64_t)world * stride * 4, 256);
  const size_t g_bytes = oneshot ? in_bytes : (size_t)round_up(n * 4, 256);
  MGW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mem), (size_t)world * (in_bytes + g_bytes), s));
  PushArgs x;
  memset(&x, 0, sizeof(x));
  for (int r = 0; r < world; ++r) {
    x.f.ar.slot[r] = mem + (size_t)r * in_bytes;
    x.gather[r] = mem + (size_t)world * in_bytes + (size_t)r * g_bytes;
  }
  x.f.ar.n = n;
  x.f.ar.world = world;
  x.f.scale = scale;
  x.stride = stride;
  int rc = MGW_OK;
  for (int step = 0; step < (oneshot ? 2 : 3) && rc == MGW_OK; ++step) {
    for (int r = 0; r < world && rc == MGW_OK; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      const int n_rows = (int)t->host.size();
      x.f.use_inline = n_rows <= kInlineRows;
      if (x.f.use_inline)
        for (int k = 0; k < n_rows; ++k) x.f.inline_rows[k] = t->host[k];
      x.f.rows = t->dev;
      x.f.n_rows = n_rows;
      x.f.ar.rank = r;
      x.f.ar.flags = kNoBarrier | (step == 0 ? kSkipPhase1 | kSkipPhase2
                                             : kSkipPack | (step == 1 ? kSkipPhase2 : kSkipPhase1));
      rc = oneshot ? launch_push1(x, 2 * kSMs, s, nullptr)
                   : (pipe ? launch_push_pipe(x, 2 * kSMs, s, nullptr) : launch_push(x, 2 * kSMs, s, nullptr));
    }
  }
  cudaError_t e = cudaFreeAsync(mem, s);
  if (rc == MGW_OK && e != cudaSuccess) rc = set_error(MGW_ECUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  return rc;
}

// emulated bf16 push two-shot: incoming rows and gather areas allocated here (test path)
static int b16_push_emulated(void* const* tables, int world, int64_t n, float scale, cudaStream_t s) {
  if (world < 2) return set_error(MGW_EINVAL, "push exchanges need >= 2 ranks");
  const int64_t stride = b16_push_stride(n, world);
  char* mem = nullptr;
  const size_t in_bytes = (size_t)round_up((int64_t)world * stride * 2, 256);
  const size_t g_bytes = (size_t)round_up(n * 2, 256);
  MGW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mem), (size_t)world * (in_bytes + g_bytes), s));
  PushArgs x;
  memset(&x, 0, sizeof(x));
  for (int r = 0; r < world; ++r) {
    x.f.ar.slot[r] = mem + (size_t)r * in_bytes;
    x.gather[r] = mem + (size_t)world * in_bytes + (size_t)r * g_bytes;
  }
  x.f.ar.n = n;
  x.f.ar.world = world;
  x.f.scale = scale;
  x.stride = stride;
  int rc = MGW_OK;
  for (int step = 0; step < 3 && rc == MGW_OK; ++step) {
    for (int r = 0; r < world && rc == MGW_OK; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      const int n_rows = (int)t->host.size();
      x.f.use_inline = n_rows <= kInlineRows;
      if (x.f.use_inline)
        for (int k = 0; k < n_rows; ++k) x.f.inline_rows[k] = t->host[k];
      x.f.rows = t->dev;
      x.f.n_rows = n_rows;
      x.f.ar.rank = r;
      x.f.ar.flags = kNoBarrier | (step == 0 ? kSkipPhase1 | kSkipPhase2
                                             : kSkipPack | (step == 1 ? kSkipPhase2 : kSkipPhase1));
      rc = launch_b16_push(x, 2 * kSMs, s);
    }
  }
  cudaError_t e = cudaFreeAsync(mem, s);
  if (rc == MGW_OK && e != cudaSuccess) rc = set_error(MGW_ECUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  return rc;
}

// emulated LL exchange (fp32 or bf16): every rank's pushes in one pass of launches, then
// every rank's fold in a second pass (no kernel ever waits on a later launch)
static int ll_emulated(void* const* tables, int world, int64_t n, float scale, cudaStream_t s, bool bf16) {
  if (world < 2) return set_error(MGW_EINVAL, "LL needs >= 2 ranks");
  if (n > (bf16 ? 2 : 1) * kLLElems) return set_error(MGW_EINVAL, "LL path takes at most %lld elements",
                                                      (long long)((bf16 ? 2 : 1) * kLLElems));
  const size_t hdr_bytes = 2 * kMaxRanks * sizeof(uint64_t);
  const size_t per_rank = kLLBytes + 256;  // LL area + headers / state / abort / error words
  char* mem = nullptr;
  MGW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mem), (size_t)world * per_rank, s));
  LLArgs l;
  memset(&l, 0, sizeof(l));
  for (int r = 0; r < world; ++r) {
    char* base = mem + (size_t)r * per_rank;
    l.ll[r] = reinterpret_cast<uint64_t*>(base);
    l.hdr[r] = reinterpret_cast<uint64_t*>(base + kLLBytes);
    l.hdr_stride = kMaxRanks;
    l.f.ar.abort_flag[r] = reinterpret_cast<uint32_t*>(base + kLLBytes + hdr_bytes);
  }
  l.f.ar.n = n;
  l.f.ar.world = world;
  l.f.ar.timeout_ns = 2000000000ull;
  l.f.scale = scale;
  int rc = MGW_OK;
  for (int step = 0; step < 2 && rc == MGW_OK; ++step) {
    for (int r = 0; r < world && rc == MGW_OK; ++r) {
      char* ctl = mem + (size_t)r * per_rank + kLLBytes + hdr_bytes;  // [abort u32][state u32 x2][err i32]
      if (step == 0 && r == 0) {
        for (int q = 0; q < world; ++q) {
          cudaError_t e = cudaMemsetAsync(mem + (size_t)q * per_rank + kLLBytes + hdr_bytes, 0, 16, s);
          if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "memset: %s", cudaGetErrorString(e));
        }
      }
      // every launch of rank r sees call counter 0 -> epoch 1 (finish_call advances it)
      cudaError_t e = cudaMemsetAsync(ctl + 4, 0, 8, s);
      if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "memset: %s", cudaGetErrorString(e));
      const mgw_table_t* t = as_table(tables[r]);
      const int n_rows = (int)t->host.size();
      l.f.use_inline = n_rows <= kInlineRows;
      if (l.f.use_inline)
        for (int k = 0; k < n_rows; ++k) l.f.inline_rows[k] = t->host[k];
      l.f.rows = t->dev;
      l.f.n_rows = n_rows;
      l.f.ar.rank = r;
      l.f.ar.state = reinterpret_cast<uint32_t*>(ctl + 4);
      l.f.ar.err = reinterpret_cast<int*>(ctl + 12);
      l.f.ar.flags = step == 0 ? kSkipPhase1 : kSkipPack;
      if (rc == MGW_OK) rc = bf16 ? launch_ll_b16(l, 2 * kSMs, s) : launch_ll(l, 2 * kSMs, s);
    }
  }
  int bad = 0;
  if (rc == MGW_OK) {  // any device error word set?
    for (int r = 0; r < world && rc == MGW_OK; ++r) {
      int w = 0;
      cudaError_t e = cudaMemcpyAsync(&w, mem + (size_t)r * per_rank + kLLBytes + hdr_bytes + 12, 4,
                                      cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "LL emulation: %s", cudaGetErrorString(e));
      bad |= w;
    }
  }
  cudaError_t e = cudaFreeAsync(mem, s);
  if (rc == MGW_OK && e != cudaSuccess) rc = set_error(MGW_ECUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  if (rc == MGW_OK && bad) rc = set_error(MGW_EPROTO, "emulated LL exchange raised device error %d", bad);
  return rc;
}

// LL128 two-shot with emulated ranks on one device: every rank's phase 1 (line stores), then
// every rank's phase 2 (poll + fold + result lines), then phase 3 -- each launch polls only
// lines that earlier, completed launches wrote, so no launch ever waits on another.
static int ll128_emulated(void* const* tables, int world, int64_t n, float scale, cudaStream_t s, bool b16, bool one) {
  if (world < 2) return set_error(MGW_EINVAL, "LL128 needs >= 2 ranks");
  const size_t area = (size_t)world * l128_row_lines(n, world, b16, one) * 128;
  const size_t hdr_bytes = 2 * kMaxRanks * sizeof(uint64_t);
  const size_t per_rank = 2 * area + hdr_bytes + 256;
  char* mem = nullptr;
  MGW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mem), (size_t)world * per_rank, s));
  int rc = MGW_OK;
  {
    cudaError_t e = cudaMemsetAsync(mem, 0, (size_t)world * per_rank, s);
    if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "memset: %s", cudaGetErrorString(e));
  }
  L128Args x;
  memset(&x, 0, sizeof(x));
  for (int r = 0; r < world; ++r) {
    char* base = mem + (size_t)r * per_rank;
    x.in[r] = base;
    x.gat[r] = base + area;
    x.hdr[r] = reinterpret_cast<uint64_t*>(base + 2 * area);
    x.f.ar.abort_flag[r] = reinterpret_cast<uint32_t*>(base + 2 * area + hdr_bytes);
  }
  x.hdr_stride = kMaxRanks;
  x.f.ar.n = n;
  x.f.ar.world = world;
  x.f.ar.timeout_ns = 2000000000ull;
  x.f.scale = scale;
  const int step_flags[3] = {kSkipPhase1 | kSkipPhase2, kSkipPack | kSkipPhase2, kSkipPack | kSkipPhase1};
  for (int step = 0; step < 3 && rc == MGW_OK; ++step) {
    for (int r = 0; r < world && rc == MGW_OK; ++r) {
      char* ctl = mem + (size_t)r * per_rank + 2 * area + hdr_bytes;  // [abort u32][state u32 x2][err i32]
      // every launch of rank r sees call counter 0 -> epoch 1 (finish_call advances it)
      cudaError_t e = cudaMemsetAsync(ctl + 4, 0, 8, s);
      if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "memset: %s", cudaGetErrorString(e));
      const mgw_table_t* t = as_table(tables[r]);
      const int n_rows = (int)t->host.size();
      x.f.use_inline = n_rows <= kInlineRows;
      if (x.f.use_inline)
        for (int k = 0; k < n_rows; ++k) x.f.inline_rows[k] = t->host[k];
      x.f.rows = t->dev;
      x.f.n_rows = n_rows;
      x.f.ar.rank = r;
      x.f.ar.state = reinterpret_cast<uint32_t*>(ctl + 4);
      x.f.ar.err = reinterpret_cast<int*>(ctl + 12);
      x.f.ar.flags = step_flags[step];
      if (rc == MGW_OK) rc = launch_ll128(x, 2 * kSMs, s, nullptr, b16, one);
    }
  }
  int bad = 0;
  for (int r = 0; r < world && rc == MGW_OK; ++r) {  // any device error word set?
    int w = 0;
    cudaError_t e = cudaMemcpyAsync(&w, mem + (size_t)r * per_rank + 2 * area + hdr_bytes + 12, 4,
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "LL128 emulation: %s", cudaGetErrorString(e));
    bad |= w;
  }
  cudaError_t e = cudaFreeAsync(mem, s);
  if (rc == MGW_OK && e != cudaSuccess) rc = set_error(MGW_ECUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  if (rc == MGW_OK && bad) rc = set_error(MGW_EPROTO, "emulated LL128 exchange raised device error %d", bad);
  return rc;
}

int mgw_allreduce_fused_emulated(void* const* tables, float* const* slots, int world, int64_t n, float scale, int algo,
                                 void* stream) {
  if (!tables || !slots || world < 1 || world > kMaxRanks || n < 0)
    return set_error(MGW_EINVAL, "bad emulated fused arguments");
  if (algo == MGW_ALGO_LL) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
      if (rc) return rc;
    }
    return n == 0 ? MGW_OK : ll_emulated(tables, world, n, scale, static_cast<cudaStream_t>(stream), false);
  }
  if (algo == MGW_ALGO_LL128 || algo == MGW_ALGO_LL128_ONESHOT) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
      if (rc) return rc;
    }
    return n == 0 ? MGW_OK
                  : ll128_emulated(tables, world, n, scale, static_cast<cudaStream_t>(stream), false,
                                   algo == MGW_ALGO_LL128_ONESHOT);
  }
  if (algo == MGW_ALGO_PUSH || algo == MGW_ALGO_PUSH_ONESHOT || algo == MGW_ALGO_PUSH_PIPE) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
      if (rc) return rc;
    }
    return n == 0 ? MGW_OK
                  : push_emulated(tables, world, n, scale, static_cast<cudaStream_t>(stream),
                                  algo == MGW_ALGO_PUSH_ONESHOT, algo == MGW_ALGO_PUSH_PIPE);
  }
  if (algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT)
    return set_error(MGW_EINVAL, "emulated all-reduce needs an explicit algorithm");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int r = 0; r < world; ++r) {
    const mgw_table_t* t = as_table(tables[r]);
    int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
    if (rc) return rc;
  }
  if (n == 0) return MGW_OK;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  for (int r = 0; r < world; ++r) f.ar.slot[r] = reinterpret_cast<char*>(slots[r]);
  f.ar.n = n;
  f.ar.world = world;
  f.scale = scale;
  // step 0: every rank packs with the kernel's own pack (one-shot: its chunk of the bucket,
  // two-shot: chunk b of every part); then the one-shot fold, or the two-shot's two phases
  const int phases = algo == MGW_ALGO_ONESHOT ? 1 : 2;
  for (int r = 0; r < world; ++r) {
    const mgw_table_t* t = as_table(tables[r]);
    const int n_rows = (int)t->host.size();
    f.use_inline = n_rows <= kInlineRows;
    if (f.use_inline)
      for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = t->host[k];
    f.rows = t->dev;
    f.n_rows = n_rows;
    f.ar.rank = r;
    f.ar.flags = kNoBarrier | kSkipPhase1 | kSkipPhase2;
    int rc = launch_fused(f, algo, 2 * kSMs, s);
    if (rc) return rc;
  }
  for (int phase = 0; phase < phases; ++phase) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      const int n_rows = (int)t->host.size();
      f.use_inline = n_rows <= kInlineRows;
      if (f.use_inline)
        for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = t->host[k];
      f.rows = t->dev;
      f.n_rows = n_rows;
      f.ar.rank = r;
      f.ar.flags = kNoBarrier | kSkipPack | (phases == 1 ? 0 : (phase == 0 ? kSkipPhase2 : kSkipPhase1));
      int rc = launch_fused(f, algo, 2 * kSMs, s);
      if (rc) return rc;
    }
  }
  return MGW_OK;
}

int mgw_allreduce_fused_bf16_emulated(void* const* tables, void* const* slots, int world, int64_t n, float scale,
                                      int algo, void* stream) {
  if (!tables || !slots || world < 1 || world > kMaxRanks || n < 0)
    return set_error(MGW_EINVAL, "bad emulated bf16 arguments");
  if (algo == MGW_ALGO_LL) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
      if (rc) return rc;
    }
    return n == 0 ? MGW_OK : ll_emulated(tables, world, n, scale, static_cast<cudaStream_t>(stream), true);
  }
  if (algo == MGW_ALGO_LL128 || algo == MGW_ALGO_LL128_ONESHOT) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
      if (rc) return rc;
    }
    return n == 0 ? MGW_OK
                  : ll128_emulated(tables, world, n, scale, static_cast<cudaStream_t>(stream), true,
                                   algo == MGW_ALGO_LL128_ONESHOT);
  }
  if (algo == MGW_ALGO_PUSH) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
      if (rc) return rc;
    }
    return n == 0 ? MGW_OK : b16_push_emulated(tables, world, n, scale, static_cast<cudaStream_t>(stream));
  }
  if (algo != MGW_ALGO_ONESHOT && algo != MGW_ALGO_TWOSHOT)
    return set_error(MGW_EINVAL, "emulated all-reduce needs an explicit algorithm");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int r = 0; r < world; ++r) {
    const mgw_table_t* t = as_table(tables[r]);
    int rc = check_table(tables[r], t ? (int)t->host.size() : 0, n);
    if (rc) return rc;
  }
  if (n == 0) return MGW_OK;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  for (int r = 0; r < world; ++r) f.ar.slot[r] = static_cast<char*>(slots[r]);
  f.ar.n = n;
  f.ar.world = world;
  f.scale = scale;
  // step 0 packs every rank, then the one-shot fold, or the two-shot's two phases
  const int steps = algo == MGW_ALGO_ONESHOT ? 2 : 3;
  for (int step = 0; step < steps; ++step) {
    for (int r = 0; r < world; ++r) {
      const mgw_table_t* t = as_table(tables[r]);
      const int n_rows = (int)t->host.size();
      f.use_inline = n_rows <= kInlineRows;
      if (f.use_inline)
        for (int k = 0; k < n_rows; ++k) f.inline_rows[k] = t->host[k];
      f.rows = t->dev;
      f.n_rows = n_rows;
      f.ar.rank = r;
      f.ar.flags = kNoBarrier | (step == 0 ? kSkipPhase1 | kSkipPhase2
                                           : kSkipPack | (step == 1 ? kSkipPhase2 : kSkipPhase1));
      int rc = launch_b16(f, algo, 2 * kSMs, s);
      if (rc) return rc;
    }
  }
  return MGW_OK;
}

// Device time of back-to-back group-exchange steps, timed as one event pair around
// `reps` repetitions (after `warmups` untimed ones) so no per-launch event cost
// enters the figure.  kind: 0 = pack -> all-reduce -> unpack (single rank: pack ->
// unpack into `local_bucket`), 1 = all-reduce kernel only, 2 = pack only, 3 = unpack only.
int mgw_time_exchange(mgw_comm* c, const void* table, int n_rows, int64_t n_elem, float* local_bucket, int algo,
                      int kind, int reps, int warmups, double* seconds_per_rep, void* stream) {
  const bool as_graph = (kind & MGW_TIME_GRAPH) != 0;  // replay the reps as one CUDA graph
  kind &= ~MGW_TIME_GRAPH;
  if (reps < 1 || warmups < 0 || !seconds_per_rep || n_elem <= 0 || kind < 0 || kind > 6)
    return set_error(MGW_EINVAL, "bad timing arguments");
  int rc = check_table(table, n_rows, n_elem);
  if (rc) return rc;
  const mgw_table_t* t = as_table(table);
  const bool multi = c && c->world > 1;
  if (!multi && !local_bucket) return set_error(MGW_EINVAL, "single-rank timing needs a local bucket");
  if ((kind == 1 || kind == 5 || kind == 6) && !multi)
    return set_error(MGW_EINVAL, "all-reduce timing needs a multi-rank communicator");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto step = [&]() -> int {
    int r = MGW_OK;
    if (kind == 4)
      return multi ? comm_allreduce_fused(c, t->host.data(), t->dev, n_rows, n_elem, 1.f, algo, s)
                   : local_fused(local_bucket, t->host.data(), t->dev, n_rows, n_elem, 1.f, s);
    if (kind == 5) return comm_allreduce_fused_bf16(c, t->host.data(), t->dev, n_rows, n_elem, 1.f, algo, s);
    if (kind == 6) {  // rendezvous only: the one-warp gate kernel (launch + one fabric round trip)
      ArArgs a = make_args(c, n_elem);
      int g = launch_gate(a, s);
      if (g) return g;
      // advance the call counter so the next gate waits for a new epoch
      finish_kernel<<<1, 32, 0, s>>>(c->state);
      MGW_CHECK_LAUNCH();
      return MGW_OK;
    }
    if (multi) {
      if (kind == 0 || kind == 2) r = comm_pack(c, t->host.data(), t->dev, n_rows, n_elem, 1.f, s);
      if (r == MGW_OK && (kind == 0 || kind == 1)) r = comm_allreduce(c, n_elem, algo, s);
      if (r == MGW_OK && (kind == 0 || kind == 3))
        r = launch_rows<RowOp::kUnpack>(t->host.data(), t->dev, n_rows, c->result, n_elem, 1.f, nullptr, nullptr, 0,
                                        nullptr, s);
    } else {
      if (kind == 0 || kind == 2)
        r = launch_rows<RowOp::kPack>(t->host.data(), t->dev, n_rows, local_bucket, n_elem, 1.f, nullptr, nullptr, 0,
                                      nullptr, s);
      if (r == MGW_OK && (kind == 0 || kind == 3))
        r = launch_rows<RowOp::kUnpack>(t->host.data(), t->dev, n_rows, local_bucket, n_elem, 1.f, nullptr, nullptr, 0,
                                        nullptr, s);
    }
    return r;
  };
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  MGW_CUDA(cudaEventCreate(&ev0));
  cudaError_t e = cudaEventCreate(&ev1);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev0);
    return set_error(MGW_ECUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
  }
  for (int r = 0; r < warmups && rc == MGW_OK; ++r) rc = step();
  cudaGraphExec_t exec = nullptr;
  if (as_graph && rc == MGW_OK) {
    // the reps as kernel nodes of one graph: the per-launch cost of the Algorithm-2
    // engine (which replays its iteration as a graph), not of eager stream launches
    cudaGraph_t graph = nullptr;
    e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "capture: %s", cudaGetErrorString(e));
    for (int r = 0; r < reps && rc == MGW_OK; ++r) rc = step();
    e = cudaStreamEndCapture(s, &graph);
    if (rc == MGW_OK && e != cudaSuccess) rc = set_error(MGW_ECUDA, "capture: %s", cudaGetErrorString(e));
    if (rc == MGW_OK) {
      e = cudaGraphInstantiate(&exec, graph, 0);
      if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "instantiate: %s", cudaGetErrorString(e));
    }
    if (graph) cudaGraphDestroy(graph);
    if (rc == MGW_OK) {  // one untimed replay (upload), then the timed one
      e = cudaGraphLaunch(exec, s);
      if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "graph launch: %s", cudaGetErrorString(e));
    }
  }
  if (rc == MGW_OK && !as_graph) spin_relative_kernel<<<1, 32, 0, s>>>(1000000 + 20000LL * reps);  // hold the
  // stream while the host enqueues the timed reps
  if (rc == MGW_OK) cudaEventRecord(ev0, s);
  if (as_graph) {
    if (rc == MGW_OK) {
      e = cudaGraphLaunch(exec, s);
      if (e != cudaSuccess) rc = set_error(MGW_ECUDA, "graph launch: %s", cudaGetErrorString(e));
    }
  } else {
    for (int r = 0; r < reps && rc == MGW_OK; ++r) rc = step();
  }
  if (rc == MGW_OK) {
    cudaEventRecord(ev1, s);
    e = cudaEventSynchronize(ev1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev0, ev1);
    if (e != cudaSuccess)
      rc = set_error(MGW_ECUDA, "timing loop: %s", cudaGetErrorString(e));
    else
      *seconds_per_rep = ms * 1e-3 / reps;
  }
  if (exec) cudaGraphExecDestroy(exec);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  return rc;
}

// ------------------------------------------------------------ schedule engine

static void sched_release(mgw_sched* s) {
  if (!s) return;
  if (s->graph_exec) cudaGraphExecDestroy(s->graph_exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  for (auto e : s->dep_ready) cudaEventDestroy(e);
  for (cudaEvent_t e : {s->dep_fork, s->dep_join, s->dep_compute, s->t_start, s->t_compute, s->t_end})
    if (e) cudaEventDestroy(e);
  for (void* p : {(void*)s->d_rows, (void*)s->d_fill, (void*)s->local_bucket, (void*)s->d_clock, (void*)s->d_stamps})
    if (p) cudaFree(p);
  delete s;
}

int mgw_sched_create(mgw_comm* comm, const mgw_tensor_desc* rows, int n_rows, const mgw_group* groups, int n_groups,
                     float scale, uint32_t flags, const float* fill_values, float* const* host_src,
                     float* const* host_dst, mgw_sched** out) {
  if (!out || (n_rows > 0 && !rows) || !groups || n_rows < 0 || n_groups <= 0)
    return set_error(MGW_EINVAL, "bad schedule arguments");
  *out = nullptr;
  if ((flags & MGW_SCHED_FILL) && !fill_values) return set_error(MGW_EINVAL, "MGW_SCHED_FILL needs fill_values");
  if ((flags & MGW_SCHED_HOSTIO) && (!host_src || !host_dst))
    return set_error(MGW_EINVAL, "MGW_SCHED_HOSTIO needs host_src and host_dst");
  if ((flags & MGW_SCHED_BF16) && (flags & MGW_SCHED_HOSTIO))
    return set_error(MGW_EINVAL, "MGW_SCHED_HOSTIO moves fp32 host buffers; it does not combine with MGW_SCHED_BF16");
  int64_t max_elems = 0;
  for (int g = 0; g < n_groups; ++g) {
    const mgw_group& gr = groups[g];
    if (gr.desc_begin < 0 || gr.desc_count < 0 || gr.desc_begin + gr.desc_count > n_rows)
      return set_error(MGW_EINVAL, "group %d: descriptor range outside the table", g);
    int64_t expect = 0;
    for (int k = gr.desc_begin; k < gr.desc_begin + gr.desc_count; ++k) {
      if (rows[k].offset != expect) return set_error(MGW_EINVAL, "group %d: rows must tile the bucket contiguously", g);
      expect += rows[k].count;
    }
    if (expect != gr.n_elem)
      return set_error(MGW_EINVAL, "group %d: n_elem %lld != rows total %lld", g, (long long)gr.n_elem, (long long)expect);
    if (gr.ready_ns < 0) return set_error(MGW_EINVAL, "group %d: negative ready time", g);
    if (g > 0 && gr.ready_ns < groups[g - 1].ready_ns) return set_error(MGW_EINVAL, "groups must be in send order");
    max_elems = std::max(max_elems, gr.n_elem);
  }
  const int world = comm ? comm->world : 1;
  if (comm && max_elems * ((flags & MGW_SCHED_BF16) ? 2 : 4) > comm->slot_bytes)
    return set_error(MGW_EINVAL, "largest group (%lld B) exceeds the communicator slot (%lld B)",
                     (long long)(max_elems * 4), (long long)comm->slot_bytes);
  mgw_sched* s = new mgw_sched();
  s->comm = comm;
  s->world = world;
  if (n_rows > 0) s->rows.assign(reinterpret_cast<const Row*>(rows), reinterpret_cast<const Row*>(rows) + n_rows);
  s->groups.assign(groups, groups + n_groups);
  s->scale = scale;
  s->flags = flags;
  if ((flags & MGW_SCHED_HOSTIO) && n_rows > 0) {
    s->host_src.assign(host_src, host_src + n_rows);
    s->host_dst.assign(host_dst, host_dst + n_rows);
  }
  s->h_stamps.assign((size_t)n_groups * kSchedStamps + 1, 0);  // + the iteration's clock mark
  cudaError_t e = cudaMalloc(&s->d_rows, sizeof(Row) * (size_t)std::max(1, n_rows));
  if (e == cudaSuccess && n_rows > 0) e = cudaMemcpy(s->d_rows, rows, sizeof(Row) * (size_t)n_rows, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && (flags & MGW_SCHED_FILL)) {
    e = cudaMalloc(&s->d_fill, sizeof(float) * (size_t)std::max(1, n_rows));
    if (e == cudaSuccess && n_rows > 0)
      e = cudaMemcpy(s->d_fill, fill_values, sizeof(float) * (size_t)n_rows, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && world == 1) e = cudaMalloc(&s->local_bucket, std::max<size_t>(256, (size_t)max_elems * 4));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_clock, sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMemset(s->d_clock, 0, sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_stamps, sizeof(uint64_t) * (size_t)n_groups * kSchedStamps);
  if (e == cudaSuccess) e = cudaMemset(s->d_stamps, 0, sizeof(uint64_t) * (size_t)n_groups * kSchedStamps);
  auto mk = [&](cudaEvent_t* ev, bool timing) {
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, timing ? cudaEventDefault : cudaEventDisableTiming);
  };
  mk(&s->dep_fork, false);
  mk(&s->dep_join, false);
  mk(&s->dep_compute, false);
  mk(&s->t_start, true);
  mk(&s->t_compute, true);
  mk(&s->t_end, true);
  s->dep_ready.assign(n_groups, nullptr);
  for (int g = 0; g < n_groups; ++g) mk(&s->dep_ready[g], false);
  if (e != cudaSuccess) {
    sched_release(s);
    return set_error(MGW_ECUDA, "schedule setup: %s", cudaGetErrorString(e));
  }
  int launches = 2 + (world > 1 ? 1 : 0);  // stamp reset + clock mark (+ start barrier)
  for (int g = 0; g < n_groups; ++g) {
    launches += 1;  // spin
    if (groups[g].n_elem == 0) continue;
    launches += (flags & MGW_SCHED_FILL) ? 1 : 0;  // gradient production
    if (flags & (MGW_SCHED_FUSED | MGW_SCHED_BF16))
      launches += 1 + (world > 1 && comm->gate ? 1 : 0);  // (gate +) fused pack + all-reduce + unpack
    else
      launches += world > 1 ? 3 : 2;               // pack (+ all-reduce) + unpack
  }
  s->launches = launches;
  *out = s;
  return MGW_OK;
}

// Timing events: inside a stream capture they must be external record nodes; in
// eager mode they are plain records.
static cudaError_t record_timing(const mgw_sched* s, cudaEvent_t ev, cudaStream_t st) {
  return s->capturing ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal) : cudaEventRecord(ev, st);
}

static int sched_enqueue(mgw_sched* s, cudaStream_t cs, cudaStream_t ms) {
  const Row* d_rows = s->d_rows;
  const int n_groups = (int)s->groups.size();
  if (s->world > 1) {
    // align the ranks' iteration starts: a zero-length collective is a barrier
    int rc = comm_allreduce(s->comm, 0, MGW_ALGO_ONESHOT, cs);
    if (rc) return rc;
  }
  stamps_reset_kernel<<<1, 256, 0, cs>>>(s->d_stamps, n_groups * kSchedStamps / 2);
  MGW_CHECK_LAUNCH();
  MGW_CUDA(record_timing(s, s->t_start, cs));
  MGW_CUDA(cudaEventRecord(s->dep_fork, cs));
  clock_mark_kernel<<<1, 32, 0, cs>>>(s->d_clock);
  MGW_CHECK_LAUNCH();
  for (int g = 0; g < n_groups; ++g) {
    const mgw_group& gr = s->groups[g];
    if ((s->flags & MGW_SCHED_HOSTIO) && gr.n_elem > 0) {
      for (int k = gr.desc_begin; k < gr.desc_begin + gr.desc_count; ++k)
        if (s->rows[k].count)
          MGW_CUDA(cudaMemcpyAsync(s->rows[k].ptr, s->host_src[k], s->rows[k].count * 4, cudaMemcpyHostToDevice, cs));
    }
    spin_until_kernel<<<1, 32, 0, cs>>>(s->d_clock, gr.ready_ns);
    MGW_CHECK_LAUNCH();
    if ((s->flags & MGW_SCHED_FILL) && gr.n_elem > 0) {
      // the layer's gradient is written at the END of its backward window (as a real
      // weight-gradient kernel would), so it does not contend with the previous group's
      // exchange for SMs and HBM.  MGW_SCHED_PDL: the ready event is the fill's
      // programmatic event, so the group's exchange launches while the fill runs and
      // waits for it on the device (grid_dep_wait) instead of paying a launch after it.
      const bool pdl = (s->flags & MGW_SCHED_PDL) != 0 && !(s->flags & MGW_SCHED_BF16);
      if (s->flags & MGW_SCHED_BF16) {
        fill_b16_kernel<<<2 * kSMs, kThreads, 0, cs>>>(d_rows + gr.desc_begin, gr.desc_count, s->d_fill + gr.desc_begin,
                                                     s->d_stamps + kSchedStamps * (size_t)g + 6);
        MGW_CHECK_LAUNCH();
        MGW_CUDA(cudaEventRecord(s->dep_ready[g], cs));
        continue;
      }
      int rc = launch_rows<RowOp::kFill>(s->rows.data() + gr.desc_begin, d_rows + gr.desc_begin, gr.desc_count, nullptr,
                                         gr.n_elem, 1.f, s->d_fill + gr.desc_begin, nullptr, 0, nullptr, cs,
                                         s->d_stamps + kSchedStamps * (size_t)g + 6, pdl ? s->dep_ready[g] : nullptr);
      if (rc) return rc;
      if (!pdl) MGW_CUDA(cudaEventRecord(s->dep_ready[g], cs));
    } else {
      MGW_CUDA(cudaEventRecord(s->dep_ready[g], cs));
    }
  }
  MGW_CUDA(record_timing(s, s->t_compute, cs));
  MGW_CUDA(cudaEventRecord(s->dep_compute, cs));

  MGW_CUDA(cudaStreamWaitEvent(ms, s->dep_fork, 0));
  for (int g = 0; g < n_groups; ++g) {
    const mgw_group& gr = s->groups[g];
    const Row* grows = d_rows + gr.desc_begin;
    const Row* hrows = s->rows.data() + gr.desc_begin;
    uint64_t* st = s->d_stamps + kSchedStamps * (size_t)g;
    MGW_CUDA(cudaStreamWaitEvent(ms, s->dep_ready[g], 0));
    if (gr.n_elem == 0) continue;  // silent group: nothing to send (allreduce_net.py:549)
    int rc;
    if (s->flags & MGW_SCHED_BF16) {  // bf16 gradients, fp32 accumulation (bf16.cuh), always fused
      rc = s->world == 1 ? local_fused_b16(reinterpret_cast<uint16_t*>(s->local_bucket), hrows, grows, gr.desc_count,
                                           gr.n_elem, s->scale, ms, st + 2)
                         : comm_allreduce_fused_bf16(s->comm, hrows, grows, gr.desc_count, gr.n_elem, s->scale, gr.algo,
                                                     ms, st + 2, (uint32_t)gr.head_layer);
      if (rc) return rc;
    } else if (s->world == 1 && (s->flags & MGW_SCHED_FUSED)) {
      rc = local_fused(s->local_bucket, hrows, grows, gr.desc_count, gr.n_elem, s->scale, ms, st + 2);
      if (rc) return rc;
    } else if (s->world == 1) {
      rc = launch_rows<RowOp::kPack>(hrows, grows, gr.desc_count, s->local_bucket, gr.n_elem, s->scale, nullptr, nullptr,
                                     0, nullptr, ms, st);
      if (rc) return rc;
      rc = launch_rows<RowOp::kUnpack>(hrows, grows, gr.desc_count, s->local_bucket, gr.n_elem, 1.f, nullptr, nullptr, 0,
                                       nullptr, ms, st + 4);
      if (rc) return rc;
    } else if (s->flags & MGW_SCHED_FUSED) {
      rc = comm_allreduce_fused(s->comm, hrows, grows, gr.desc_count, gr.n_elem, s->scale, gr.algo, ms, st + 2, 0,
                                (uint32_t)gr.head_layer);
      if (rc) return rc;
    } else {
      rc = comm_pack(s->comm, hrows, grows, gr.desc_count, gr.n_elem, s->scale, ms, st);
      if (rc) return rc;
      rc = comm_allreduce(s->comm, gr.n_elem, gr.algo, ms, st + 2, (uint32_t)gr.head_layer);
      if (rc) return rc;
      rc = launch_rows<RowOp::kUnpack>(hrows, grows, gr.desc_count, s->comm->result, gr.n_elem, 1.f, nullptr, nullptr, 0,
                                       nullptr, ms, st + 4);
      if (rc) return rc;
    }
    if (s->flags & MGW_SCHED_HOSTIO) {
      for (int k = gr.desc_begin; k < gr.desc_begin + gr.desc_count; ++k)
        if (s->rows[k].count)
          MGW_CUDA(cudaMemcpyAsync(s->host_dst[k], s->rows[k].ptr, s->rows[k].count * 4, cudaMemcpyDeviceToHost, ms));
    }
  }
  MGW_CUDA(cudaStreamWaitEvent(ms, s->dep_compute, 0));  // iteration ends no earlier than backward
  MGW_CUDA(record_timing(s, s->t_end, ms));
  MGW_CUDA(cudaEventRecord(s->dep_join, ms));
  MGW_CUDA(cudaStreamWaitEvent(cs, s->dep_join, 0));
  return MGW_OK;
}

int mgw_sched_run(mgw_sched* s, void* compute_stream, void* comm_stream) {
  if (!s) return set_error(MGW_EINVAL, "schedule is null");
  cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
  cudaStream_t ms = static_cast<cudaStream_t>(comm_stream);
  if (cs == ms) return set_error(MGW_EINVAL, "compute and comm streams must differ");
  if (!(s->flags & MGW_SCHED_GRAPH)) return sched_enqueue(s, cs, ms);
  if (!s->graph_exec) {
    MGW_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    s->capturing = true;
    int rc = sched_enqueue(s, cs, ms);
    s->capturing = false;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return set_error(MGW_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    s->graph = graph;
    MGW_CUDA(cudaGraphInstantiate(&s->graph_exec, graph, cudaGraphInstantiateFlagUseNodePriority));  // keep the comm stream's priority
  }
  MGW_CUDA(cudaGraphLaunch(s->graph_exec, cs));
  return MGW_OK;
}

static int sched_fetch_stamps(mgw_sched* s) {
  MGW_CUDA(cudaEventSynchronize(s->t_end));
  const size_t n = s->groups.size() * kSchedStamps;
  MGW_CUDA(cudaMemcpy(s->h_stamps.data(), s->d_stamps, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  MGW_CUDA(cudaMemcpy(s->h_stamps.data() + n, s->d_clock, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return MGW_OK;
}

// the group's exchange window from its kernel stamps [pack, all-reduce / fused, unpack]
static bool exchange_window(const uint64_t* st, uint64_t* t0, uint64_t* t1) {
  uint64_t lo = ~0ull, hi = 0;
  for (int k = 0; k < 3; ++k) {
    if (st[2 * k] == ~0ull || st[2 * k + 1] < st[2 * k]) continue;  // kernel not launched
    lo = st[2 * k] < lo ? st[2 * k] : lo;
    hi = st[2 * k + 1] > hi ? st[2 * k + 1] : hi;
  }
  *t0 = lo;
  *t1 = hi;
  return lo != ~0ull;
}

static double span_s(const uint64_t* st) {
  return (st[0] == ~0ull || st[1] < st[0]) ? 0.0 : (double)(st[1] - st[0]) * 1e-9;
}

int mgw_sched_times(mgw_sched* s, double* t_iter_s, double* compute_s, double* group_comm_s) {
  if (!s) return set_error(MGW_EINVAL, "schedule is null");
  int rc = sched_fetch_stamps(s);
  if (rc) return rc;
  float ms = 0.f;
  if (t_iter_s) {
    MGW_CUDA(cudaEventElapsedTime(&ms, s->t_start, s->t_end));
    *t_iter_s = ms * 1e-3;
  }
  if (compute_s) {
    MGW_CUDA(cudaEventElapsedTime(&ms, s->t_start, s->t_compute));
    *compute_s = ms * 1e-3;
  }
  if (group_comm_s) {
    for (size_t g = 0; g < s->groups.size(); ++g) {
      // first kernel entry .. last kernel exit of the group's exchange on the comm stream
      // (unfused: pack .. unpack; fused: the one kernel)
      uint64_t t0, t1;
      group_comm_s[g] = exchange_window(&s->h_stamps[kSchedStamps * g], &t0, &t1) ? (double)(t1 - t0) * 1e-9 : 0.0;
    }
  }
  return MGW_OK;
}

int mgw_sched_kernel_times(mgw_sched* s, double* pack_s, double* allreduce_s, double* unpack_s) {
  if (!s || !pack_s || !allreduce_s || !unpack_s) return set_error(MGW_EINVAL, "bad arguments");
  int rc = sched_fetch_stamps(s);
  if (rc) return rc;
  for (size_t g = 0; g < s->groups.size(); ++g) {
    const uint64_t* st = &s->h_stamps[kSchedStamps * g];
    pack_s[g] = span_s(st);
    allreduce_s[g] = span_s(st + 2);
    unpack_s[g] = span_s(st + 4);
  }
  return MGW_OK;
}

int mgw_sched_events(mgw_sched* s, double* ready_s, double* comm_start_s, double* comm_end_s) {
  if (!s || !ready_s || !comm_start_s || !comm_end_s) return set_error(MGW_EINVAL, "bad arguments");
  int rc = sched_fetch_stamps(s);
  if (rc) return rc;
  const uint64_t origin = s->h_stamps[s->groups.size() * kSchedStamps];  // the iteration's clock mark
  for (size_t g = 0; g < s->groups.size(); ++g) {
    const uint64_t* st = &s->h_stamps[kSchedStamps * g];
    const bool filled = st[6] != ~0ull && st[7] >= st[6];
    ready_s[g] = filled ? ((double)st[7] - (double)origin) * 1e-9 : -1.0;
    uint64_t t0, t1;
    if (exchange_window(st, &t0, &t1)) {
      comm_start_s[g] = ((double)t0 - (double)origin) * 1e-9;
      comm_end_s[g] = ((double)t1 - (double)origin) * 1e-9;
    } else {
      comm_start_s[g] = comm_end_s[g] = -1.0;
    }
  }
  return MGW_OK;
}

int mgw_sched_launches(mgw_sched* s, int* per_iteration) {
  if (!s || !per_iteration) return set_error(MGW_EINVAL, "bad arguments");
  *per_iteration = s->launches;
  return MGW_OK;
}

int mgw_sched_destroy(mgw_sched* s) {
  if (s) {
    cudaDeviceSynchronize();
    sched_release(s);
  }
  return MGW_OK;
}

}  // extern "C"
