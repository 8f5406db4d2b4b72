/*
 * mgwfbp_b200.h -- C ABI of the B200-native MG-WFBP merged-gradient data path.
 *
 * Plain C types only (pointers, sizes, ints); no torch types cross this
 * boundary.  Every function returns an int status:
 *
 *   MGW_OK     0  success
 *   MGW_EINVAL 1  invalid argument                     -> Python ValueError
 *   MGW_EPROTO 2  peer / length / timeout disagreement -> Python ProtocolError
 *   MGW_ECUDA  3  CUDA runtime failure                 -> Python RuntimeError
 *
 * and leaves a message readable with mgw_last_error().  Data-path calls are
 * asynchronous on the caller's cudaStream_t (passed as void*).
 *
 * Which reference interface each entry point replaces
 * (reference = /root/reference/pkg/src/mgwfbp):
 *
 *   mgw_spin_ns / sched spins    <- allreduce_net.py:448-460  (_delay, simulated backward)
 *   mgw_pack / mgw_comm_pack     <- allreduce_net.py:544-546  (per-layer fill of the group
 *                                   buffer, layout :495-509: layer `high` at offset 0)
 *   mgw_comm_create / open_peers <- allreduce_net.py:180-262  (rendezvous + RingSession:
 *                                   here CUDA-IPC handles instead of TCP ports)
 *   mgw_allreduce                <- allreduce_net.py:370-411  (ring_allreduce; same per-
 *                                   element fold order)
 *   mgw_comm_error               <- allreduce_net.py:309-357  (frame/header validation ->
 *                                   ProtocolError; here a device error word)
 *   mgw_unpack                   <- (no reference counterpart: the reference verifies the
 *                                   reduced buffer in place, allreduce_net.py:556)
 *   mgw_sched_*                  <- allreduce_net.py:463-578  (run_emulation: compute agent
 *                                   thread + queue -> compute stream + comm stream)
 *   mgw_check_const              <- allreduce_net.py:556      (np.array_equal verification)
 */
#ifndef MGWFBP_B200_H
#define MGWFBP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGW_OK 0
#define MGW_EINVAL 1
#define MGW_EPROTO 2
#define MGW_ECUDA 3

#define MGW_MAX_RANKS 8
#define MGW_IPC_HANDLE_BYTES 64

/* device error word values (mgw_comm_error) */
#define MGW_DEV_OK 0
#define MGW_DEV_MISMATCH 1        /* ranks disagree on the collective: bucket length, kernel,
                                     grid, dtype, scale or group tag (allreduce_net.py:340-345) */
#define MGW_DEV_LENGTH_MISMATCH MGW_DEV_MISMATCH /* round-1 name */
#define MGW_DEV_TIMEOUT 2         /* a peer never arrived at the barrier */
#define MGW_DEV_PEER_ABORT 3      /* a peer detected an error and aborted */

/* all-reduce algorithm selection */
#define MGW_ALGO_AUTO 0
#define MGW_ALGO_ONESHOT 1
#define MGW_ALGO_TWOSHOT 2
#define MGW_ALGO_LL 3 /* push-based low-latency one-shot (fused path only, <= 262,144 elements) */
#define MGW_ALGO_NVLS 4 /* NVSwitch in-switch reduction (opt-in; fp32 sum, NOT the reference fold order) */
#define MGW_ALGO_PUSH 5 /* push-based two-shot (fused path only): every NVLink byte is a store */
#define MGW_ALGO_PUSH_ONESHOT 6 /* push-based one-shot (fused path only): stores out, local fold */
#define MGW_ALGO_PUSH_PIPE 7 /* pipelined push two-shot (fused path only): per-sub-chunk flags overlap the phases */
#define MGW_ALGO_LL128 8 /* flag-in-line two-shot (fused fp32 and bf16 paths): 128-B lines of 120 B payload + flag, no barrier */
#define MGW_ALGO_LL128_ONESHOT 9 /* flag-in-line one-shot (fused paths): the whole bucket to every rank in 128-B lines, one hop */

/* schedule flags */
#define MGW_SCHED_FILL 1u  /* "backward" writes fill_values into each layer before its deadline */
#define MGW_SCHED_GRAPH 2u /* capture the iteration once into a CUDA graph and replay it */
#define MGW_SCHED_HOSTIO 4u /* e2e: H2D of each layer from host_src, D2H of the result to host_dst */
#define MGW_SCHED_FUSED 8u  /* one kernel per group: pack + all-reduce + unpack (N > 1) */
#define MGW_SCHED_PDL 16u   /* the group's exchange launches while its fill runs (programmatic event) */
#define MGW_SCHED_BF16 32u  /* rows are bf16 tensors (counts in bf16 elements): bf16 fill, bf16 group
                               exchange with fp32 accumulation (mgw_allreduce_fused_bf16), always fused */

typedef struct mgw_comm mgw_comm;
typedef struct mgw_sched mgw_sched;

/* One layer tensor inside a bucket: `count` fp32 elements at `ptr` (device, or
 * pinned host for host_src/host_dst) occupying bucket elements
 * [offset, offset + count). */
typedef struct {
  float* ptr;
  int64_t count;
  int64_t offset;
} mgw_tensor_desc;

/* One merge group of a schedule, given in send order (descending layer index). */
typedef struct {
  int32_t head_layer; /* lowest layer of the group: the sender (merge_planner.py:67-84) */
  int32_t desc_begin; /* first row of the schedule's descriptor table for this group */
  int32_t desc_count; /* rows belonging to this group (layers high..low) */
  int32_t algo;       /* MGW_ALGO_* */
  int64_t n_elem;     /* bucket elements = sum of the group's layer params */
  int64_t ready_ns;   /* tau_b[head] + t_b[head]: when the head's gradient exists (ns from
                         iteration start, schedule_sim.py:103-127) */
} mgw_group;

/* ---- library ---------------------------------------------------------- */
const char* mgw_version(void);
int mgw_last_error(char* buf, size_t len);
int mgw_device_count(int* out);

/* ---- K5: simulated backward ------------------------------------------- */
int mgw_spin_ns(int64_t ns, void* stream);

/* ---- K1 pack+scale / K4 unpack ---------------------------------------- */
/* A descriptor table handle: rows (layer `high` first) must tile [0, extent)
 * contiguously; the handle keeps a device copy and a host mirror. */
int mgw_desc_upload(const mgw_tensor_desc* rows, int n, void** table);
int mgw_desc_free(void* table);
int mgw_pack(const void* dev_table, int n, float* bucket, int64_t bucket_elems, float scale, void* stream);
int mgw_unpack(const void* dev_table, int n, const float* bucket, int64_t bucket_elems, void* stream);
int mgw_fill_const(const void* dev_table, int n, const float* values_dev, void* stream);
int mgw_check_const(const void* dev_table, int n, const float* values_dev, int64_t* mismatches, void* stream);

/* ---- communicator: CUDA-IPC peer buckets over NVLink/NVSwitch --------- */
int mgw_comm_create(int rank, int world, int device, int64_t capacity_bytes, mgw_comm** out,
                    uint8_t* ipc_handle_out);
int mgw_comm_open_peers(mgw_comm* comm, const uint8_t* handles /* world * 64 bytes */);
int mgw_comm_destroy(mgw_comm* comm);
int mgw_comm_set_timeout_ms(mgw_comm* comm, int64_t ms);
int mgw_comm_set_oneshot_max(mgw_comm* comm, int64_t bytes);
int mgw_comm_set_max_ctas(mgw_comm* comm, int ctas);
int mgw_comm_set_ll_max(mgw_comm* comm, int64_t bytes);
/* gate: precede every collective with a one-warp kernel that waits until all peers
 * have reached the same collective (the reference ring's blocking receive,
 * allreduce_net.py:277-307), so overlapped bulk kernels never hold SMs in a barrier
 * while a peer is still computing.  Off by default. */
int mgw_comm_set_gate(mgw_comm* comm, int enable);
/* tuning: key 0 = one-shot 16-B slots per CTA, key 1 = two-shot slots per CTA (0 = default) */
int mgw_comm_set_tuning(mgw_comm* comm, int key, int64_t value);
/* group tag: folded (with length, kernel, grid, dtype and scale) into the 32-bit tag every
 * barrier flag and LL header carries, so ranks issuing different groups, iterations or
 * per-rank settings raise MGW_DEV_MISMATCH instead of reducing unrelated buckets
 * (the reference's frame header check, allreduce_net.py:340-345).  Sticky until changed;
 * the Algorithm-2 engine tags every group with its head layer. */
int mgw_comm_set_group_tag(mgw_comm* comm, uint32_t tag);
/* the algorithm a fused group exchange of n_elem elements of element_bytes (4: fp32, 2: bf16)
 * runs under AUTO on this communicator, fallbacks included (TransportCounters accounting) */
int mgw_comm_pick_algo(mgw_comm* comm, int64_t n_elem, int element_bytes, int* algo);
/* clear the device error word and this rank's abort flag after a ProtocolError.  Collective
 * in spirit: every rank calls it after a host-level barrier, before the next collective. */
int mgw_comm_clear_error(mgw_comm* comm);
/* In-process rank group on ONE device (tests and single-GPU emulation of the real barrier
 * protocol): `world` communicators whose peer tables point at each other's regions directly
 * (no IPC).  Their collectives run through mgw_group_allreduce_fused; the CTA cap defaults
 * to 2 * 148 / world so all ranks' grids fit one co-resident cooperative launch. */
int mgw_comm_create_local(int world, int device, int64_t capacity_bytes, mgw_comm** comms /* world */);
/* Every rank of such a group runs its fused group exchange (rows in tables[r], n_elem[r]
 * elements, scale[r]; element_bytes 4 = fp32, 2 = bf16) in ONE cooperative launch on
 * `stream`: arguments, algorithm, grid and tag come from each rank's own communicator as
 * in mgw_allreduce_fused[_bf16], so the real barrier / LL / push protocol -- and any
 * disagreement between the ranks -- runs between co-resident CTAs (kernels that wait on
 * one another are never separate launches on one device).  n_elem[r] < 0: rank r is
 * absent.  Afterwards read each rank's outcome with mgw_comm_error. */
int mgw_group_allreduce_fused(mgw_comm* const* comms, void* const* tables, const int64_t* n_elem, const float* scale,
                              int world, int algo, int element_bytes, void* stream);
/* process-wide options (A/B runs): MGW_OPT_ROWS_PATH 0 = auto (TMA bulk copies for
 * pack / unpack of large buckets with 16-B aligned rows), 1 = LDG kernel only, 2 = bulk
 * wherever the alignment allows */
#define MGW_OPT_ROWS_PATH 1
#define MGW_OPT_PIPE_SUB_SLOTS 2 /* pipelined two-shot: 16-B slots per sub-chunk per part (default 512) */
#define MGW_OPT_LOCAL_MIN_SLOTS 3 /* single-rank group kernel: minimum 16-B slots per CTA (128..2048) */
#define MGW_OPT_WIDE_MIN_BYTES 4  /* push two-shot over IPC: buckets >= this many bytes launch 512 CTAs
                                     (default 112 MiB, 0 = always the comm's CTA cap) */
int mgw_set_option(int key, int64_t value);
/* bounds-checked build (-DMGW_CHECKED, libmgwfbp_b200_checked.so): index violations the
 * kernels counted since the last reset (every row walk, bucket / slot / LL / push index and
 * flag slot is validated); *checked = 0 in the production build (total always 0) */
int mgw_checked_violations(int reset, uint64_t* total, int* checked);
/* the 32-bit collective tag the launchers stamp into barrier flags / LL headers
 * (kind: 1..11, see TagKind in csrc/allreduce.cuh) -- exposed for host-side tests */
int mgw_debug_collective_tag(uint32_t group_tag, int64_t n_elem, int kind, int grid, float scale, uint32_t* out);
int mgw_comm_input(mgw_comm* comm, float** slot); /* slot the next collective reads (syncs) */
int mgw_comm_result(mgw_comm* comm, float** result);
int mgw_comm_pack(mgw_comm* comm, const void* dev_table, int n, int64_t n_elem, float scale, void* stream);
int mgw_allreduce(mgw_comm* comm, int64_t n_elem, int algo, void* stream);
/* pack -> all-reduce -> unpack of one group in one kernel, in place on the layer tensors */
int mgw_allreduce_fused(mgw_comm* comm, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                        void* stream);
int mgw_comm_error(mgw_comm* comm, int* code);
int mgw_comm_calls(mgw_comm* comm, int64_t* calls);

/* Device seconds per step of `reps` back-to-back exchange steps under one event pair
 * (the (a, b) fit's input and the bus-bandwidth sweep).  kind: 0 pack+all-reduce+unpack,
 * 1 all-reduce only, 2 pack only, 3 unpack only, 4 fused kernel, 5 fused bf16 kernel
 * (n_elem bf16 elements), 6 peer rendezvous only (gate kernel).  comm NULL: single rank.
 * kind | MGW_TIME_GRAPH: the reps are captured into one CUDA graph and replayed (the
 * per-launch cost inside the Algorithm-2 engine's graph). */
#define MGW_TIME_GRAPH 256
int mgw_time_exchange(mgw_comm* comm, const void* dev_table, int n_rows, int64_t n_elem, float* local_bucket,
                      int algo, int kind, int reps, int warmups, double* seconds_per_rep, void* stream);

/* Self-timed phases of `reps` fused group exchanges (ncu cannot replay a multi-rank
 * kernel): out[r * 8 + k], %globaltimer ns -- k = 0 first-CTA entry, 1 last-CTA exit,
 * 2.. CTA 0's phase boundaries (entry, after pack/push, after barrier, after reduce,
 * [after 2nd barrier, after unpack]); unused entries are 0.  Collective. */
int mgw_probe_phases(mgw_comm* comm, const void* table, int n_rows, int64_t n_elem, int algo, int reps,
                     uint64_t* out, void* stream);

/* ---- emulated ranks on one device (test path; no barriers) ------------ */
int mgw_allreduce_emulated(float* const* ins, float* const* outs, int world, int64_t n_elem, int algo,
                           void* stream);

/* ---- NVLS (opt-in): one multicast object per communicator --------------
 * rank 0 mgw_nvls_create -> pass the fd (SCM_RIGHTS) -> others mgw_nvls_import ->
 * all mgw_nvls_add_device -> barrier -> all mgw_nvls_bind -> barrier */
int mgw_nvls_supported(int device, int* ok);
int mgw_nvls_create(mgw_comm* comm, int64_t bytes, int* fd_out);
int mgw_nvls_import(mgw_comm* comm, int fd, int64_t bytes);
int mgw_nvls_add_device(mgw_comm* comm);
int mgw_nvls_bind(mgw_comm* comm);
int mgw_comm_set_nvls_min(mgw_comm* comm, int64_t bytes);

/* autograd hook path: record `event` on compute_stream, make comm_stream wait on it, then
 * mgw_allreduce_fused on comm_stream -- one call per ready merge group */
int mgw_group_launch(mgw_comm* comm, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                     void* compute_stream, void* comm_stream, void* event);
int mgw_event_create(void** event);
int mgw_event_destroy(void* event);
int mgw_allreduce_fused_emulated(void* const* tables, float* const* slots, int world, int64_t n_elem, float scale,
                                 int algo, void* stream);

/* ---- bf16 gradients, fp32 accumulation ------------------
 * Same tables (rows' ptr point at bf16 data; count / offset in bf16 elements), bf16
 * bucket and wire format.  Element e of reference segment s (allreduce_net.py:360-367)
 * becomes bf16_rn((((f32(x_s) + f32(x_s+1)) + ...) + f32(x_s+N-1)) * scale), the
 * multiply only when scale != 1: the reference ring's fold order (allreduce_net.py:401)
 * in fp32 over exactly-upcast inputs, rounded once.  Algorithms: AUTO, LL (<= 2 MB of bf16,
 * two bf16 per pushed word), one-shot, two-shot.  Replaces ring_allreduce (allreduce_net.py:370-411) for element_bytes = 2
 * profiles (model_profile.py:24). */
int mgw_allreduce_fused_bf16(mgw_comm* comm, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                             void* stream);
int mgw_group_launch_bf16(mgw_comm* comm, const void* table, int n_rows, int64_t n_elem, float scale, int algo,
                          void* compute_stream, void* comm_stream, void* event);
int mgw_allreduce_fused_bf16_emulated(void* const* tables, void* const* slots, int world, int64_t n_elem,
                                      float scale, int algo, void* stream);

/* ---- Algorithm 2 on streams ------------------------------------------- */
int mgw_sched_create(mgw_comm* comm /* NULL: single rank */, const mgw_tensor_desc* rows, int n_rows,
                     const mgw_group* groups, int n_groups, float scale, uint32_t flags,
                     const float* fill_values /* per row, or NULL */, float* const* host_src /* per row */,
                     float* const* host_dst /* per row */, mgw_sched** out);
int mgw_sched_run(mgw_sched* sched, void* compute_stream, void* comm_stream);
int mgw_sched_times(mgw_sched* sched, double* t_iter_s, double* compute_s, double* group_comm_s);
/* per-group kernel execution spans of the last iteration, from %globaltimer stamps the
 * kernels write themselves (first CTA entry .. last CTA exit) */
int mgw_sched_kernel_times(mgw_sched* sched, double* pack_s, double* allreduce_s, double* unpack_s);
/* measured schedule of the last iteration, seconds from its clock mark (the simulated
 * backward's time origin, schedule_sim.py:103-127): per group, when its gradients were
 * produced (end of its fill kernel; -1 without MGW_SCHED_FILL) and its exchange window
 * (first kernel entry .. last kernel exit) -- the rows of a measured Timeline (Timeline.events) */
int mgw_sched_events(mgw_sched* sched, double* ready_s, double* comm_start_s, double* comm_end_s);
int mgw_sched_launches(mgw_sched* sched, int* kernels_per_iteration);
int mgw_sched_destroy(mgw_sched* sched);

#ifdef __cplusplus
}
#endif

#endif /* MGWFBP_B200_H */
