/*
 * rs_reshard.h -- C ABI of the B200-native live-handoff reshard path
 * (libreshard_b200.so).  Plain pointers and sizes only; no exceptions cross
 * it.  Status codes mirror the SPEC exit classes:
 *   RS_OK 0, RS_EDOMAIN 1 (validation / bad argument),
 *   RS_EINTEGRITY 2 (plan or data integrity), RS_ESYSTEM 3 (CUDA / system).
 * rs_last_error() returns the calling thread's last message.
 *
 * Entry points and the reference interface each one replaces:
 *   rs_plan_compute    compute_transfer_plan   proj/include/reshard/planner.hpp:35-38
 *   rs_plan_verify     verify_plan             proj/include/reshard/planner.hpp:44-47
 *   rs_plan_write      write_plan              proj/include/reshard/transfer_plan.hpp:81
 *   rs_plan_read       read_plan               proj/include/reshard/transfer_plan.hpp:82
 *   rs_plan_summary    plan_cost_summary       proj/include/reshard/transfer_plan.hpp:77
 *   rs_plan_placement  (extension) rank-list search over compute_transfer_plan
 *   rs_validate_config validate_config         proj/include/reshard/parallel_config.hpp:73-74
 *   rs_view            view / tp_block         proj/include/reshard/topology.hpp:20-25
 *   rs_chunk_bounds    chunk_bounds            proj/include/reshard/executor.hpp:43-44
 *   rs_engine_create   Transport (+ staging B) proj/include/reshard/transport.hpp:25-48
 *   rs_store_*         ShardStore              proj/include/reshard/shard_store.hpp:19-47
 *   rs_fill_pattern    ShardStore::fill_pattern proj/include/reshard/shard_store.hpp:34
 *   rs_verify_pattern  gather-reslice oracle compare (SPEC.md cmd_verify)
 *   rs_execute         execute_plan            proj/include/reshard/executor.hpp:50-53
 *   rs_execute_host    execute_plan on host ShardStore buffers (H2D/D2H inside)
 *   rs_switch          GenerationMachine::run_switch + atomic_switch, executed
 *                      (proj/src/generation.cpp:239-290) instead of priced
 *   rs_trace_read      RecordingTransport          proj/include/reshard/transport.hpp:50-75
 *   rs_comm_alloc*, rs_arena_*  the staging buffers + NCCL/TCPStore bootstrap of the
 *                      paper's executor, as CUDA-IPC peer arenas
 *   rs_xfer_*          the paper's NCCL isend/irecv executor,
 *                      kept as a measured comparator
 */
#ifndef RS_RESHARD_H
#define RS_RESHARD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_OK 0
#define RS_EDOMAIN 1
#define RS_EINTEGRITY 2
#define RS_ESYSTEM 3

#define RS_SRC 0 /* store of the source configuration C_old */
#define RS_DST 1 /* store of the destination configuration C_new */

#define RS_MODE_DIRECT 0 /* every byte moved straight src -> dst (peer stores), zero staging */
#define RS_MODE_STAGED 1 /* remote frames through bounded per-link staging rings */
#define RS_MODE_XFER 2   /* comparator: kernels pack/unpack, the caller moves bytes (NCCL) */

typedef struct rs_plan rs_plan;
typedef struct rs_engine rs_engine;

typedef struct {
  uint64_t generation_id;
  int32_t tp, pp, dp;
  int32_t num_ranks;
  const int32_t* ranks;       /* ordered rank ids (placement is semantic) */
  const int32_t* layer_stage; /* num_layers entries, or NULL: default ceil split */
  int32_t distributed_optimizer; /* extension: DP-shard the tensors with a dp_shard_axis (ZeRO-1):
                                    0 off, 1 per-tensor dim chunks of the TP block, 2 Megatron
                                    flat buckets (the rank holds a contiguous element range of its
                                    TP block, rs_view_range; reshard::bucket_range) */
  int32_t dist_opt_bucket_elems; /* flat buckets: bucket size in elements (0: max(40M, 1M x dp)) */
} rs_config;

typedef struct {
  int32_t balance_sources;
} rs_plan_options;

typedef struct {
  int64_t total_bytes;     /* remote + local task bytes (TransferPlan::total_bytes) */
  int64_t max_link_bytes;  /* max over remote (src,dst) links */
  int64_t task_count;
  int64_t remote_bytes;
  int64_t local_bytes;
  int64_t carryover_bytes;
  int64_t carryover_count;
  int64_t pairs_checked;
  int32_t num_tensors;
  int32_t num_layers_with_work;
} rs_plan_summary_t;

typedef struct {
  int32_t num_devices;      /* CUDA ordinals this process drives */
  const int32_t* device_ids;
  int64_t staging_bytes;    /* per-destination-rank staging budget B */
  int32_t mode;             /* RS_MODE_* */
  int32_t slots_per_link;   /* ring depth K (>= 2; 0: default 2), STAGED */
  int32_t lanes_per_link;   /* parallel rings per (src,dst) link, STAGED */
  int32_t strict_layers;    /* 1: layer barriers (DIRECT: one launch per layer; STAGED: a device-wide
                               barrier after each layer, the local copies run inside the lane
                               launch; stream-lane CTAs meet only the barriers of their lane's
                               layer range), 0: fused */
  int64_t item_bytes;       /* work-item granularity of the copy engine (0: default) */
  int32_t blocks_per_sm;    /* 0: occupancy maximum */
  int32_t copy_kernel;      /* RS_COPY_*: LDG/STG warp engine or TMA bulk-copy ring */
  int32_t world_slots;      /* device slots in the whole job (0: = num_devices) */
  int32_t first_local_slot; /* slots [first, first+num_devices) are driven by this process */
  int64_t spin_limit;       /* ring flag polls before a wait fails (0: default ~10 s) */
  int32_t fault_inject;     /* test hook: 1 = ring receivers drop out (peer failure) */
  int32_t ring_slot_kib;    /* STAGED: cap on one ring slot in KiB (0: default 64 stream / 128 classic, -1: no cap,
                               slot = B / (inbound lanes x K)); B stays the upper bound */
  int32_t ring_discard;     /* STAGED ring mode bit flags (0 = default 1|4; 2 = none):
                               1 receivers drop drained slot lines (discard.global.L2);
                               4 L2 policies (shards evict-first, slots evict-last);
                               8 warp-specialised lanes (control-warp event loop);
                               16 (with 8, 256-thread lanes) TMA bulk copies in the copy warps */
  int32_t ring_cta_threads; /* STAGED: threads per ring-lane CTA, 256 / 512 / 1024 (0: default) */
  int32_t trace;            /* STAGED: 1 = record a per-batch transport trace (rs_trace_read) */
  int32_t ring_same_slot;   /* STAGED, cross-rank tasks whose ranks share a GPU: 0 = auto (rings
                               on a one-slot engine -- the transport is what runs -- and direct
                               copies in a multi-slot job), 1 = always rings, 2 = always direct */
  int32_t ring_kernel;      /* STAGED lane kernel: 0 = auto (TMA stream lanes when every frame --
                               and under strict_layers every local copy -- is 16 B aligned with
                               runs <= 16 KB, else classic), 1 = classic
                               register lanes (rs_exchange_kernel), 2 = TMA stream lanes
                               (rs_stream_lane_kernel; falls back to classic when ineligible) */
  int32_t ring_stages;      /* stream lanes: 16 KB shared-memory stages per lane end (0: default 2;
                               1, 2, 3, 4, 6, 8, 10 or 13) */
  int32_t relay;            /* STAGED, multi-slot jobs: 1 = relay chains for DP broadcasts (a box
                               several destination GPUs need from one source leaves the source once;
                               each destination's ring receiver forwards it to the next,
                               reshard::relay_chains); needs stream lanes.  0 = point to point */
} rs_engine_options;

#define RS_COPY_AUTO 0     /* engine default: RS_COPY_TMA_NP when every descriptor is 16 B aligned with
                              runs <= 16 KB and no descriptor stores into another slot, else RS_COPY_LDG8_NP */
#define RS_COPY_LDG4 1     /* warp-per-row 16 B vectors, 4 loads in flight per lane */
#define RS_COPY_LDG8 2     /* same, 8 loads in flight per lane, persistent grid (3 CTAs/SM) */
#define RS_COPY_BULK 3     /* cp.async.bulk global->smem->global ring, one issuer per CTA */
#define RS_COPY_LDG4_CS 4  /* LDG4 with evict-first (st.global.cs) stores */
#define RS_COPY_LDG8_CS 5  /* LDG8 with evict-first (st.global.cs) stores */
#define RS_COPY_LDG16 6    /* warp engine, 16 loads in flight per lane */
#define RS_COPY_CTA8 7     /* CTA-cooperative items (rows dealt to the CTA's warps), 8 loads/lane */
#define RS_COPY_BULK_MW 8  /* TMA bulk rings, 4 independent issuer warps per SM */
#define RS_COPY_LDG8_PF 13 /* LDG8 with the L2::256B prefetch hint on loads */
#define RS_COPY_LDG8_EF 14 /* LDG8 with an evict-first L2 policy on loads */
#define RS_COPY_LDG8_NP 15 /* LDG8, non-persistent grid (one work item per warp) */
#define RS_COPY_TMA_NP 17  /* TMA bulk copy (cp.async.bulk), one 1-warp CTA per 16 KB item, non-persistent */
#define RS_COPY_TMA_NP32 18 /* same with 32 KB items */
#define RS_COPY_CE 16      /* comparator: copy engines (one cudaMemcpy2DAsync per descriptor row
                              plane), no kernel of ours -- DIRECT mode only */

typedef struct {
  int32_t ok;
  int32_t failed_layer;       /* -1: none */
  int64_t peak_staging_bytes; /* max over destination ranks of resident ring capacity */
  int64_t bytes_moved;        /* remote (cross-rank) task bytes */
  int64_t local_copy_bytes;   /* local task bytes */
  int64_t carryover_bytes;    /* carryover bytes materialised */
  int32_t layers_processed;
  int32_t kernel_launches;
  double device_ms;           /* CUDA-event time of the run on the slowest device */
  double host_ms;             /* host wall time of the call */
  char error[512];
  /* What ran (so a caller / the bench can tell which kernel moved the bytes
   * without assuming it): the RS_COPY_* variant device 0's copy launches
   * resolved to (DIRECT / host path; -1 none), and the STAGED policy for
   * cross-rank tasks whose ranks share a GPU (1 rings, 2 direct, 0 n/a). */
  int32_t copy_kernel;
  int32_t ring_same_slot;
  int32_t ring_kernel;        /* STAGED lane kernel of device 0: 1 classic (rs_exchange_kernel),
                                 2 TMA stream lanes (rs_stream_lane_kernel), 0 n/a */
  int32_t relay_routes;       /* STAGED relay: distinct (source, destination chain) routes forwarded */
} rs_exec_report;

const char* rs_last_error(void);
const char* rs_version(void);

/* ----------------------------------------------------------------- planning */
int rs_validate_config(const char* model_spec, const rs_config* cfg, char* buf, size_t cap,
                       size_t* needed, int32_t* num_violations);
int rs_view(const char* model_spec, const rs_config* cfg, int32_t tensor_index, int32_t rank,
            int64_t* lo, int64_t* hi, int32_t* present);
/* Flat-bucket distributed optimizer (extension): the
 * element range [*lo, *hi) of the rank's TP block (rs_view) it holds, row
 * major; *flat = 0 when the tensor is not flat-bucket sharded under cfg (then
 * the range is the whole view).  A store entry holds exactly these elements. */
int rs_view_range(const char* model_spec, const rs_config* cfg, int32_t tensor_index, int32_t rank, int64_t* lo,
                  int64_t* hi, int32_t* flat);
int rs_plan_compute(const char* model_spec, const rs_config* c_old, const rs_config* c_new,
                    const rs_plan_options* opts, rs_plan** out);
int rs_plan_read(const char* model_spec, const char* plan_text, rs_plan** out);
int rs_plan_write(const rs_plan* plan, char* buf, size_t cap, size_t* needed);
int rs_plan_summary(const rs_plan* plan, rs_plan_summary_t* out);
int rs_plan_verify(const rs_plan* plan, const rs_config* c_old, const rs_config* c_new, char* buf,
                   size_t cap, size_t* needed, int32_t* num_violations);
void rs_plan_destroy(rs_plan* plan);
int rs_chunk_bounds(int32_t ndims, const int64_t* lo, const int64_t* hi, int64_t max_bytes,
                    int64_t bytes_per_element, int64_t* out_lo, int64_t* out_hi, int64_t cap,
                    int64_t* count);

/* ------------------------------------------------------------------- engine */
int rs_engine_create(const rs_engine_options* opts, rs_engine** out);
void rs_engine_destroy(rs_engine* e);

/* Shard stores.  rank_device[i] = engine device slot of cfg->ranks[i]. */
int rs_store_layout(rs_engine* e, int32_t which, const char* model_spec, const rs_config* cfg,
                    const int32_t* rank_device);
int rs_store_alloc(rs_engine* e, int32_t which);      /* one arena per device */
int rs_store_bind(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index, void* dptr,
                  int64_t nbytes);                     /* caller-owned device memory */
int rs_store_ptr(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index, void** dptr,
                 int64_t* nbytes);
int rs_store_bytes(rs_engine* e, int32_t which, int64_t* total);
/* Entries in store order (tensor, ascending rank): up to cap triples. */
int rs_store_entries(rs_engine* e, int32_t which, int32_t* tensor_index, int32_t* rank,
                     int64_t* nbytes, int64_t cap, int64_t* count);
int rs_store_read(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index, int64_t offset,
                  int64_t nbytes, void* host);
int rs_store_write(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index,
                   int64_t offset, int64_t nbytes, const void* host);
int rs_store_free(rs_engine* e, int32_t which);

/* One process per GPU: every process lays out the same stores over the same
 * global slots; each allocates its local slots, exports the arenas
 * (CUDA IPC handle, RS_IPC_HANDLE_BYTES bytes), and imports every peer's.
 * which: RS_SRC, RS_DST or RS_COMM (the staging arena: B per destination rank
 * on the slot + ring flags, allocated by rs_comm_alloc). */
#define RS_COMM 2
#define RS_IPC_HANDLE_BYTES 64
int rs_comm_alloc(rs_engine* e);                           /* B per destination rank */
/* Plan-sized staging: each destination rank's region holds exactly the
 * plan's rings (<= B; ring slots are capped, so usually far less than B).
 * rs_prepare allocates this itself in a single process when the arena is
 * missing or too small; with several processes every process calls it with
 * the same plan before exchanging the RS_COMM handles. */
int rs_comm_alloc_plan(rs_engine* e, const rs_plan* plan);
int rs_arena_export(rs_engine* e, int32_t which, int32_t slot, void* handle, int64_t* arena_bytes);
int rs_arena_import(rs_engine* e, int32_t which, int32_t slot, const void* handle, int64_t arena_bytes);

/* Per-slot traffic of a plan under a placement (host only): egress / ingress
 * of remote task bytes, local task bytes, carryover bytes, out[4*slot + k]. */
int rs_plan_traffic(const rs_plan* plan, const rs_config* c_old, const int32_t* slot_old,
                    const rs_config* c_new, const int32_t* slot_new, int32_t nslots, int64_t* out);
/* Same with flags: RS_TRAFFIC_RELAY counts each relay-chained task (DP
 * broadcast forwarding, rs_engine_options.relay) as egress of the slot that
 * forwards it (reshard::relay_chains), i.e. the traffic a relay run moves. */
#define RS_TRAFFIC_RELAY 1
int rs_plan_traffic_ex(const rs_plan* plan, const rs_config* c_old, const int32_t* slot_old,
                       const rs_config* c_new, const int32_t* slot_new, int32_t nslots, int32_t flags,
                       int64_t* out);

/* Placement-aware destination rank ordering (extension):
 * fills ranks_out[c_new->num_ranks] with the rank list for c_new's shape,
 * drawn from candidates[ncand] (one rank per GPU), that minimises the per-GPU
 * NVLink/HBM roofline of the plan c_old -> c_new; the planner's self-held
 * regions (proj/src/planner.cpp:139-152) make the list decide how many bytes
 * cross links.  out reports the chosen and the given (c_new->ranks) lists. */
typedef struct {
  double nvlink_gbs;        /* 0: 900 (per direction per GPU) */
  double hbm_gbs;           /* 0: 6552 (measured copy peak) */
  int64_t exhaustive_limit; /* 0: 2,000,000 assignments */
  int32_t balance_sources;
  int32_t reserved;
} rs_placement_options;

typedef struct {
  double roofline_ms, given_roofline_ms;
  int64_t remote_bytes, local_bytes, carryover_bytes, max_link_bytes;
  int64_t given_remote_bytes, given_local_bytes, given_carryover_bytes, given_max_link_bytes;
  int64_t evaluated;
  int32_t exhaustive;
  int32_t reserved;
} rs_placement_result;

int rs_plan_placement(const char* model_spec, const rs_config* c_old, const rs_config* c_new,
                      const int32_t* candidates, int32_t ncand, const rs_placement_options* opts,
                      int32_t* ranks_out, rs_placement_result* out);

int rs_fill_pattern(rs_engine* e, int32_t which, uint64_t seed);
int rs_verify_pattern(rs_engine* e, int32_t which, uint64_t seed, int64_t* mismatches,
                      int64_t* first_bad_entry);

/* --------------------------------------------------------------- execution */
int rs_prepare(rs_engine* e, const rs_plan* plan);  /* compile + upload work lists */
int rs_run(rs_engine* e, rs_exec_report* report);   /* launch + wait */
int rs_execute(rs_engine* e, const rs_plan* plan, rs_exec_report* report);

/* Host-resident stores: host_src[k] / host_dst[k] follow the (tensor, ascending
 * rank) entry order of the src / dst layout (rs_store_entries); entries on
 * other processes' slots are ignored.  Each layer's source shards are copied
 * H2D, resharded on the device, and the destination shards copied D2H,
 * pipelined across layers on three streams (DIRECT mode; STAGED copies all in,
 * runs, copies all out).  window_layers == 0: the allocated / bound device
 * stores are used.  window_layers > 0: only that many layers' shards are
 * device-resident at a time (layer l in slot l % window_layers; a slot is
 * refilled after its previous layer's D2H completes) -- device memory is
 * bounded by window_layers x the largest layer, so states larger than HBM
 * stream through one GPU (the reference's per-layer bound). */
int rs_execute_host(rs_engine* e, const rs_plan* plan, void* const* host_src,
                    void* const* host_dst, int32_t window_layers, rs_exec_report* report);

/* ------------------------------------------------------------ live handoff */
/* One Switch step of the dual-world handoff, executed for real: the
 * reference's GenerationMachine::run_switch + atomic_switch
 * (proj/src/generation.cpp:239-290) price drain + transfer + swap with cost
 * model constants (transfer_time_s, cost_model.hpp:48-49); here
 *   drain    = every local reshard stream waits for drain_events[d] (a
 *              cudaEvent_t the training stream recorded at its iteration
 *              boundary on local device d; NULL array or entry = nothing
 *              in flight), device-timed from the call;
 *   transfer = the prepared plan (rs_prepare / rs_execute), device-timed;
 *   swap     = RS_SRC and RS_DST exchange roles (the shadow generation's
 *              store becomes the active one; the old store becomes the next
 *              handoff's destination) -- the pointer swap of atomic_switch.
 * A failed transfer leaves the active store untouched and returns
 * RS_EINTEGRITY with ok = 0 in stats->exec (abort_and_fallback semantics:
 * generation.cpp:315-340).  Multi-process: every process calls rs_switch;
 * the caller's barrier after it is the commit point. */
typedef struct rs_switch_stats {
  double drain_ms;     /* device time from the call until the last drain event fired */
  double transfer_ms;  /* device time of the reshard kernels (max over local devices) */
  double swap_ms;      /* host time of the store swap */
  double pause_ms;     /* drain + transfer + swap (SwitchStats::pause_s) */
  int64_t transfer_bytes;  /* plan.total_bytes() (SwitchStats::transfer_bytes) */
  int32_t swapped;         /* 1 when the stores exchanged roles */
  int32_t reserved;
  rs_exec_report exec;
} rs_switch_stats;

int rs_switch(rs_engine* e, const rs_plan* plan, void* const* drain_events, int32_t swap,
              rs_switch_stats* stats);
/* Exchange the RS_SRC and RS_DST stores (layouts, allocations, bindings,
 * imported peer arenas); the prepared program is dropped. */
int rs_store_swap(rs_engine* e);

/* RS_MODE_XFER (the NCCL send/recv comparator, one local device): after
 * rs_prepare, the caller runs step 0 (local copies) once, then for every
 * round r: step 1 (pack r), moves each tx link's round_bytes[r] from its
 * buffer to the peer's matching rx link buffer (ncclSend/ncclRecv, links in
 * index order on both sides), then step 2 (unpack r).  Steps synchronise the
 * engine stream before returning, unless `what` carries RS_XFER_ASYNC: then
 * the step is only enqueued on the stream rs_xfer_stream returns and the
 * caller orders its NCCL calls against it with events (no host round trip
 * per round).  dir: 0 tx, 1 rx. */
#define RS_XFER_ASYNC 16
int rs_xfer_info(rs_engine* e, int32_t* rounds, int32_t* ntx, int32_t* nrx);
int rs_xfer_link(rs_engine* e, int32_t dir, int32_t index, int32_t* peer_slot, int32_t* src_rank,
                 int32_t* dst_rank, void** buffer, int64_t* buffer_bytes, int64_t* round_bytes);
int rs_xfer_step(rs_engine* e, int32_t what, int32_t round);
int rs_xfer_stream(rs_engine* e, void** stream); /* the engine stream xfer steps run on (cudaStream_t) */

/* Transport trace of the last STAGED run on local device `device` (engine
 * created with trace = 1): the RecordingTransport of the reference
 * (proj/include/reshard/transport.hpp:50-75) on the device -- one record per
 * (batch, role) this device ran, globaltimer nanoseconds. */
typedef struct {
  uint32_t lane;    /* the lane's first batch index */
  uint32_t batch;   /* batch index within the lane */
  uint32_t layer;
  uint32_t role;    /* 0 sender, 1 receiver */
  uint64_t bytes;
  uint64_t t_begin; /* flag acquired */
  uint64_t t_end;   /* flag published */
} rs_trace_record_t;
int rs_trace_read(rs_engine* e, int32_t device, rs_trace_record_t* out, int64_t cap, int64_t* count);

/* Page-locked host memory for host shard stores (full-bandwidth H2D/D2H). */
int rs_host_alloc(size_t bytes, void** out);
int rs_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* RS_RESHARD_H */
