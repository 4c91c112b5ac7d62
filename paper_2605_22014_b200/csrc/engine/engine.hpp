// Device reshard engine: shard stores over global device slots (a slot is
// one GPU of the job; this process drives a contiguous range of them), plan
// compilation into per-device work lists, and execution.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <set>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "desc.h"
#include "reshard_b200/reshard.hpp"
#include "rs_reshard.h"

namespace rsb {

struct DomainError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct IntegrityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SystemError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

// Device allocation owned by the engine.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(int device, std::size_t bytes);
  ~DeviceBuffer();
  DeviceBuffer(DeviceBuffer&& o) noexcept { *this = std::move(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  char* data() const { return ptr_; }
  std::size_t size() const { return bytes_; }
  void upload(const void* host, std::size_t bytes, cudaStream_t s);

 private:
  int device_ = -1;
  char* ptr_ = nullptr;
  std::size_t bytes_ = 0;
};

// A peer arena mapped into this process through CUDA IPC.
class ImportedArena {
 public:
  ImportedArena() = default;
  ImportedArena(int device, const cudaIpcMemHandle_t& h);
  ~ImportedArena();
  ImportedArena(ImportedArena&& o) noexcept { *this = std::move(o); }
  ImportedArena& operator=(ImportedArena&& o) noexcept;
  char* data() const { return ptr_; }

 private:
  int device_ = -1;
  char* ptr_ = nullptr;
};

struct Entry {
  std::uint32_t ti = 0;
  int rank = 0;
  int slot = 0;            // global device slot holding the buffer
  reshard::ShardView view;
  std::int64_t nbytes = 0;
  // flat-bucket shards (reshard::bucket_range): the buffer holds the element
  // range [flat_lo, flat_lo + nbytes / eb) of the view's row-major order, so
  // view-relative addressing starts flat_off = flat_lo * eb bytes before ptr
  bool flat = false;
  std::int64_t flat_lo = 0, flat_off = 0, flat_elems = 0;
  std::size_t off = 0;     // offset in the slot's engine arena (rs_store_alloc)
  char* ptr = nullptr;     // local, peer-mapped (IPC) or caller-bound address
};

struct Store {
  bool laid_out = false;
  reshard::ModelSpec model;
  reshard::ParallelConfig config;
  std::vector<Entry> entries;  // (tensor, ascending rank)
  std::unordered_map<std::uint64_t, std::uint32_t> index;
  std::vector<std::size_t> arena_bytes;            // per slot
  std::vector<DeviceBuffer> arenas;                // per local device
  std::vector<std::unique_ptr<ImportedArena>> imported;  // per slot
  const Entry* find(int rank, std::uint32_t ti) const;
  Entry* find(int rank, std::uint32_t ti);
  std::int64_t total_bytes() const;
};

struct LayerRange {
  int layer;
  std::uint64_t item_begin, item_end;  // copy items of this layer (per device)
};

// Per local device compiled work.
struct DeviceProgram {
  std::vector<rs_copy_desc> local;  // DIRECT copies executed here
  std::vector<std::uint64_t> local_item0;
  std::uint64_t local_items = 0;
  std::vector<LayerRange> layers;
  // STAGED
  std::vector<rs_lane_desc> lanes;  // ntx sender lanes then nrx receiver lanes
  int ntx = 0, nrx = 0;
  std::vector<rs_batch_desc> batches;
  std::vector<rs_copy_desc> frames;
  DeviceBuffer d_local, d_item0, d_lanes, d_batches, d_frames, d_error, d_trace;
  // STAGED strict layers: [arrival counters: nlayers][role ticket][release flag][done_all: nslots ptrs]
  // [layer item ends][stream lanes: per-layer expected arrivals, role table (u32)]
  DeviceBuffer d_sync;
  rs_layer_sync layer_sync{};
  int strict_local_ctas = 0;   // stream lanes, strict: local-copy CTAs of the lane launch
  int strict_max_active = 0;   // stream lanes, strict: most lane CTAs active in one layer
  std::uint64_t local_bytes = 0;
  bool all_aligned = true;  // every local descriptor is 16 B aligned (bulk-copy eligible)
  std::uint64_t launch_bytes = 0;  // bytes of the largest single copy launch (grid / item sizing)
  std::uint64_t max_row_bytes = 0; // longest contiguous run (TMA-NP items must fit shared memory)
  bool peer_stores = false;        // some descriptor writes another slot's memory (NVLink peer / IPC)
  bool stream_lanes = false;       // STAGED: this device's lanes run rs_stream_lane_kernel
};

struct Device {
  int ordinal = 0;
  int slot = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;              // reshard kernels
  cudaStream_t h2d = nullptr, d2h = nullptr;  // host-store copies (rs_execute_host)
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  cudaEvent_t ev_call = nullptr;  // rs_switch: the moment the switch was requested
  cudaStream_t aux = nullptr;     // STAGED stream lanes: the local copies beside the lane kernel
  cudaEvent_t ev_aux = nullptr;
};

class Engine {
 public:
  explicit Engine(const rs_engine_options& opts);
  ~Engine();

  void layout(int which, const reshard::ModelSpec& model, const reshard::ParallelConfig& cfg,
              const std::vector<int>& rank_slot);
  void alloc(int which);
  void free_store(int which);
  void bind(int which, int rank, std::uint32_t ti, void* ptr, std::int64_t nbytes);
  const Store& store(int which) const { return stores_[which]; }
  Store& store(int which) { return stores_[which]; }

  void comm_alloc();                                      // B per dst rank
  void comm_alloc_plan(const reshard::TransferPlan& plan);  // exactly this plan's rings
  // Layer window for host-resident stores: only `layers` layers' source and
  // destination shards live on each local device at a time (slot l % layers),
  // bounding device memory like the reference's per-layer staging.
  void set_window(int layers);
  int window_layers() const { return window_layers_; }
  std::int64_t export_arena(int which, int slot, void* handle) const;
  void import_arena(int which, int slot, const void* handle, std::int64_t bytes);

  void fill_pattern(int which, std::uint64_t seed);
  std::int64_t verify_pattern(int which, std::uint64_t seed, std::int64_t* first_bad);

  void prepare(const reshard::TransferPlan& plan, std::uint64_t plan_id = 0);
  bool prepared_for(std::uint64_t plan_id) const { return prepared_ && plan_id && plan_id == prepared_id_; }
  rs_exec_report run();
  rs_exec_report run_host(void* const* host_src, void* const* host_dst, int window_layers);
  // Live-handoff Switch step (rs_switch): drain -> transfer -> swap.
  rs_switch_stats switch_step(void* const* drain_events, bool swap);
  void swap_stores();
  std::vector<rs_trace_record> trace(int dev) const;  // STAGED transport trace of the last run

  int num_devices() const { return static_cast<int>(devices_.size()); }
  int num_slots() const { return nslots_; }
  int local_of(int slot) const;  // local device index of a slot, -1 if remote

  // RS_MODE_XFER (engine_xfer.cpp): host-driven point-to-point transport --
  // the comparator path.  Per round, our kernels pack each cross-GPU link's
  // chunks into a send buffer, the caller moves the buffers (NCCL
  // send/recv), our kernels unpack the receive buffers.
  struct XferLink {
    int peer_slot = 0;
    int src_rank = 0, dst_rank = 0;
    char* buf = nullptr;
    std::uint64_t buf_bytes = 0;
    std::vector<std::uint64_t> round_bytes;
  };
  int xfer_rounds() const { return xfer_rounds_; }
  const std::vector<XferLink>& xfer_links(int dir) const { return dir ? xfer_rx_ : xfer_tx_; }
  void xfer_step(int what, int round);  // 0 local copies, 1 pack round, 2 unpack round (| RS_XFER_ASYNC)
  void* xfer_stream() const;            // the stream xfer steps run on (cudaStream_t)

 private:
  void compile_xfer(const reshard::TransferPlan& plan);
  struct XferRound {
    std::uint64_t pack_begin = 0, pack_end = 0, unpack_begin = 0, unpack_end = 0;  // item ranges
  };
  int xfer_rounds_ = 0;
  std::vector<XferLink> xfer_tx_, xfer_rx_;  // this process's links (single local device)
  std::vector<XferRound> xfer_round_items_;
  std::vector<rs_copy_desc> xfer_descs_;
  DeviceBuffer xfer_buffers_, d_xfer_descs_, d_xfer_item0_;
  std::int64_t pattern_pass(int which, std::uint64_t seed, bool verify, std::int64_t* first_bad);
  void copy_runs(const Store& s, const std::vector<std::size_t>& idx, void* const* host, bool to_device);
  void compile_direct(const reshard::TransferPlan& plan);
  void compile_staged(const reshard::TransferPlan& plan);
  // A ring link: (source rank, first destination rank, relay route or -1).
  // Route r's lanes carry src -> chain[0] and are forwarded hop by hop.
  using LaneKey = std::tuple<int, int, int>;
  struct RingGeometry {
    std::map<LaneKey, int> lanes_of;                 // link -> lanes
    // relay chains (rs_engine_options.relay): (layer, task index) -> (route, hop)
    std::map<std::pair<int, std::size_t>, std::pair<int, int>> relay_of;
    std::vector<std::vector<int>> route_chain;       // route -> destination ranks in hop order
    std::vector<std::uint64_t> route_slot_bytes;     // route -> ring slot bytes on every hop
    std::vector<int> route_k;                        // route -> ring depth on every hop
    std::map<int, std::uint64_t> inbound_lanes;      // dst rank -> lanes into it
    std::map<int, std::uint64_t> slot_bytes_of;      // dst rank -> ring slot bytes
    std::map<int, std::uint64_t> ring_bytes_of;      // dst rank -> bytes of all its rings
    std::map<int, int> k_of;                         // dst rank -> ring depth (K, or 1 for a tiny B)
    std::set<int> direct_dst;                        // dst ranks whose B cannot hold a ring: direct stores
    bool stream = false;                             // lanes run rs_stream_lane_kernel (stream_lanes_for)
  };
  RingGeometry ring_geometry(const reshard::TransferPlan& plan) const;
  // STAGED: does this cross-rank task go through a ring (else a direct copy)?
  bool ringed(const reshard::TransferTask& t) const;
  int same_slot_policy() const;  // resolved ring_same_slot: 1 rings, 2 direct copies
  bool stream_lanes_for(const reshard::TransferPlan& plan) const;  // STAGED: TMA stream lanes run this plan
  int lane_capacity(int dev, bool stream) const;  // co-resident lane CTAs of the lane kernel
  int run_stream_lanes(std::size_t dev);  // enqueue the stream-lane launch + local copies; returns launches
  void describe_run(rs_exec_report& rep) const;  // which kernels / policy the run used
  void upload_layer_sync(std::size_t dev);         // STAGED strict layers: barrier state of a device
  char* layer_done_flag(int slot) const;           // a slot's layer-done flag in its comm arena
  struct CommLayout {
    std::vector<std::map<int, std::pair<std::size_t, std::size_t>>> regions;  // per slot: rank -> (offset, bytes)
    std::vector<std::size_t> slot_bytes;                                      // per slot, incl. flags
  };
  CommLayout make_comm_layout(const std::map<int, std::uint64_t>* ring_bytes) const;
  void alloc_comm_arenas();
  int ce_copies(const std::vector<rs_copy_desc>& descs, std::uint64_t b, std::uint64_t e, cudaStream_t stream);
  void upload_programs();
  int grid_for(int dev, int which_kernel) const;
  int exchange_kernel_id() const {  // occupancy query id (exchange_max_blocks_per_sm)
    const int l2 = opts_.ring_discard == 0 ? 5 : opts_.ring_discard;
    if ((l2 & 24) == 24 && opts_.ring_cta_threads == 256) return 9;  // TMA lanes: shared memory bounds residency
    const int base = opts_.ring_cta_threads == 1024 ? 2 : opts_.ring_cta_threads == 512 ? 1 : 0;
    if (l2 & 8) return 10 + base;
    return base == 2 ? 8 : base == 1 ? 7 : 2;
  }
  int copy_variant(int dev) const;
  int copy_grid(int dev) const;
  void check_laid_out() const;
  std::size_t comm_bytes(int slot) const;
  char* comm_base(int slot) const;

  rs_engine_options opts_{};
  int nslots_ = 1;
  int first_local_ = 0;
  std::vector<Device> devices_;
  Store stores_[2];
  std::vector<DeviceProgram> programs_;
  std::vector<DeviceBuffer> comm_;                        // per local device
  CommLayout comm_layout_;                                // layout of the comm arenas, every slot
  bool comm_layout_valid_ = false;
  std::vector<std::unique_ptr<ImportedArena>> comm_imported_;  // per slot
  std::vector<std::size_t> comm_imported_bytes_;               // per slot
  int window_layers_ = 0;
  std::vector<DeviceBuffer> window_;  // per local device: window_layers_ layer slots
  bool prepared_ = false;
  std::uint64_t prepared_id_ = 0;  // rs_plan identity of the compiled program (0: none)
  std::uint64_t epoch_ = 0;
  rs_exec_report planned_{};  // compile-time report fields (reference semantics)
  std::int64_t planned_total_bytes_ = 0;
  std::vector<int> plan_layers_;
  int relay_routes_ = 0;  // STAGED relay routes of the compiled plan
};

}  // namespace rsb
