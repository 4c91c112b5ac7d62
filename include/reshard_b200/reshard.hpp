// reshard_b200 -- host C++ API of the B200-native live-handoff reshard path.
//
// Same names, argument meaning and error behaviour as the reference's
// planning surface, so a caller such as GenerationMachine::run_switch
// (proj/src/generation.cpp:242) compiles unchanged against this header:
//   geometry   proj/include/reshard/shard_view.hpp:15-112
//   model      proj/include/reshard/model_spec.hpp:13-87
//   layout     proj/include/reshard/parallel_config.hpp:12-74
//   topology   proj/include/reshard/topology.hpp:20-28
//   plan       proj/include/reshard/transfer_plan.hpp:18-82
//   planner    proj/include/reshard/planner.hpp:14-47
//   chunking   proj/include/reshard/executor.hpp:43-44
//   execution  proj/include/reshard/{executor,shard_store,transport}.hpp
// execute_plan keeps the reference's signature (executor.hpp:50-53) and runs
// the plan on the B200 engine (the same code as rs_execute_host); the
// Transport argument selects the device transport and receives the per-frame
// accounting.  include/reshard/*.hpp forward the reference's header names
// here, so a reference caller compiles unchanged.
//
// Extension over the reference: TensorSpec::element_bytes (0 = the model's
// bytes_per_element) so bf16 params and fp32 master/Adam state share one plan.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <map>
#include <optional>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace reshard {

constexpr int kMaxDims = 8;

struct Interval {
  std::int64_t lo = 0;
  std::int64_t hi = 0;
  std::int64_t length() const { return hi - lo; }
  bool operator==(const Interval&) const = default;
};

// Non-empty half-open hyper-rectangle; fixed capacity, no heap.
class ShardView {
 public:
  ShardView() = default;
  explicit ShardView(const std::vector<Interval>& bounds);  // throws std::invalid_argument
  static ShardView full(const std::vector<std::int64_t>& shape);

  std::size_t ndims() const { return nd_; }
  const Interval& dim(std::size_t i) const;
  std::vector<Interval> bounds() const { return {iv_.begin(), iv_.begin() + nd_}; }
  std::int64_t element_count() const;
  std::vector<std::int64_t> extents() const;
  bool contains(const ShardView& other) const;
  bool contains_point(const std::vector<std::int64_t>& p) const;
  bool operator==(const ShardView& o) const;
  std::string to_string() const;

  // unchecked mutable access for planners that build boxes in place
  Interval& raw(std::size_t i) { return iv_[i]; }
  void set_ndims(std::size_t n) { nd_ = static_cast<std::uint8_t>(n); }

 private:
  std::uint8_t nd_ = 0;
  std::array<Interval, kMaxDims> iv_{};
};

std::optional<ShardView> intersect(const ShardView& a, const ShardView& b);

enum class TensorRole { kParameter, kOptimizerMoment1, kOptimizerMoment2 };
const char* to_string(TensorRole r);

struct TensorSpec {
  std::string tensor_id;
  int layer = 0;
  std::vector<std::int64_t> shape;
  std::optional<int> tp_shard_axis;
  TensorRole role = TensorRole::kParameter;
  std::int64_t element_bytes = 0;  // extension: 0 -> ModelSpec::bytes_per_element
  // extension (distributed optimizer, BASELINE config 3): under a config with
  // distributed_optimizer() the TP block is further split into dp ceil chunks
  // along this axis, one per DP rank; nullopt = DP-replicated
  std::optional<int> dp_shard_axis;
  std::int64_t element_count() const;
};

struct ModelSpec {
  std::string name;
  int num_layers = 1;
  std::vector<TensorSpec> tensors;
  std::int64_t bytes_per_element = 4;
  double state_multiplier = 16.0;

  std::int64_t element_bytes(const TensorSpec& t) const {
    return t.element_bytes > 0 ? t.element_bytes : bytes_per_element;
  }
  std::int64_t total_param_elements() const;
  double total_state_bytes() const;
  std::int64_t total_tensor_bytes() const;
  std::vector<std::string> validate() const;

  // Shared spec text ("model ... / tensor ..." records); see specs.py.
  static ModelSpec parse(const std::string& text);  // throws std::invalid_argument
  std::string to_text() const;
};

struct RankCoord {
  int tp = 0;
  int pp = 0;
  int dp = 0;
  bool operator==(const RankCoord&) const = default;
};

// Rank-list position i -> tp = i % tp, dp = (i / tp) % dp, pp = i / (tp*dp).
class ParallelConfig {
 public:
  ParallelConfig() = default;
  ParallelConfig(std::uint64_t generation_id, int tp, int pp, int dp, std::vector<int> ranks,
                 std::vector<int> layer_assignment);
  static std::vector<int> default_layer_assignment(int num_layers, int pp);

  std::uint64_t generation_id() const { return gen_; }
  int tp() const { return tp_; }
  int pp() const { return pp_; }
  int dp() const { return dp_; }
  int world_size() const { return static_cast<int>(ranks_.size()); }
  const std::vector<int>& ranks() const { return ranks_; }
  const std::vector<int>& layer_assignment() const { return stage_of_; }

  bool contains(int rank) const { return index_.count(rank) != 0; }
  int index_of(int rank) const;  // throws std::invalid_argument
  RankCoord coord_of(int rank) const;
  int rank_at(const RankCoord& c) const;
  int stage_of_layer(int layer) const;
  std::vector<int> stage_ranks(int stage) const;
  bool same_layout(const ParallelConfig& o) const;
  ParallelConfig with_generation(std::uint64_t gen) const;
  // extension: DP ranks shard tensors that declare a dp_shard_axis (ZeRO-1)
  bool distributed_optimizer() const { return dist_opt_; }
  ParallelConfig with_distributed_optimizer(bool on) const;
  // extension: the distributed optimizer's Megatron flat-bucket layout (the
  // DP shard of a tensor is a contiguous range of its TP-local elements,
  // see bucket_range) instead of per-tensor dim chunks; bucket_elems 0 =
  // Megatron's default max(40M, 1M x dp)
  bool flat_buckets() const { return dist_opt_ && flat_; }
  std::int64_t bucket_elems() const;
  ParallelConfig with_flat_buckets(std::int64_t bucket_elems = 0) const;

 private:
  std::uint64_t gen_ = 0;
  int tp_ = 1, pp_ = 1, dp_ = 1;
  std::vector<int> ranks_;
  std::vector<int> stage_of_;
  std::unordered_map<int, int> index_;  // rank id -> position (first occurrence)
  bool dist_opt_ = false;
  bool flat_ = false;
  std::int64_t bucket_elems_ = 0;
};

std::vector<std::string> validate_config(const ParallelConfig& config, const ModelSpec& model);

std::optional<Interval> tp_block(std::int64_t axis_len, int tp_degree, int tp_index);
// Ceil chunk `index` of `parts` over [iv.lo, iv.hi) (extension: DP chunks inside a TP block)
std::optional<Interval> dp_chunk(const Interval& iv, int parts, int index);
std::optional<ShardView> view(const TensorSpec& tensor, const ParallelConfig& config, int rank);
std::map<int, ShardView> owners(const TensorSpec& tensor, const ParallelConfig& config);

// Megatron flat-bucket distributed optimizer (extension).
// On each pipeline stage and TP index the DP-sharded tensors of one role form
// a flat buffer in reverse spec order (backward order), each start padded to a
// multiple of 64 elements; a bucket closes once it holds >= bucket_elems and
// its end is padded to a multiple of lcm(dp, 128); DP rank d owns the d-th of
// dp equal contiguous parts of every bucket.  (Megatron-LM megatron/core/
// distributed/param_and_grad_buffer.py, _ParamAndGradBuffer: params[::-1],
// _pad_start_of_param_if_needed, _pad_end_of_bucket_if_needed;
// megatron/core/optimizer/distrib_optimizer.py, _build_model_gbuf_range.)
// Under such a config view() is the rank's TP block and the rank holds the
// contiguous element range [lo, hi) of that block's row-major order (nullopt:
// the whole block; an empty range: view() is nullopt).
std::optional<std::pair<std::int64_t, std::int64_t>> bucket_range(const ModelSpec& model, std::uint32_t tensor_index,
                                                                  const ParallelConfig& config, int rank);
// The boxes (global coordinates, row-major order) of the elements [lo, hi) of
// `block`'s row-major order: each box is one contiguous run of the block, at
// most 2 (ndims - 1) + 1 of them (<= 3 for a matrix).
std::vector<ShardView> flat_range_boxes(const ShardView& block, std::int64_t lo, std::int64_t hi);
// What `rank` holds of a tensor as boxes: view(), or the boxes of its bucket range.
std::vector<ShardView> held_boxes(const ModelSpec& model, std::uint32_t tensor_index, const ParallelConfig& config,
                                  int rank);

struct TransferTask {
  std::uint32_t tensor_index = 0;
  int layer = 0;
  int src_rank = 0;
  int dst_rank = 0;
  ShardView bounds;
  std::int64_t byte_size = 0;
  bool is_local() const { return src_rank == dst_rank; }
};

struct CarryoverRegion {
  std::uint32_t tensor_index = 0;
  int layer = 0;
  int rank = 0;
  ShardView bounds;
  std::int64_t byte_size = 0;
};

struct LinkKey {
  int src = 0;
  int dst = 0;
  bool operator<(const LinkKey& o) const { return src != o.src ? src < o.src : dst < o.dst; }
  bool operator==(const LinkKey&) const = default;
};

class TransferPlan {
 public:
  std::uint64_t src_config_gen = 0;
  std::uint64_t dst_config_gen = 0;
  std::vector<std::string> tensor_ids;
  std::map<int, std::vector<TransferTask>> tasks_by_layer;
  std::map<int, std::vector<CarryoverRegion>> carryover_by_layer;

  std::int64_t total_bytes() const;
  std::int64_t task_count() const;
  std::map<LinkKey, std::int64_t> per_link_bytes() const;
  bool empty() const { return task_count() == 0; }
  const std::string& tensor_id(std::uint32_t index) const { return tensor_ids.at(index); }
};

struct PlanCostSummary {
  std::int64_t total_bytes = 0;
  std::int64_t max_link_bytes = 0;
  std::int64_t task_count = 0;
};

PlanCostSummary plan_cost_summary(const TransferPlan& plan);
void write_plan(std::ostream& os, const TransferPlan& plan);
TransferPlan read_plan(std::istream& is);

struct PlanOptions {
  bool balance_sources = false;
};

struct PlannerStats {
  std::int64_t pairs_checked = 0;
};

TransferPlan compute_transfer_plan(const ParallelConfig& c_old, const ParallelConfig& c_new,
                                   const ModelSpec& model, const PlanOptions& options = {},
                                   PlannerStats* stats = nullptr);

// Exact completeness check (same verdicts and messages as the reference's
// brute-force oracle) computed on a coordinate-compressed cell grid, so it
// runs on full-size plans in milliseconds instead of O(elements).
std::vector<std::string> verify_plan(const TransferPlan& plan, const ParallelConfig& c_old,
                                     const ParallelConfig& c_new, const ModelSpec& model);

std::vector<ShardView> chunk_bounds(const ShardView& bounds, std::int64_t max_bytes,
                                    std::int64_t bytes_per_element);

// Placement-aware destination rank ordering (extension):
// the rank list of c_new (same tp/pp/dp/layer split), drawn from `candidates`
// (one rank per GPU), that minimises the per-GPU roofline
//   max_g max(max(out_g, in_g) / nvlink, (out_g + in_g + 2 local_g + 2 carry_g) / hbm)
// of the plan c_old -> c_new (ties: fewer remote bytes).  Exhaustive when the
// number of assignments is <= exhaustive_limit, else local search from c_new's
// own list.  Never returns a list scoring worse than c_new's own (when that
// list is drawn from the candidates).
struct PlacementOptions {
  double nvlink_gbs = 900.0;   // per direction, per GPU
  double hbm_gbs = 6552.0;     // copy bandwidth (MEASURED_PEAKS.json)
  std::int64_t exhaustive_limit = 2000000;
  bool balance_sources = false;
};

struct PlacementResult {
  std::vector<int> ranks;  // the chosen rank list for c_new
  double roofline_s = 0, given_roofline_s = 0;
  std::int64_t remote_bytes = 0, local_bytes = 0, carryover_bytes = 0, max_link_bytes = 0;
  std::int64_t given_remote_bytes = 0, given_local_bytes = 0, given_carryover_bytes = 0,
               given_max_link_bytes = 0;
  std::int64_t evaluated = 0;
  bool exhaustive = false;
};

PlacementResult choose_placement(const ParallelConfig& c_old, const ParallelConfig& c_new,
                                 const ModelSpec& model, const std::vector<int>& candidates,
                                 const PlacementOptions& options = {});

// Relay chains for DP broadcasts (extension): tasks of one
// layer with the same source rank, tensor and bounds but destinations on
// different slots are served src -> d0 -> d1 -> ... (each destination's ring
// receiver forwards the drained batches to the next), so the source sends the
// box once.  Only groups where chaining lowers the highest per-slot egress
// are returned (greedy, largest first; deterministic).  `tasks` are indices
// into plan.tasks_by_layer.at(layer) in hop order.
struct RelayChain {
  int layer = 0;
  std::vector<std::size_t> tasks;
};
std::vector<RelayChain> relay_chains(const TransferPlan& plan, const std::function<int(int)>& src_slot,
                                     const std::function<int(int)>& dst_slot);

// ------------------------------------------------------------------ execution
// The reference's execution surface (proj/include/reshard/executor.hpp:16-53,
// shard_store.hpp:14-50, transport.hpp:16-75) over the device engine.

struct ExecutionReport {
  bool ok = false;
  std::string error;
  std::optional<int> failed_layer;
  std::int64_t peak_staging_bytes = 0;  // resident ring capacity per destination rank, max (<= staging_bytes)
  std::int64_t bytes_moved = 0;         // cross-rank task bytes
  std::int64_t local_copy_bytes = 0;
  int layers_processed = 0;
};

// One framed point-to-point chunk of a transfer task.
struct Frame {
  std::uint32_t tensor_index = 0;
  int layer = 0;
  ShardView bounds;
  std::vector<std::uint8_t> data;
};

// Point-to-point transport (reference interface).  On the device path no
// host Frame is materialised: execute_plan reports every chunk the engine
// moved across ranks through on_device_frame (plan order, layer by layer)
// and calls barrier() after each layer, like the reference's executor.
class Transport {
 public:
  virtual ~Transport() = default;
  virtual void send(int src, int dst, Frame frame) = 0;
  virtual std::optional<std::pair<int, Frame>> receive(int dst) = 0;
  virtual void barrier() = 0;
  virtual std::int64_t bytes_sent() const = 0;
  // extension: a chunk of `bytes` payload bytes went src -> dst on the device
  virtual void on_device_frame(int layer, int src, int dst, std::uint32_t tensor_index, const ShardView& bounds,
                               std::int64_t bytes);
};

// In-memory loopback: per-link FIFOs for host frames (lowest source first),
// plus the byte count of device frames.
class LoopbackTransport : public Transport {
 public:
  void send(int src, int dst, Frame frame) override;
  std::optional<std::pair<int, Frame>> receive(int dst) override;
  void barrier() override {}
  std::int64_t bytes_sent() const override { return bytes_sent_; }
  void on_device_frame(int layer, int src, int dst, std::uint32_t tensor_index, const ShardView& bounds,
                       std::int64_t bytes) override;

 private:
  std::map<std::pair<int, int>, std::vector<Frame>> queues_;  // (dst, src) -> FIFO
  std::map<std::pair<int, int>, std::size_t> heads_;
  std::int64_t bytes_sent_ = 0;
};

// Per-event trace (layer, src, dst, bytes) of everything passing through.
class RecordingTransport : public Transport {
 public:
  struct Event {
    std::int64_t sequence = 0;
    int layer = 0;
    int src = 0;
    int dst = 0;
    std::int64_t bytes = 0;
  };
  explicit RecordingTransport(Transport& inner) : inner_(inner) {}
  void send(int src, int dst, Frame frame) override;
  std::optional<std::pair<int, Frame>> receive(int dst) override { return inner_.receive(dst); }
  void barrier() override { inner_.barrier(); }
  std::int64_t bytes_sent() const override { return inner_.bytes_sent(); }
  void on_device_frame(int layer, int src, int dst, std::uint32_t tensor_index, const ShardView& bounds,
                       std::int64_t bytes) override;
  const std::vector<Event>& events() const { return events_; }

 private:
  Transport& inner_;
  std::vector<Event> events_;
  std::int64_t next_sequence_ = 0;
};

// Extension: choose how the device moves cross-rank chunks -- bounded
// staging rings (STAGED, the reference's staging-budget semantics; default for
// any other Transport) or direct stores into the destination shards (DIRECT).
class DeviceTransport : public LoopbackTransport {
 public:
  enum class Mode { kStaged, kDirect };
  explicit DeviceTransport(Mode mode = Mode::kStaged, int device = 0) : mode_(mode), device_(device) {}
  Mode mode() const { return mode_; }
  int device() const { return device_; }

 private:
  Mode mode_;
  int device_;
};

// Host-resident per-(rank, tensor) shard buffers, row-major over each view.
class ShardStore {
 public:
  struct Entry {
    ShardView view;
    std::vector<std::uint8_t> bytes;
  };
  // zero-filled buffers for every present view under `config`
  static ShardStore allocate(const ModelSpec& model, const ParallelConfig& config);

  bool has(int rank, std::uint32_t tensor_index) const;
  Entry& at(int rank, std::uint32_t tensor_index);
  const Entry& at(int rank, std::uint32_t tensor_index) const;
  // the reference pattern (shard_store.cpp:51-85), generated on the device
  void fill_pattern(const ModelSpec& model, std::uint64_t seed);
  static std::uint8_t pattern_byte(std::uint32_t tensor_index, std::int64_t element, std::int64_t byte_in_element,
                                   std::uint64_t seed);
  std::int64_t total_bytes() const;
  std::size_t entry_count() const { return entries_.size(); }
  // extension: the model and layout the store was allocated for (the device
  // engine lays its shard buffers out from them)
  const ModelSpec& model() const { return model_; }
  const ParallelConfig& config() const { return config_; }

 private:
  std::map<std::pair<int, std::uint32_t>, Entry> entries_;
  ModelSpec model_;
  ParallelConfig config_;
};

// Runs `plan` from src_store (C_old) into dst_store (C_new) on the device:
// stores go H2D, the engine executes layer by layer within `staging_bytes`
// of staging per destination rank, results come back D2H.  Integrity
// failures come back as ok = false + error + failed_layer (executor.cpp:210-215);
// CUDA errors throw std::runtime_error.
ExecutionReport execute_plan(const TransferPlan& plan, const ShardStore& src_store, ShardStore& dst_store,
                             Transport& transport, std::int64_t staging_bytes, std::int64_t bytes_per_element);

}  // namespace reshard
