// The reference's C++ execution surface on the B200 engine:
// ShardStore / Transport / execute_plan with the shapes of
// proj/include/reshard/{shard_store,transport,executor}.hpp, so a caller
// written against the reference (e.g. SPEC.md:514 cmd_verify, or its tests)
// compiles against include/reshard/*.hpp and runs the plan on the device.
//
// execute_plan = rs_execute_host: host stores go H2D, one device program
// runs the plan (STAGED rings within staging_bytes per destination rank, or
// DIRECT stores when the caller passes DeviceTransport(kDirect)), results
// come back D2H.  No byte is moved on the host: the Transport receives the
// per-chunk accounting of what the device moved (on_device_frame) and one
// barrier() per layer (executor.cpp:208).
#include <cuda_runtime.h>

#include <algorithm>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine/engine.hpp"
#include "engine/engine_internal.hpp"
#include "reshard_b200/reshard.hpp"

namespace reshard {

// ------------------------------------------------------------- transports

void Transport::on_device_frame(int, int, int, std::uint32_t, const ShardView&, std::int64_t) {}

void LoopbackTransport::send(int src, int dst, Frame frame) {
  bytes_sent_ += static_cast<std::int64_t>(frame.data.size());
  queues_[{dst, src}].push_back(std::move(frame));
}

std::optional<std::pair<int, Frame>> LoopbackTransport::receive(int dst) {
  // lowest source rank with a pending frame first (transport.hpp:35)
  for (auto it = queues_.lower_bound({dst, std::numeric_limits<int>::min()}); it != queues_.end() && it->first.first == dst;
       ++it) {
    std::size_t& head = heads_[it->first];
    if (head < it->second.size()) {
      Frame f = std::move(it->second[head++]);
      if (head == it->second.size()) {
        it->second.clear();
        head = 0;
      }
      return std::make_pair(it->first.second, std::move(f));
    }
  }
  return std::nullopt;
}

void LoopbackTransport::on_device_frame(int, int, int, std::uint32_t, const ShardView&, std::int64_t bytes) {
  bytes_sent_ += bytes;
}

void RecordingTransport::send(int src, int dst, Frame frame) {
  events_.push_back({next_sequence_++, frame.layer, src, dst, static_cast<std::int64_t>(frame.data.size())});
  inner_.send(src, dst, std::move(frame));
}

void RecordingTransport::on_device_frame(int layer, int src, int dst, std::uint32_t tensor_index,
                                         const ShardView& bounds, std::int64_t bytes) {
  events_.push_back({next_sequence_++, layer, src, dst, bytes});
  inner_.on_device_frame(layer, src, dst, tensor_index, bounds, bytes);
}

// ------------------------------------------------------------- shard store

ShardStore ShardStore::allocate(const ModelSpec& model, const ParallelConfig& config) {
  if (config.flat_buckets())  // the reference's store holds whole views (shard_store.hpp:21-24)
    throw std::invalid_argument("ShardStore: flat-bucket configs hold element ranges; use the rs_* C ABI stores");
  ShardStore s;
  s.model_ = model;
  s.config_ = config;
  for (std::uint32_t ti = 0; ti < model.tensors.size(); ++ti) {
    const auto& t = model.tensors[ti];
    for (int rank : config.ranks()) {
      auto v = view(t, config, rank);
      if (!v) continue;
      Entry e;
      e.view = *v;
      e.bytes.assign(static_cast<std::size_t>(v->element_count() * model.element_bytes(t)), 0);
      s.entries_.emplace(std::make_pair(rank, ti), std::move(e));
    }
  }
  return s;
}

bool ShardStore::has(int rank, std::uint32_t tensor_index) const { return entries_.count({rank, tensor_index}) != 0; }

ShardStore::Entry& ShardStore::at(int rank, std::uint32_t tensor_index) {
  auto it = entries_.find({rank, tensor_index});
  if (it == entries_.end())
    throw std::out_of_range("shard store: no buffer for rank " + std::to_string(rank) + " tensor " +
                            std::to_string(tensor_index));
  return it->second;
}

const ShardStore::Entry& ShardStore::at(int rank, std::uint32_t tensor_index) const {
  return const_cast<ShardStore*>(this)->at(rank, tensor_index);
}

std::int64_t ShardStore::total_bytes() const {
  std::int64_t n = 0;
  for (const auto& [k, e] : entries_) n += static_cast<std::int64_t>(e.bytes.size());
  return n;
}

std::uint8_t ShardStore::pattern_byte(std::uint32_t tensor_index, std::int64_t element, std::int64_t byte_in_element,
                                      std::uint64_t seed) {
  std::uint64_t x = (seed ^ (0x1000003ull * tensor_index)) ^ static_cast<std::uint64_t>(element);
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  x ^= x >> 31;
  return static_cast<std::uint8_t>(x >> (8 * (byte_in_element % 8)));
}

namespace {

int current_device() {
  int dev = 0;
  rsb::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  return dev;
}

rs_engine_options engine_options(const int* device, std::int64_t staging_bytes, int mode) {
  rs_engine_options o{};
  o.num_devices = 1;
  o.device_ids = device;
  o.staging_bytes = staging_bytes;
  o.mode = mode;
  return o;
}

// A store's entries in engine order (tensor, ascending rank), as host pointers.
template <class Store>
std::vector<void*> host_pointers(const rsb::Store& layout, Store& s) {
  std::vector<void*> out;
  out.reserve(layout.entries.size());
  for (const auto& e : layout.entries)
    out.push_back(const_cast<std::uint8_t*>(s.at(e.rank, e.ti).bytes.data()));
  return out;
}

}  // namespace

void ShardStore::fill_pattern(const ModelSpec& model, std::uint64_t seed) {
  // the pattern kernel writes a device copy of the store, then D2H
  const int dev = current_device();
  rsb::Engine eng(engine_options(&dev, 1, RS_MODE_DIRECT));
  eng.layout(RS_SRC, model, config_, std::vector<int>(static_cast<std::size_t>(config_.world_size()), 0));
  eng.alloc(RS_SRC);
  eng.fill_pattern(RS_SRC, seed);
  for (const auto& e : eng.store(RS_SRC).entries) {
    auto& buf = at(e.rank, e.ti).bytes;
    if (static_cast<std::int64_t>(buf.size()) != e.nbytes) throw std::invalid_argument("fill_pattern: store does not match model");
    rsb::cuda_check(cudaMemcpy(buf.data(), e.ptr, buf.size(), cudaMemcpyDeviceToHost), "fill_pattern D2H");
  }
}

// -------------------------------------------------------------- execution

ExecutionReport execute_plan(const TransferPlan& plan, const ShardStore& src_store, ShardStore& dst_store,
                             Transport& transport, std::int64_t staging_bytes, std::int64_t bytes_per_element) {
  if (bytes_per_element < 1) throw std::invalid_argument("execute_plan: bytes_per_element must be >= 1");
  // one element size for every tensor, as the reference executes (executor.hpp:53)
  ModelSpec model = src_store.model();
  model.bytes_per_element = bytes_per_element;
  for (auto& t : model.tensors) t.element_bytes = 0;
  // plan tensor indices -> model order by id (read_plan interns in appearance order)
  TransferPlan p = plan;
  if (p.tensor_ids.size() != model.tensors.size()) throw std::invalid_argument("execute_plan: plan does not match the store model");
  std::vector<std::uint32_t> remap(p.tensor_ids.size());
  for (std::size_t i = 0; i < p.tensor_ids.size(); ++i) {
    auto it = std::find_if(model.tensors.begin(), model.tensors.end(),
                           [&](const TensorSpec& t) { return t.tensor_id == p.tensor_ids[i]; });
    if (it == model.tensors.end()) throw std::invalid_argument("execute_plan: plan references unknown tensor " + p.tensor_ids[i]);
    remap[i] = static_cast<std::uint32_t>(it - model.tensors.begin());
  }
  for (auto& [layer, tasks] : p.tasks_by_layer)
    for (auto& t : tasks) t.tensor_index = remap[t.tensor_index];
  for (auto& [layer, keeps] : p.carryover_by_layer)
    for (auto& k : keeps) k.tensor_index = remap[k.tensor_index];
  p.tensor_ids.clear();
  for (const auto& t : model.tensors) p.tensor_ids.push_back(t.tensor_id);

  const auto* dt = dynamic_cast<const DeviceTransport*>(&transport);
  const int dev = dt ? dt->device() : current_device();
  const int mode = dt && dt->mode() == DeviceTransport::Mode::kDirect ? RS_MODE_DIRECT : RS_MODE_STAGED;
  rsb::Engine eng(engine_options(&dev, staging_bytes, mode));
  eng.layout(RS_SRC, model, src_store.config(), std::vector<int>(static_cast<std::size_t>(src_store.config().world_size()), 0));
  eng.layout(RS_DST, model, dst_store.config(), std::vector<int>(static_cast<std::size_t>(dst_store.config().world_size()), 0));
  for (int which : {RS_SRC, RS_DST}) {
    const ShardStore& hs = which == RS_SRC ? src_store : dst_store;
    for (const auto& e : eng.store(which).entries)
      if (!hs.has(e.rank, e.ti) || static_cast<std::int64_t>(hs.at(e.rank, e.ti).bytes.size()) != e.nbytes)
        throw std::invalid_argument("execute_plan: store entry (rank " + std::to_string(e.rank) + ", tensor " +
                                    std::to_string(e.ti) + ") does not match its view at bytes_per_element " +
                                    std::to_string(bytes_per_element));
  }
  eng.alloc(RS_SRC);
  eng.alloc(RS_DST);
  // dst is updated in place (executor.hpp:50): bytes the plan does not write
  // -- all of a failed layer's and later layers' -- keep their host values
  for (const auto& e : eng.store(RS_DST).entries)
    rsb::cuda_check(cudaMemcpy(e.ptr, dst_store.at(e.rank, e.ti).bytes.data(), static_cast<std::size_t>(e.nbytes),
                               cudaMemcpyHostToDevice),
                    "execute_plan dst H2D");
  eng.prepare(p);
  const auto src_ptrs = host_pointers(eng.store(RS_SRC), src_store);
  const auto dst_ptrs = host_pointers(eng.store(RS_DST), dst_store);
  const rs_exec_report r = eng.run_host(src_ptrs.data(), dst_ptrs.data(), 0);

  ExecutionReport rep;
  rep.ok = r.ok != 0;
  rep.error = r.error;
  if (r.failed_layer >= 0) rep.failed_layer = r.failed_layer;
  rep.peak_staging_bytes = r.peak_staging_bytes;
  rep.bytes_moved = r.bytes_moved;
  rep.local_copy_bytes = r.local_copy_bytes;
  rep.layers_processed = r.layers_processed;
  // transport accounting: the frames the reference's executor would have sent
  // (every cross-rank task chunked to the budget, executor.cpp:183-206), for
  // the layers the device completed, and one barrier per layer (:208)
  int done = 0;
  for (const auto& [layer, tasks] : p.tasks_by_layer) {
    if (done == rep.layers_processed || (rep.failed_layer && layer >= *rep.failed_layer)) break;
    for (const auto& t : tasks) {
      if (t.is_local()) continue;
      for (const auto& c : chunk_bounds(t.bounds, staging_bytes, bytes_per_element))
        transport.on_device_frame(layer, t.src_rank, t.dst_rank, t.tensor_index, c,
                                  c.element_count() * bytes_per_element);
    }
    transport.barrier();
    ++done;
  }
  return rep;
}

}  // namespace reshard
