// Device reshard engine.
//
// prepare() turns a TransferPlan into per-device work lists, validating every
// task and carryover with the reference executor's integrity rules and error
// messages (proj/src/executor.cpp:142-206): a failing layer is reported as
// failed_layer with every earlier layer executed, like execute_plan's
// per-layer try/catch (executor.cpp:210-215).
//
// DIRECT mode: every task and carryover is one strided->strided copy issued
//   by the device holding its source (push); cross-device destinations are
//   written through peer mappings (NVLink stores).  Zero staging.
// STAGED mode: cross-rank tasks are chunked to the ring slot size and
//   streamed through per-(src,dst) single-producer/single-consumer rings that
//   live in the destination's staging budget B; local tasks and carryovers
//   run as DIRECT copies in the same launch.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <set>

#include "compile.hpp"
#include "kernels.h"

namespace rsb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw SystemError(std::string(what) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
}

namespace {

constexpr std::size_t kAlign = 256;

std::uint64_t key(int rank, std::uint32_t ti) {
  return (static_cast<std::uint64_t>(ti) << 32) | static_cast<std::uint32_t>(rank);
}

std::size_t align_up(std::size_t x, std::size_t a) { return (x + a - 1) / a * a; }

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

// ------------------------------------------------------------ DeviceBuffer

DeviceBuffer::DeviceBuffer(int device, std::size_t bytes) : device_(device), bytes_(bytes) {
  if (bytes == 0) return;
  DeviceGuard g(device);
  cuda_check(cudaMalloc(&ptr_, bytes), "cudaMalloc");
}

DeviceBuffer::~DeviceBuffer() {
  if (ptr_) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    cudaFree(ptr_);
    cudaSetDevice(prev);
  }
}

DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
  if (this != &o) {
    this->~DeviceBuffer();
    device_ = o.device_;
    ptr_ = o.ptr_;
    bytes_ = o.bytes_;
    o.ptr_ = nullptr;
    o.bytes_ = 0;
  }
  return *this;
}

void DeviceBuffer::upload(const void* host, std::size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  DeviceGuard g(device_);
  cuda_check(cudaMemcpyAsync(ptr_, host, bytes, cudaMemcpyHostToDevice, s), "upload");
}

// ------------------------------------------------------------------- Store

const Entry* Store::find(int rank, std::uint32_t ti) const {
  auto it = index.find(key(rank, ti));
  return it == index.end() ? nullptr : &entries[it->second];
}

Entry* Store::find(int rank, std::uint32_t ti) {
  auto it = index.find(key(rank, ti));
  return it == index.end() ? nullptr : &entries[it->second];
}

std::int64_t Store::total_bytes() const {
  std::int64_t n = 0;
  for (const auto& e : entries) n += e.nbytes;
  return n;
}

// ------------------------------------------------------------------ Engine

Engine::Engine(const rs_engine_options& opts) : opts_(opts) {
  if (opts.num_devices < 1 || !opts.device_ids) throw DomainError("engine: no devices");
  if (opts.staging_bytes < 1) throw DomainError("engine: staging_bytes must be >= 1");
  if (opts.mode != RS_MODE_DIRECT && opts.mode != RS_MODE_STAGED) throw DomainError("engine: unknown mode");
  if (opts_.slots_per_link < 2) opts_.slots_per_link = 2;
  if (opts_.lanes_per_link < 1) opts_.lanes_per_link = 1;
  int count = 0;
  cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  for (int i = 0; i < opts.num_devices; ++i) {
    Device d;
    d.ordinal = opts.device_ids[i];
    if (d.ordinal < 0 || d.ordinal >= count) throw DomainError("engine: bad device id " + std::to_string(d.ordinal));
    DeviceGuard g(d.ordinal);
    cuda_check(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, d.ordinal), "sm count");
    cuda_check(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&d.h2d, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&d.d2h, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreate(&d.ev_begin), "event");
    cuda_check(cudaEventCreate(&d.ev_end), "event");
    devices_.push_back(d);
  }
  for (auto& a : devices_)
    for (auto& b : devices_) {
      if (a.ordinal == b.ordinal) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a.ordinal, b.ordinal);
      if (!can) continue;
      DeviceGuard g(a.ordinal);
      cudaError_t e = cudaDeviceEnablePeerAccess(b.ordinal, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else cuda_check(e, "cudaDeviceEnablePeerAccess");
    }
}

Engine::~Engine() {
  programs_.clear();
  rings_.clear();
  for (auto& s : stores_) s.arenas.clear();
  for (auto& d : devices_) {
    cudaSetDevice(d.ordinal);
    if (d.stream) cudaStreamDestroy(d.stream);
    if (d.h2d) cudaStreamDestroy(d.h2d);
    if (d.d2h) cudaStreamDestroy(d.d2h);
    if (d.ev_begin) cudaEventDestroy(d.ev_begin);
    if (d.ev_end) cudaEventDestroy(d.ev_end);
  }
}

void Engine::layout(int which, const reshard::ModelSpec& model, const reshard::ParallelConfig& cfg,
                    const std::vector<int>& rank_device) {
  if (which != RS_SRC && which != RS_DST) throw DomainError("store: which must be RS_SRC or RS_DST");
  if (auto v = model.validate(); !v.empty()) throw DomainError("model: " + v.front());
  if (auto v = reshard::validate_config(cfg, model); !v.empty()) throw DomainError("config: " + v.front());
  if (static_cast<int>(rank_device.size()) != cfg.world_size())
    throw DomainError("store: rank_device must have one entry per rank");
  for (int d : rank_device)
    if (d < 0 || d >= num_devices()) throw DomainError("store: rank_device entry out of range");
  Store s;
  s.model = model;
  s.config = cfg;
  for (std::uint32_t ti = 0; ti < model.tensors.size(); ++ti) {
    const auto& t = model.tensors[ti];
    for (const auto& [rank, v] : reshard::owners(t, cfg)) {
      Entry e;
      e.ti = ti;
      e.rank = rank;
      e.dev = rank_device[static_cast<std::size_t>(cfg.index_of(rank))];
      e.view = v;
      e.nbytes = v.element_count() * model.element_bytes(t);
      s.index.emplace(key(rank, ti), static_cast<std::uint32_t>(s.entries.size()));
      s.entries.push_back(e);
    }
  }
  s.laid_out = true;
  stores_[which] = std::move(s);
  prepared_ = false;
}

void Engine::alloc(int which) {
  Store& s = stores_[which];
  if (!s.laid_out) throw DomainError("store: layout first");
  s.arenas.clear();
  std::vector<std::size_t> need(devices_.size(), 0);
  for (const auto& e : s.entries) need[static_cast<std::size_t>(e.dev)] += align_up(static_cast<std::size_t>(e.nbytes), kAlign);
  for (std::size_t d = 0; d < devices_.size(); ++d)
    s.arenas.emplace_back(devices_[d].ordinal, need[d]);
  std::vector<std::size_t> off(devices_.size(), 0);
  for (auto& e : s.entries) {
    const auto d = static_cast<std::size_t>(e.dev);
    e.ptr = s.arenas[d].data() + off[d];
    off[d] += align_up(static_cast<std::size_t>(e.nbytes), kAlign);
  }
  prepared_ = false;
}

void Engine::free_store(int which) {
  Store& s = stores_[which];
  s.arenas.clear();
  for (auto& e : s.entries) e.ptr = nullptr;
  prepared_ = false;
}

void Engine::bind(int which, int rank, std::uint32_t ti, void* ptr, std::int64_t nbytes) {
  Store& s = stores_[which];
  if (!s.laid_out) throw DomainError("store: layout first");
  Entry* e = s.find(rank, ti);
  if (!e) throw DomainError("shard store: no buffer for rank " + std::to_string(rank) + " tensor " + std::to_string(ti));
  if (nbytes != e->nbytes)
    throw DomainError("store bind: buffer size " + std::to_string(nbytes) + " does not match view size " +
                      std::to_string(e->nbytes));
  e->ptr = static_cast<char*>(ptr);
  prepared_ = false;
}

void Engine::check_stores_ready() const {
  for (int w = 0; w < 2; ++w) {
    if (!stores_[w].laid_out) throw DomainError(w ? "dst store not laid out" : "src store not laid out");
    for (const auto& e : stores_[w].entries)
      if (!e.ptr && e.nbytes)
        throw DomainError(std::string(w ? "dst" : "src") + " store: entry rank " + std::to_string(e.rank) +
                          " tensor " + std::to_string(e.ti) + " has no device memory");
  }
}

int Engine::grid_for(int dev, int which_kernel) const {
  int per_sm = rs_kernel_max_blocks_per_sm(which_kernel);
  if (per_sm < 1) per_sm = 1;
  if (opts_.blocks_per_sm > 0) per_sm = std::min(per_sm, opts_.blocks_per_sm);
  return devices_[static_cast<std::size_t>(dev)].sms * per_sm;
}

int Engine::copy_variant(int dev) const {
  switch (opts_.copy_kernel) {
    case RS_COPY_LDG8: return 2;
    case RS_COPY_BULK: return programs_[static_cast<std::size_t>(dev)].all_aligned ? 3 : 1;
    case RS_COPY_LDG4_CS: return 4;
    case RS_COPY_LDG8_CS: return 5;
    default: return 1;
  }
}

int Engine::copy_grid(int dev) const {
  switch (copy_variant(dev)) {
    case 2:
    case 5: return grid_for(dev, 3);
    case 3: return devices_[static_cast<std::size_t>(dev)].sms;  // one bulk issuer CTA per SM
    default: return grid_for(dev, 0);
  }
}

// ---------------------------------------------------------------- patterns

void Engine::fill_pattern(int which, std::uint64_t seed) { (void)verify_pattern(-1 - which, seed, nullptr); }

std::int64_t Engine::verify_pattern(int which_in, std::uint64_t seed, std::int64_t* first_bad) {
  const bool verify = which_in >= 0;
  const int which = verify ? which_in : -1 - which_in;
  const Store& s = stores_[which];
  if (!s.laid_out) throw DomainError("store: layout first");
  std::int64_t total_bad = 0;
  std::uint64_t first = ~0ull;
  for (int d = 0; d < num_devices(); ++d) {
    std::vector<rs_pattern_desc> descs;
    std::uint64_t bytes = 0;
    for (std::uint32_t k = 0; k < s.entries.size(); ++k) {
      const Entry& e = s.entries[k];
      if (e.dev != d) continue;
      if (!e.ptr) throw DomainError("store: entry without device memory");
      bytes += static_cast<std::uint64_t>(e.nbytes);
    }
    if (bytes == 0) continue;
    const int grid = grid_for(d, 1);
    const std::uint64_t warps = static_cast<std::uint64_t>(grid) * 8;
    const std::uint64_t item_bytes = std::clamp<std::uint64_t>(bytes / (warps * 8), 16384, 1 << 20);
    for (std::uint32_t k = 0; k < s.entries.size(); ++k) {
      const Entry& e = s.entries[k];
      if (e.dev != d) continue;
      const auto& t = s.model.tensors[e.ti];
      append_pattern(descs, reinterpret_cast<std::uint64_t>(e.ptr), t, e.view, s.model.element_bytes(t), e.ti, k,
                     item_bytes);
    }
    std::vector<std::uint64_t> item0(descs.size());
    std::uint64_t items = 0;
    for (std::size_t i = 0; i < descs.size(); ++i) {
      descs[i].item0 = items;
      item0[i] = items;
      items += (descs[i].rows + descs[i].rows_per_item - 1) / descs[i].rows_per_item;
    }
    const Device& dv = devices_[static_cast<std::size_t>(d)];
    DeviceGuard g(dv.ordinal);
    DeviceBuffer dd(dv.ordinal, descs.size() * sizeof(rs_pattern_desc));
    DeviceBuffer di(dv.ordinal, item0.size() * sizeof(std::uint64_t));
    DeviceBuffer dc(dv.ordinal, 2 * sizeof(unsigned long long));
    dd.upload(descs.data(), descs.size() * sizeof(rs_pattern_desc), dv.stream);
    di.upload(item0.data(), item0.size() * sizeof(std::uint64_t), dv.stream);
    unsigned long long init[2] = {0ull, ~0ull};
    dc.upload(init, sizeof init, dv.stream);
    auto* counters = reinterpret_cast<unsigned long long*>(dc.data());
    cuda_check(rs_launch_pattern(reinterpret_cast<const rs_pattern_desc*>(dd.data()),
                                 reinterpret_cast<const std::uint64_t*>(di.data()),
                                 static_cast<std::uint32_t>(descs.size()), items, seed, verify ? 1 : 0,
                                 counters, counters + 1, grid, dv.stream),
               "pattern kernel launch");
    unsigned long long out[2] = {0, 0};
    cuda_check(cudaMemcpyAsync(out, counters, sizeof out, cudaMemcpyDeviceToHost, dv.stream), "readback");
    cuda_check(cudaStreamSynchronize(dv.stream), "pattern kernel");
    total_bad += static_cast<std::int64_t>(out[0]);
    first = std::min<std::uint64_t>(first, out[1]);
  }
  if (first_bad) *first_bad = first == ~0ull ? -1 : static_cast<std::int64_t>(first);
  return total_bad;
}

// ----------------------------------------------------------------- prepare

namespace {

std::string escape_msg(const char* who, const reshard::ShardView& b, const reshard::ShardView& owner) {
  return std::string(who) + ": bounds " + b.to_string() + " escape owner view " + owner.to_string();
}

std::string no_buffer(int rank, std::uint32_t ti) {
  return "shard store: no buffer for rank " + std::to_string(rank) + " tensor " + std::to_string(ti);
}

}  // namespace

void Engine::prepare(const reshard::TransferPlan& plan) {
  check_stores_ready();
  const auto& m = stores_[RS_SRC].model;
  if (plan.tensor_ids.size() != m.tensors.size())
    throw DomainError("plan does not match the store model (tensor count)");
  for (std::size_t i = 0; i < m.tensors.size(); ++i)
    if (plan.tensor_ids[i] != m.tensors[i].tensor_id)
      throw DomainError("plan does not match the store model (tensor " + plan.tensor_ids[i] + ")");
  const auto& md = stores_[RS_DST].model;
  if (md.tensors.size() != m.tensors.size()) throw DomainError("src and dst stores use different models");

  planned_ = rs_exec_report{};
  planned_.failed_layer = -1;
  plan_layers_.clear();
  std::set<int> layers;
  for (const auto& kv : plan.tasks_by_layer) layers.insert(kv.first);
  for (const auto& kv : plan.carryover_by_layer) layers.insert(kv.first);
  plan_layers_.assign(layers.begin(), layers.end());

  programs_.clear();
  programs_.resize(devices_.size());
  rings_.clear();
  if (opts_.mode == RS_MODE_DIRECT) compile_direct(plan);
  else compile_staged(plan);
  upload_programs();
  prepared_ = true;
}

void Engine::compile_direct(const reshard::TransferPlan& plan) {
  const Store& src = stores_[RS_SRC];
  const Store& dst = stores_[RS_DST];
  const auto& m = src.model;
  const std::int64_t B = opts_.staging_bytes;
  std::vector<std::size_t> mark(devices_.size());

  for (int layer : plan_layers_) {
    for (std::size_t d = 0; d < devices_.size(); ++d) mark[d] = programs_[d].local.size();
    rs_exec_report delta{};
    try {
      if (auto it = plan.carryover_by_layer.find(layer); it != plan.carryover_by_layer.end()) {
        for (const auto& k : it->second) {
          const Entry* se = src.find(k.rank, k.tensor_index);
          const Entry* de = se ? dst.find(k.rank, k.tensor_index) : nullptr;
          if (!se) throw IntegrityError(no_buffer(k.rank, k.tensor_index));
          if (!de) throw IntegrityError(no_buffer(k.rank, k.tensor_index));
          if (!se->view.contains(k.bounds)) throw IntegrityError(escape_msg("slice_local", k.bounds, se->view));
          if (!de->view.contains(k.bounds)) throw IntegrityError(escape_msg("scatter_local", k.bounds, de->view));
          const std::int64_t eb = m.element_bytes(m.tensors[k.tensor_index]);
          append_copy(programs_[static_cast<std::size_t>(se->dev)].local, reinterpret_cast<std::uint64_t>(se->ptr),
                      se->view, reinterpret_cast<std::uint64_t>(de->ptr), de->view, k.bounds, eb,
                      static_cast<std::uint32_t>(layer));
          delta.carryover_bytes += k.bounds.element_count() * eb;
        }
      }
      if (auto it = plan.tasks_by_layer.find(layer); it != plan.tasks_by_layer.end()) {
        for (const auto& t : it->second) {
          const Entry* se = src.find(t.src_rank, t.tensor_index);
          if (!se) throw IntegrityError(no_buffer(t.src_rank, t.tensor_index));
          if (!se->view.contains(t.bounds)) throw IntegrityError("integrity: task bounds escape source view");
          const std::int64_t eb = m.element_bytes(m.tensors[t.tensor_index]);
          if (eb > B)
            throw IntegrityError("chunk_bounds: one element exceeds the staging budget");
          const Entry* de = dst.find(t.dst_rank, t.tensor_index);
          if (!de) throw IntegrityError(no_buffer(t.dst_rank, t.tensor_index));
          if (!de->view.contains(t.bounds)) throw IntegrityError(escape_msg("scatter_local", t.bounds, de->view));
          append_copy(programs_[static_cast<std::size_t>(se->dev)].local, reinterpret_cast<std::uint64_t>(se->ptr),
                      se->view, reinterpret_cast<std::uint64_t>(de->ptr), de->view, t.bounds, eb,
                      static_cast<std::uint32_t>(layer));
          const std::int64_t n = t.bounds.element_count() * eb;
          if (t.is_local()) delta.local_copy_bytes += n;
          else delta.bytes_moved += n;
        }
      }
    } catch (const std::exception& e) {
      for (std::size_t d = 0; d < devices_.size(); ++d) programs_[d].local.resize(mark[d]);
      planned_.ok = 0;
      planned_.failed_layer = layer;
      std::snprintf(planned_.error, sizeof planned_.error, "%s", e.what());
      return;
    }
    planned_.carryover_bytes += delta.carryover_bytes;
    planned_.local_copy_bytes += delta.local_copy_bytes;
    planned_.bytes_moved += delta.bytes_moved;
    planned_.layers_processed++;
    // descriptor index ranges for now; upload_programs() turns them into item ranges
    for (std::size_t d = 0; d < devices_.size(); ++d)
      programs_[d].layers.push_back({layer, mark[d], programs_[d].local.size()});
  }
  planned_.ok = 1;
}

void Engine::compile_staged(const reshard::TransferPlan& plan) {
  const Store& src = stores_[RS_SRC];
  const Store& dst = stores_[RS_DST];
  const auto& m = src.model;
  const std::int64_t B = opts_.staging_bytes;
  const int P = opts_.lanes_per_link, K = opts_.slots_per_link;

  // inbound links per destination rank (remote tasks only)
  std::map<int, std::set<int>> inbound;
  for (const auto& kv : plan.tasks_by_layer)
    for (const auto& t : kv.second)
      if (!t.is_local()) inbound[t.dst_rank].insert(t.src_rank);

  struct LaneBuild {
    int src_rank, dst_rank, sdev, ddev;
    std::uint64_t slot_bytes;
    char* slots = nullptr;          // on ddev
    std::uint64_t* ready = nullptr; // on ddev
    std::uint64_t* credit = nullptr;// on sdev
    struct Frame {
      const Entry* se;
      const Entry* de;
      reshard::ShardView region;
      std::int64_t eb;
      std::uint64_t off;
      int layer;
    };
    std::vector<std::vector<Frame>> batches;
    std::uint64_t fill = 0;
  };
  std::vector<LaneBuild> lanes;
  std::map<std::pair<int, int>, int> link_first_lane;
  std::map<std::pair<int, int>, int> link_cursor;
  std::map<int, std::uint64_t> slot_bytes_of;  // per dst rank
  for (const auto& [d, srcs] : inbound) {
    std::uint64_t sb = static_cast<std::uint64_t>(B) / (srcs.size() * static_cast<std::uint64_t>(P * K));
    sb = sb / kAlign * kAlign;
    slot_bytes_of[d] = sb;
  }

  // layer-ordered frames
  std::vector<std::size_t> mark(devices_.size());
  for (int layer : plan_layers_) {
    for (std::size_t d = 0; d < devices_.size(); ++d) mark[d] = programs_[d].local.size();
    std::vector<std::size_t> lane_mark_batches(lanes.size());
    std::vector<std::uint64_t> lane_mark_fill(lanes.size());
    std::vector<std::size_t> lane_mark_frames(lanes.size());
    for (std::size_t i = 0; i < lanes.size(); ++i) {
      lane_mark_batches[i] = lanes[i].batches.size();
      lane_mark_fill[i] = lanes[i].fill;
      lane_mark_frames[i] = lanes[i].batches.empty() ? 0 : lanes[i].batches.back().size();
    }
    const std::size_t lanes_before = lanes.size();
    rs_exec_report delta{};
    try {
      if (auto it = plan.carryover_by_layer.find(layer); it != plan.carryover_by_layer.end()) {
        for (const auto& k : it->second) {
          const Entry* se = src.find(k.rank, k.tensor_index);
          const Entry* de = se ? dst.find(k.rank, k.tensor_index) : nullptr;
          if (!se || !de) throw IntegrityError(no_buffer(k.rank, k.tensor_index));
          if (!se->view.contains(k.bounds)) throw IntegrityError(escape_msg("slice_local", k.bounds, se->view));
          if (!de->view.contains(k.bounds)) throw IntegrityError(escape_msg("scatter_local", k.bounds, de->view));
          const std::int64_t eb = m.element_bytes(m.tensors[k.tensor_index]);
          append_copy(programs_[static_cast<std::size_t>(se->dev)].local, reinterpret_cast<std::uint64_t>(se->ptr),
                      se->view, reinterpret_cast<std::uint64_t>(de->ptr), de->view, k.bounds, eb,
                      static_cast<std::uint32_t>(layer));
          delta.carryover_bytes += k.bounds.element_count() * eb;
        }
      }
      if (auto it = plan.tasks_by_layer.find(layer); it != plan.tasks_by_layer.end()) {
        for (const auto& t : it->second) {
          const Entry* se = src.find(t.src_rank, t.tensor_index);
          if (!se) throw IntegrityError(no_buffer(t.src_rank, t.tensor_index));
          if (!se->view.contains(t.bounds)) throw IntegrityError("integrity: task bounds escape source view");
          const std::int64_t eb = m.element_bytes(m.tensors[t.tensor_index]);
          const Entry* de = dst.find(t.dst_rank, t.tensor_index);
          if (t.is_local()) {
            if (eb > B) throw IntegrityError("chunk_bounds: one element exceeds the staging budget");
            if (!de) throw IntegrityError(no_buffer(t.dst_rank, t.tensor_index));
            if (!de->view.contains(t.bounds)) throw IntegrityError(escape_msg("scatter_local", t.bounds, de->view));
            append_copy(programs_[static_cast<std::size_t>(se->dev)].local, reinterpret_cast<std::uint64_t>(se->ptr),
                        se->view, reinterpret_cast<std::uint64_t>(de->ptr), de->view, t.bounds, eb,
                        static_cast<std::uint32_t>(layer));
            delta.local_copy_bytes += t.bounds.element_count() * eb;
            continue;
          }
          const std::uint64_t sb = slot_bytes_of.at(t.dst_rank);
          if (eb > B) throw IntegrityError("chunk_bounds: one element exceeds the staging budget");
          if (static_cast<std::uint64_t>(eb) > sb)
            throw IntegrityError("staging: ring slot of " + std::to_string(sb) + " bytes cannot hold one element (B=" +
                                 std::to_string(B) + " over " + std::to_string(inbound[t.dst_rank].size()) +
                                 " inbound links)");
          auto chunks = reshard::chunk_bounds(t.bounds, static_cast<std::int64_t>(sb), eb);
          if (!de) throw IntegrityError(no_buffer(t.dst_rank, t.tensor_index));
          if (!de->view.contains(t.bounds)) throw IntegrityError(escape_msg("scatter_local", t.bounds, de->view));
          const auto lk = std::make_pair(t.src_rank, t.dst_rank);
          if (!link_first_lane.count(lk)) {
            link_first_lane[lk] = static_cast<int>(lanes.size());
            for (int p = 0; p < P; ++p) {
              LaneBuild lb;
              lb.src_rank = t.src_rank;
              lb.dst_rank = t.dst_rank;
              lb.sdev = se->dev;
              lb.ddev = de->dev;
              lb.slot_bytes = sb;
              lanes.push_back(std::move(lb));
            }
          }
          for (const auto& c : chunks) {
            int& cur = link_cursor[lk];
            LaneBuild& lb = lanes[static_cast<std::size_t>(link_first_lane[lk] + cur)];
            cur = (cur + 1) % P;
            const std::uint64_t n = static_cast<std::uint64_t>(c.element_count() * eb);
            std::uint64_t off = align_up(lb.fill, 16);
            if (lb.batches.empty() || off + n > lb.slot_bytes) {
              lb.batches.emplace_back();
              off = 0;
            }
            lb.batches.back().push_back({se, de, c, eb, off, layer});
            lb.fill = off + n;
          }
          delta.bytes_moved += t.bounds.element_count() * eb;
        }
      }
    } catch (const std::exception& e) {
      for (std::size_t d = 0; d < devices_.size(); ++d) programs_[d].local.resize(mark[d]);
      lanes.resize(lanes_before);
      for (std::size_t i = 0; i < lanes_before; ++i) {
        lanes[i].batches.resize(lane_mark_batches[i]);
        if (!lanes[i].batches.empty()) lanes[i].batches.back().resize(lane_mark_frames[i]);
        lanes[i].fill = lane_mark_fill[i];
      }
      for (auto it = link_first_lane.begin(); it != link_first_lane.end();)
        it = it->second >= static_cast<int>(lanes_before) ? link_first_lane.erase(it) : std::next(it);
      planned_.ok = 0;
      planned_.failed_layer = layer;
      std::snprintf(planned_.error, sizeof planned_.error, "%s", e.what());
      break;
    }
    planned_.carryover_bytes += delta.carryover_bytes;
    planned_.local_copy_bytes += delta.local_copy_bytes;
    planned_.bytes_moved += delta.bytes_moved;
    planned_.layers_processed++;
    for (std::size_t d = 0; d < devices_.size(); ++d)
      programs_[d].layers.push_back({layer, mark[d], programs_[d].local.size()});
  }
  if (planned_.failed_layer < 0) planned_.ok = 1;

  // staging memory: slots + ready flags on the destination device, credit
  // flags on the source device
  std::vector<std::size_t> ring_need(devices_.size(), 0), flag_need(devices_.size(), 0);
  std::map<int, std::int64_t> ring_per_dst;
  for (const auto& lb : lanes) {
    ring_need[static_cast<std::size_t>(lb.ddev)] += lb.slot_bytes * static_cast<std::uint64_t>(K);
    flag_need[static_cast<std::size_t>(lb.ddev)] += align_up(sizeof(std::uint64_t) * K, kAlign);
    flag_need[static_cast<std::size_t>(lb.sdev)] += align_up(sizeof(std::uint64_t) * K, kAlign);
    ring_per_dst[lb.dst_rank] += static_cast<std::int64_t>(lb.slot_bytes) * K;
  }
  for (const auto& kv : ring_per_dst) planned_.peak_staging_bytes = std::max(planned_.peak_staging_bytes, kv.second);
  std::vector<std::size_t> ring_off(devices_.size(), 0), flag_off(devices_.size(), 0);
  for (std::size_t d = 0; d < devices_.size(); ++d) {
    rings_.emplace_back(devices_[d].ordinal, ring_need[d] + flag_need[d]);
    if (ring_need[d] + flag_need[d]) {
      DeviceGuard g(devices_[d].ordinal);
      cuda_check(cudaMemset(rings_.back().data(), 0, ring_need[d] + flag_need[d]), "ring memset");
    }
    flag_off[d] = ring_need[d];
  }
  for (auto& lb : lanes) {
    const auto dd = static_cast<std::size_t>(lb.ddev), sd = static_cast<std::size_t>(lb.sdev);
    lb.slots = rings_[dd].data() + ring_off[dd];
    ring_off[dd] += lb.slot_bytes * static_cast<std::uint64_t>(K);
    lb.ready = reinterpret_cast<std::uint64_t*>(rings_[dd].data() + flag_off[dd]);
    flag_off[dd] += align_up(sizeof(std::uint64_t) * K, kAlign);
    lb.credit = reinterpret_cast<std::uint64_t*>(rings_[sd].data() + flag_off[sd]);
    flag_off[sd] += align_up(sizeof(std::uint64_t) * K, kAlign);
  }

  // serialise lanes / batches / frames (global tables, uploaded to every device)
  std::vector<rs_lane_desc> all_lanes;
  std::vector<rs_batch_desc> batches;
  std::vector<rs_copy_desc> frames;
  for (const auto& lb : lanes) {
    rs_lane_desc L{};
    L.slot_base = L.slot_base_rx = reinterpret_cast<std::uint64_t>(lb.slots);
    L.slot_bytes = lb.slot_bytes;
    L.ready_flags = L.ready_flags_rx = reinterpret_cast<std::uint64_t>(lb.ready);
    L.credit_flags = L.credit_flags_tx = reinterpret_cast<std::uint64_t>(lb.credit);
    L.slots = static_cast<std::uint32_t>(K);
    L.batch0 = static_cast<std::uint32_t>(batches.size());
    L.nbatches = static_cast<std::uint32_t>(lb.batches.size());
    for (std::size_t b = 0; b < lb.batches.size(); ++b) {
      const std::uint64_t slot_addr = reinterpret_cast<std::uint64_t>(lb.slots) + (b % static_cast<std::size_t>(K)) * lb.slot_bytes;
      rs_batch_desc B{};
      B.pack0 = static_cast<std::uint32_t>(frames.size());
      for (const auto& f : lb.batches[b]) {
        append_copy(frames, reinterpret_cast<std::uint64_t>(f.se->ptr), f.se->view, slot_addr + f.off, f.region,
                    f.region, f.eb, static_cast<std::uint32_t>(f.layer));
        B.bytes += static_cast<std::uint64_t>(f.region.element_count() * f.eb);
      }
      B.npack = static_cast<std::uint32_t>(frames.size()) - B.pack0;
      B.unpack0 = static_cast<std::uint32_t>(frames.size());
      for (const auto& f : lb.batches[b])
        append_copy(frames, slot_addr + f.off, f.region, reinterpret_cast<std::uint64_t>(f.de->ptr), f.de->view,
                    f.region, f.eb, static_cast<std::uint32_t>(f.layer));
      B.nunpack = static_cast<std::uint32_t>(frames.size()) - B.unpack0;
      batches.push_back(B);
    }
    all_lanes.push_back(L);
  }
  assign_items(frames, 0, 0, 1ull << 16);  // rows_per_item inside frames (per-warp slices)
  for (std::size_t d = 0; d < devices_.size(); ++d) {
    DeviceProgram& p = programs_[d];
    p.batches = batches;
    p.frames = frames;
    std::vector<rs_lane_desc> tx, rx;
    for (std::size_t i = 0; i < lanes.size(); ++i) {
      if (static_cast<std::size_t>(lanes[i].sdev) == d) tx.push_back(all_lanes[i]);
    }
    for (std::size_t i = 0; i < lanes.size(); ++i) {
      if (static_cast<std::size_t>(lanes[i].ddev) == d) rx.push_back(all_lanes[i]);
    }
    p.lanes = tx;
    p.lanes.insert(p.lanes.end(), rx.begin(), rx.end());
  }
  staged_tx_.assign(devices_.size(), 0);
  staged_rx_.assign(devices_.size(), 0);
  for (const auto& lb : lanes) {
    staged_tx_[static_cast<std::size_t>(lb.sdev)]++;
    staged_rx_[static_cast<std::size_t>(lb.ddev)]++;
  }
}

void Engine::upload_programs() {
  for (std::size_t d = 0; d < devices_.size(); ++d) {
    DeviceProgram& p = programs_[d];
    const Device& dv = devices_[d];
    std::uint64_t bytes = 0;
    p.all_aligned = true;
    for (const auto& c : p.local) {
      bytes += bytes_of(c);
      p.all_aligned = p.all_aligned && c.vec_log2 == 4;
    }
    p.local_bytes = bytes;
    std::uint64_t item_bytes = static_cast<std::uint64_t>(opts_.item_bytes);
    if (item_bytes == 0) {
      // ~8 items per worker (warp, or bulk-issuer CTA) for load balance
      const int variant = copy_variant(static_cast<int>(d));
      const std::uint64_t workers = variant == 3 ? static_cast<std::uint64_t>(dv.sms)
                                                 : static_cast<std::uint64_t>(copy_grid(static_cast<int>(d))) * 8;
      item_bytes = std::clamp<std::uint64_t>(bytes / (workers * 8 + 1), 32768, variant == 3 ? 8u << 20 : 1u << 20);
    }
    // item ranges per layer
    std::uint64_t item = 0;
    for (auto& lr : p.layers) {
      const std::size_t first = static_cast<std::size_t>(lr.item_begin), last = static_cast<std::size_t>(lr.item_end);
      std::vector<rs_copy_desc> tmp(p.local.begin() + static_cast<std::ptrdiff_t>(first),
                                    p.local.begin() + static_cast<std::ptrdiff_t>(last));
      const std::uint64_t end = assign_items(tmp, 0, item, item_bytes);
      std::copy(tmp.begin(), tmp.end(), p.local.begin() + static_cast<std::ptrdiff_t>(first));
      lr.item_begin = item;
      lr.item_end = end;
      item = end;
    }
    p.local_items = item;
    p.local_item0.resize(p.local.size());
    for (std::size_t i = 0; i < p.local.size(); ++i) p.local_item0[i] = p.local[i].item0;
    DeviceGuard g(dv.ordinal);
    p.d_local = DeviceBuffer(dv.ordinal, p.local.size() * sizeof(rs_copy_desc));
    p.d_item0 = DeviceBuffer(dv.ordinal, p.local_item0.size() * sizeof(std::uint64_t));
    p.d_local.upload(p.local.data(), p.local.size() * sizeof(rs_copy_desc), dv.stream);
    p.d_item0.upload(p.local_item0.data(), p.local_item0.size() * sizeof(std::uint64_t), dv.stream);
    if (opts_.mode == RS_MODE_STAGED) {
      p.d_lanes = DeviceBuffer(dv.ordinal, p.lanes.size() * sizeof(rs_lane_desc));
      p.d_batches = DeviceBuffer(dv.ordinal, p.batches.size() * sizeof(rs_batch_desc));
      p.d_frames = DeviceBuffer(dv.ordinal, p.frames.size() * sizeof(rs_copy_desc));
      p.d_error = DeviceBuffer(dv.ordinal, sizeof(unsigned int));
      p.d_lanes.upload(p.lanes.data(), p.lanes.size() * sizeof(rs_lane_desc), dv.stream);
      p.d_batches.upload(p.batches.data(), p.batches.size() * sizeof(rs_batch_desc), dv.stream);
      p.d_frames.upload(p.frames.data(), p.frames.size() * sizeof(rs_copy_desc), dv.stream);
      cuda_check(cudaMemsetAsync(p.d_error.data(), 0, sizeof(unsigned int), dv.stream), "memset");
    }
    cuda_check(cudaStreamSynchronize(dv.stream), "program upload");
  }
}

// --------------------------------------------------------------------- run

rs_exec_report Engine::run() {
  if (!prepared_) throw DomainError("engine: prepare a plan first");
  rs_exec_report rep = planned_;
  const auto t0 = std::chrono::steady_clock::now();
  int launches = 0;
  for (auto& dv : devices_) {
    DeviceGuard g(dv.ordinal);
    cuda_check(cudaEventRecord(dv.ev_begin, dv.stream), "event");
  }
  if (opts_.mode == RS_MODE_DIRECT) {
    if (!opts_.strict_layers) {
      for (std::size_t d = 0; d < devices_.size(); ++d) {
        DeviceProgram& p = programs_[d];
        if (!p.local_items) continue;
        DeviceGuard g(devices_[d].ordinal);
        cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                                  reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                                  static_cast<std::uint32_t>(p.local.size()), 0, p.local_items,
                                  copy_grid(static_cast<int>(d)), copy_variant(static_cast<int>(d)), devices_[d].stream),
                   "copy kernel launch");
        ++launches;
      }
    } else {
      const std::size_t nl = programs_.empty() ? 0 : programs_[0].layers.size();
      for (std::size_t li = 0; li < nl; ++li) {
        for (std::size_t d = 0; d < devices_.size(); ++d) {
          DeviceProgram& p = programs_[d];
          const LayerRange& lr = p.layers[li];
          if (lr.item_end == lr.item_begin) continue;
          DeviceGuard g(devices_[d].ordinal);
          cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                                    reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                                    static_cast<std::uint32_t>(p.local.size()), lr.item_begin, lr.item_end,
                                    copy_grid(static_cast<int>(d)), copy_variant(static_cast<int>(d)), devices_[d].stream),
                     "copy kernel launch");
          ++launches;
        }
        if (devices_.size() > 1) {  // layer barrier across devices
          for (auto& a : devices_) {
            DeviceGuard g(a.ordinal);
            cuda_check(cudaEventRecord(a.ev_end, a.stream), "event");
            for (auto& b : devices_)
              if (&a != &b) cuda_check(cudaStreamWaitEvent(b.stream, a.ev_end, 0), "wait");
          }
        }
      }
    }
  } else {
    epoch_ += 1ull << 32;
    for (std::size_t d = 0; d < devices_.size(); ++d) {
      DeviceProgram& p = programs_[d];
      const int ntx = staged_tx_[d], nrx = staged_rx_[d];
      const int cap = grid_for(static_cast<int>(d), 2);
      if (ntx + nrx >= cap)
        throw DomainError("staged: " + std::to_string(ntx + nrx) + " ring lanes exceed the co-resident CTA capacity " +
                          std::to_string(cap) + "; lower lanes_per_link");
      if (!ntx && !nrx && !p.local_items) continue;
      DeviceGuard g(devices_[d].ordinal);
      const auto* lanes = reinterpret_cast<const rs_lane_desc*>(p.d_lanes.data());
      cuda_check(rs_launch_exchange(lanes, static_cast<std::uint32_t>(ntx), lanes + ntx, static_cast<std::uint32_t>(nrx),
                                    reinterpret_cast<const rs_batch_desc*>(p.d_batches.data()),
                                    reinterpret_cast<const rs_copy_desc*>(p.d_frames.data()),
                                    reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                                    reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                                    static_cast<std::uint32_t>(p.local.size()), p.local_items, epoch_,
                                    reinterpret_cast<unsigned int*>(p.d_error.data()), 200000000ull,
                                    cap - ntx - nrx, devices_[d].stream),
                 "exchange kernel launch");
      ++launches;
    }
  }
  for (auto& dv : devices_) {
    DeviceGuard g(dv.ordinal);
    cuda_check(cudaEventRecord(dv.ev_end, dv.stream), "event");
  }
  double worst = 0;
  for (auto& dv : devices_) {
    DeviceGuard g(dv.ordinal);
    cuda_check(cudaEventSynchronize(dv.ev_end), "reshard kernels");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, dv.ev_begin, dv.ev_end), "elapsed");
    worst = std::max(worst, static_cast<double>(ms));
  }
  if (opts_.mode == RS_MODE_STAGED) {
    for (std::size_t d = 0; d < devices_.size(); ++d) {
      unsigned int flag = 0;
      DeviceGuard g(devices_[d].ordinal);
      cuda_check(cudaMemcpy(&flag, programs_[d].d_error.data(), sizeof flag, cudaMemcpyDeviceToHost), "error flag");
      if (flag) {
        rep.ok = 0;
        std::snprintf(rep.error, sizeof rep.error, "staged transfer: ring wait timed out on device %d", devices_[d].ordinal);
        cuda_check(cudaMemset(programs_[d].d_error.data(), 0, sizeof flag), "memset");
      }
    }
  }
  rep.device_ms = worst;
  rep.kernel_launches = launches;
  rep.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return rep;
}

rs_exec_report Engine::run_host(void* const* host_src, void* const* host_dst, int window_layers) {
  (void)window_layers;
  if (!prepared_) throw DomainError("engine: prepare a plan first");
  const auto t0 = std::chrono::steady_clock::now();
  if (opts_.mode != RS_MODE_DIRECT) {
    // staged transfers run as one launch: stage everything in, run, stage out
    for (std::size_t k = 0; k < stores_[RS_SRC].entries.size(); ++k) {
      const Entry& e = stores_[RS_SRC].entries[k];
      const Device& dv = devices_[static_cast<std::size_t>(e.dev)];
      DeviceGuard g(dv.ordinal);
      cuda_check(cudaMemcpyAsync(e.ptr, host_src[k], static_cast<std::size_t>(e.nbytes), cudaMemcpyHostToDevice,
                                 dv.stream), "H2D");
    }
    rs_exec_report rep = run();
    for (std::size_t k = 0; k < stores_[RS_DST].entries.size(); ++k) {
      const Entry& e = stores_[RS_DST].entries[k];
      const Device& dv = devices_[static_cast<std::size_t>(e.dev)];
      DeviceGuard g(dv.ordinal);
      cuda_check(cudaMemcpyAsync(host_dst[k], e.ptr, static_cast<std::size_t>(e.nbytes), cudaMemcpyDeviceToHost,
                                 dv.stream), "D2H");
    }
    for (auto& dv : devices_) {
      DeviceGuard g(dv.ordinal);
      cuda_check(cudaStreamSynchronize(dv.stream), "D2H");
    }
    rep.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return rep;
  }

  // DIRECT: layer pipeline over three streams per device.  Layer l's source
  // shards go H2D (h2d stream), its copy kernel waits for them (compute
  // stream), its destination shards go D2H once every device finished layer l
  // (d2h stream) -- so H2D of l+1, the kernel of l and D2H of l-1 overlap and
  // PCIe runs full duplex.  The layers are the plan's (executor.cpp:134-138).
  rs_exec_report rep = planned_;
  const std::size_t nlayers = programs_.empty() ? 0 : programs_[0].layers.size();
  std::map<int, std::size_t> layer_slot;
  for (std::size_t li = 0; li < nlayers; ++li) layer_slot[programs_[0].layers[li].layer] = li;
  const std::size_t ndev = devices_.size();
  std::vector<cudaEvent_t> ev_in(nlayers * ndev), ev_done(nlayers * ndev);
  auto mk = [](cudaEvent_t& e) { cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event"); };
  for (std::size_t d = 0; d < ndev; ++d) {
    DeviceGuard g(devices_[d].ordinal);
    for (std::size_t li = 0; li < nlayers; ++li) {
      mk(ev_in[li * ndev + d]);
      mk(ev_done[li * ndev + d]);
    }
    cuda_check(cudaEventRecord(devices_[d].ev_begin, devices_[d].h2d), "event");
  }
  auto layer_of = [&](const Store& s, const Entry& e) { return s.model.tensors[e.ti].layer; };
  // H2D per layer, in layer order
  for (std::size_t li = 0; li < nlayers; ++li) {
    const int layer = programs_[0].layers[li].layer;
    for (std::size_t k = 0; k < stores_[RS_SRC].entries.size(); ++k) {
      const Entry& e = stores_[RS_SRC].entries[k];
      if (layer_of(stores_[RS_SRC], e) != layer) continue;
      const Device& dv = devices_[static_cast<std::size_t>(e.dev)];
      DeviceGuard g(dv.ordinal);
      cuda_check(cudaMemcpyAsync(e.ptr, host_src[k], static_cast<std::size_t>(e.nbytes), cudaMemcpyHostToDevice,
                                 dv.h2d), "H2D");
    }
    for (std::size_t d = 0; d < ndev; ++d) {
      DeviceGuard g(devices_[d].ordinal);
      cuda_check(cudaEventRecord(ev_in[li * ndev + d], devices_[d].h2d), "event");
    }
  }
  // kernels per layer; a layer's copies may read any device's sources
  int launches = 0;
  for (std::size_t li = 0; li < nlayers; ++li) {
    for (std::size_t d = 0; d < ndev; ++d) {
      DeviceProgram& p = programs_[d];
      const LayerRange& lr = p.layers[li];
      DeviceGuard g(devices_[d].ordinal);
      for (std::size_t o = 0; o < ndev; ++o)
        cuda_check(cudaStreamWaitEvent(devices_[d].stream, ev_in[li * ndev + o], 0), "wait");
      if (lr.item_end > lr.item_begin) {
        cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                                  reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                                  static_cast<std::uint32_t>(p.local.size()), lr.item_begin, lr.item_end,
                                  copy_grid(static_cast<int>(d)), copy_variant(static_cast<int>(d)), devices_[d].stream),
                   "copy kernel launch");
        ++launches;
      }
      cuda_check(cudaEventRecord(ev_done[li * ndev + d], devices_[d].stream), "event");
    }
  }
  // D2H per layer after every device finished that layer
  for (std::size_t li = 0; li < nlayers; ++li) {
    const int layer = programs_[0].layers[li].layer;
    for (std::size_t d = 0; d < ndev; ++d) {
      DeviceGuard g(devices_[d].ordinal);
      for (std::size_t o = 0; o < ndev; ++o)
        cuda_check(cudaStreamWaitEvent(devices_[d].d2h, ev_done[li * ndev + o], 0), "wait");
    }
    for (std::size_t k = 0; k < stores_[RS_DST].entries.size(); ++k) {
      const Entry& e = stores_[RS_DST].entries[k];
      if (layer_of(stores_[RS_DST], e) != layer) continue;
      const Device& dv = devices_[static_cast<std::size_t>(e.dev)];
      DeviceGuard g(dv.ordinal);
      cuda_check(cudaMemcpyAsync(host_dst[k], e.ptr, static_cast<std::size_t>(e.nbytes), cudaMemcpyDeviceToHost,
                                 dv.d2h), "D2H");
    }
  }
  double worst = 0;
  for (auto& dv : devices_) {
    DeviceGuard g(dv.ordinal);
    cuda_check(cudaEventRecord(dv.ev_end, dv.d2h), "event");
    cuda_check(cudaEventSynchronize(dv.ev_end), "host-store reshard");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, dv.ev_begin, dv.ev_end), "elapsed");
    worst = std::max(worst, static_cast<double>(ms));
  }
  for (std::size_t i = 0; i < ev_in.size(); ++i) {
    cudaEventDestroy(ev_in[i]);
    cudaEventDestroy(ev_done[i]);
  }
  rep.device_ms = worst;
  rep.kernel_launches = launches;
  rep.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return rep;
}

}  // namespace rsb
