// Device reshard engine.
//
// prepare() turns a TransferPlan into per-device work lists, validating every
// task and carryover with the reference executor's integrity rules and error
// messages (proj/src/executor.cpp:142-206): a failing layer is reported as
// failed_layer with every earlier layer executed, like execute_plan's
// per-layer try/catch (executor.cpp:210-215).
//
// Devices are global *slots*: every process lays out the same stores over the
// same slots and drives the slots it owns (one process per GPU, or one
// process for several GPUs).  Peer arenas are mapped with CUDA IPC, so a
// process reaches a peer GPU's shards and staging rings by plain loads and
// stores over NVLink.
//
// DIRECT mode: every task and carryover is one strided->strided copy issued
//   by the slot holding its source (push); destinations on other GPUs are
//   written through the peer mapping.  Zero staging.
// STAGED mode: cross-rank tasks are chunked to the ring slot size and
//   streamed through per-(src,dst) single-producer/single-consumer rings that
//   live in the destination's staging budget B (the comm arena); local tasks
//   and carryovers run as DIRECT copies in the same launch.
#include "engine.hpp"

#include <algorithm>
#include <tuple>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <map>
#include <set>

#include "compile.hpp"
#include "engine_internal.hpp"
#include "kernels.h"

namespace rsb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    // clear a non-sticky error (e.g. a failed cudaMalloc) so the next launch's
    // cudaGetLastError does not report it again; sticky faults stay sticky
    cudaGetLastError();
    throw SystemError(std::string(what) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
  }
}

using namespace detail;


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

ImportedArena::ImportedArena(int device, const cudaIpcMemHandle_t& h) : device_(device) {
  DeviceGuard g(device);
  void* p = nullptr;
  cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  ptr_ = static_cast<char*>(p);
}

ImportedArena::~ImportedArena() {
  if (ptr_) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    cudaIpcCloseMemHandle(ptr_);
    cudaSetDevice(prev);
  }
}

ImportedArena& ImportedArena::operator=(ImportedArena&& o) noexcept {
  if (this != &o) {
    this->~ImportedArena();
    device_ = o.device_;
    ptr_ = o.ptr_;
    o.ptr_ = nullptr;
  }
  return *this;
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
  if (opts.strict_layers && opts.mode == RS_MODE_XFER)
    // XFER rounds are host-driven chunk rounds of the comparator, not layers
    throw DomainError("engine: strict_layers applies to RS_MODE_DIRECT and RS_MODE_STAGED");
  if (opts.strict_layers && opts.mode == RS_MODE_STAGED && (opts.ring_discard & 8))
    // the layer barriers live in the classic lane loop
    throw DomainError("engine: strict_layers needs classic ring lanes (ring_discard without bit 8)");
  for (int i = 0; i < opts.num_devices; ++i)
    for (int j = 0; j < i; ++j)
      if (opts.device_ids[i] == opts.device_ids[j])
        // two slots of one process on one GPU would run two launches whose ring
        // lanes wait on each other without being co-resident
        throw DomainError("engine: device " + std::to_string(opts.device_ids[i]) +
                          " listed twice; one slot per GPU per process (several processes may share a GPU)");
  if (opts.mode != RS_MODE_DIRECT && opts.mode != RS_MODE_STAGED && opts.mode != RS_MODE_XFER)
    throw DomainError("engine: unknown mode");
  if (opts.ring_same_slot < 0 || opts.ring_same_slot > 2)
    throw DomainError("engine: ring_same_slot must be 0 (auto), 1 (rings) or 2 (direct)");
  if (opts.ring_kernel < 0 || opts.ring_kernel > 2)
    throw DomainError("engine: ring_kernel must be 0 (auto), 1 (classic) or 2 (stream)");
  // stream lanes: 2 x 16 KB stages -> 7 lane CTAs per SM; more lanes beat
  // deeper lanes (profiles/r2/stream_sweep.jsonl)
  if (opts_.ring_stages == 0) opts_.ring_stages = 2;
  if (opts_.ring_stages != 1 && opts_.ring_stages != 2 && opts_.ring_stages != 3 && opts_.ring_stages != 4 && opts_.ring_stages != 6 &&
      opts_.ring_stages != 8 && opts_.ring_stages != 10 && opts_.ring_stages != 13)
    throw DomainError("engine: ring_stages must be 1, 2, 3, 4, 6, 8, 10 or 13");
  if (opts_.ring_cta_threads == 0) opts_.ring_cta_threads = 256;
  if (opts_.ring_cta_threads != 256 && opts_.ring_cta_threads != 512 && opts_.ring_cta_threads != 1024)
    throw DomainError("engine: ring_cta_threads must be 256, 512 or 1024");
  if (opts_.slots_per_link == 0) opts_.slots_per_link = 2;  // ring depth default (profiles/r1/ring_sweep_v3.jsonl)
  if (opts_.slots_per_link < 2) opts_.slots_per_link = 2;
  if (opts_.lanes_per_link < 0) opts_.lanes_per_link = 0;  // 0: automatic (compile_staged)
  nslots_ = opts.world_slots > 0 ? opts.world_slots : opts.num_devices;
  first_local_ = opts.first_local_slot;
  if (first_local_ < 0 || first_local_ + opts.num_devices > nslots_)
    throw DomainError("engine: local slots [" + std::to_string(first_local_) + "," +
                      std::to_string(first_local_ + opts.num_devices) + ") outside world of " +
                      std::to_string(nslots_) + " slots");
  int count = 0;
  cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  for (int i = 0; i < opts.num_devices; ++i) {
    Device d;
    d.ordinal = opts.device_ids[i];
    d.slot = first_local_ + i;
    if (d.ordinal < 0 || d.ordinal >= count) throw DomainError("engine: bad device id " + std::to_string(d.ordinal));
    DeviceGuard g(d.ordinal);
    cuda_check(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, d.ordinal), "sm count");
    cuda_check(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&d.h2d, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&d.d2h, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreate(&d.ev_begin), "event");
    cuda_check(cudaEventCreate(&d.ev_end), "event");
    cuda_check(cudaEventCreate(&d.ev_call), "event");
    cuda_check(cudaStreamCreateWithFlags(&d.aux, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreateWithFlags(&d.ev_aux, cudaEventDisableTiming), "event");
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
  comm_imported_.resize(static_cast<std::size_t>(nslots_));
  comm_imported_bytes_.assign(static_cast<std::size_t>(nslots_), 0);
}

Engine::~Engine() {
  programs_.clear();
  comm_.clear();
  comm_imported_.clear();
  for (auto& s : stores_) {
    s.arenas.clear();
    s.imported.clear();
  }
  for (auto& d : devices_) {
    cudaSetDevice(d.ordinal);
    if (d.stream) cudaStreamDestroy(d.stream);
    if (d.h2d) cudaStreamDestroy(d.h2d);
    if (d.d2h) cudaStreamDestroy(d.d2h);
    if (d.ev_begin) cudaEventDestroy(d.ev_begin);
    if (d.ev_end) cudaEventDestroy(d.ev_end);
    if (d.ev_call) cudaEventDestroy(d.ev_call);
    if (d.aux) cudaStreamDestroy(d.aux);
    if (d.ev_aux) cudaEventDestroy(d.ev_aux);
  }
}

int Engine::local_of(int slot) const {
  const int i = slot - first_local_;
  return (i >= 0 && i < num_devices()) ? i : -1;
}

void Engine::layout(int which, const reshard::ModelSpec& model, const reshard::ParallelConfig& cfg,
                    const std::vector<int>& rank_slot) {
  if (which != RS_SRC && which != RS_DST) throw DomainError("store: which must be RS_SRC or RS_DST");
  if (auto v = model.validate(); !v.empty()) throw DomainError("model: " + v.front());
  if (auto v = reshard::validate_config(cfg, model); !v.empty()) throw DomainError("config: " + v.front());
  if (static_cast<int>(rank_slot.size()) != cfg.world_size())
    throw DomainError("store: rank_device must have one entry per rank");
  for (int d : rank_slot)
    if (d < 0 || d >= nslots_) throw DomainError("store: rank_device entry out of range");
  Store s;
  s.model = model;
  s.config = cfg;
  s.arena_bytes.assign(static_cast<std::size_t>(nslots_), 0);
  for (std::uint32_t ti = 0; ti < model.tensors.size(); ++ti) {
    const auto& t = model.tensors[ti];
    for (const auto& [rank, v] : reshard::owners(t, cfg)) {
      Entry e;
      e.ti = ti;
      e.rank = rank;
      e.slot = rank_slot[static_cast<std::size_t>(cfg.index_of(rank))];
      e.view = v;
      e.nbytes = v.element_count() * model.element_bytes(t);
      if (auto r = reshard::bucket_range(model, ti, cfg, rank)) {  // flat-bucket distributed optimizer
        e.flat = true;
        e.flat_lo = r->first;
        e.flat_off = r->first * model.element_bytes(t);
        e.flat_elems = r->second - r->first;
        e.nbytes = (r->second - r->first) * model.element_bytes(t);
      }
      // deterministic arena offsets for every slot: peers compute the same
      auto& used = s.arena_bytes[static_cast<std::size_t>(e.slot)];
      e.off = used;
      used += align_up(static_cast<std::size_t>(e.nbytes), kAlign);
      s.index.emplace(key(rank, ti), static_cast<std::uint32_t>(s.entries.size()));
      s.entries.push_back(e);
    }
  }
  s.imported.resize(static_cast<std::size_t>(nslots_));
  s.laid_out = true;
  stores_[which] = std::move(s);
  if (which == RS_DST) {
    comm_.clear();
    for (auto& c : comm_imported_) c.reset();
  }
  prepared_ = false;
}

void Engine::check_laid_out() const {
  if (!stores_[RS_SRC].laid_out) throw DomainError("src store not laid out");
  if (!stores_[RS_DST].laid_out) throw DomainError("dst store not laid out");
}

void Engine::alloc(int which) {
  Store& s = stores_[which];
  if (!s.laid_out) throw DomainError("store: layout first");
  if (window_layers_ > 0) {  // back to full device stores
    window_.clear();
    window_layers_ = 0;
    for (auto& st : stores_)
      for (auto& e : st.entries) e.ptr = nullptr;
  }
  s.arenas.clear();
  for (const auto& dv : devices_) s.arenas.emplace_back(dv.ordinal, s.arena_bytes[static_cast<std::size_t>(dv.slot)]);
  for (auto& e : s.entries) {
    const int l = local_of(e.slot);
    if (l >= 0) e.ptr = s.arenas[static_cast<std::size_t>(l)].data() + e.off;
  }
  prepared_ = false;
}

void Engine::set_window(int layers) {
  check_laid_out();
  if (layers < 1) throw DomainError("window: layers must be >= 1");
  const int L = stores_[RS_SRC].model.num_layers;
  window_.clear();
  for (auto& s : stores_) s.arenas.clear();
  for (const auto& dv : devices_) {
    // per model layer: bytes of this slot's source + destination shards
    std::vector<std::size_t> need(static_cast<std::size_t>(L), 0);
    for (const auto& s : stores_)
      for (const auto& e : s.entries)
        if (e.slot == dv.slot)
          need[static_cast<std::size_t>(s.model.tensors[e.ti].layer)] += align_up(static_cast<std::size_t>(e.nbytes), kAlign);
    const std::size_t slot_bytes = need.empty() ? 0 : *std::max_element(need.begin(), need.end());
    window_.emplace_back(dv.ordinal, slot_bytes * static_cast<std::size_t>(layers));
    char* base = window_.back().data();
    std::vector<std::size_t> used(static_cast<std::size_t>(L), 0);  // per layer: its own slot cursor
    for (auto& s : stores_)
      for (auto& e : s.entries) {
        if (e.slot != dv.slot) continue;
        const int layer = s.model.tensors[e.ti].layer;
        const auto w = static_cast<std::size_t>(layer % layers);
        // layer l's source then destination shards fill slot l % layers
        e.ptr = base + w * slot_bytes + used[static_cast<std::size_t>(layer)];
        used[static_cast<std::size_t>(layer)] += align_up(static_cast<std::size_t>(e.nbytes), kAlign);
      }
  }
  window_layers_ = layers;
  prepared_ = false;
}

void Engine::free_store(int which) {
  Store& s = stores_[which];
  s.arenas.clear();
  for (auto& a : s.imported) a.reset();
  for (auto& e : s.entries) e.ptr = nullptr;
  prepared_ = false;
}

void Engine::bind(int which, int rank, std::uint32_t ti, void* ptr, std::int64_t nbytes) {
  Store& s = stores_[which];
  if (!s.laid_out) throw DomainError("store: layout first");
  Entry* e = s.find(rank, ti);
  if (!e) throw DomainError(no_buffer(rank, ti));
  if (nbytes != e->nbytes)
    throw DomainError("store bind: buffer size " + std::to_string(nbytes) + " does not match view size " +
                      std::to_string(e->nbytes));
  e->ptr = static_cast<char*>(ptr);
  prepared_ = false;
}

// ------------------------------------------------------ comm arenas and IPC

std::int64_t Engine::export_arena(int which, int slot, void* handle) const {
  const int l = local_of(slot);
  if (l < 0) throw DomainError("export: slot " + std::to_string(slot) + " is not local");
  const char* base = nullptr;
  std::int64_t bytes = 0;
  if (which == RS_COMM) {
    if (static_cast<std::size_t>(l) >= comm_.size()) throw DomainError("export: comm arena not allocated");
    base = comm_[static_cast<std::size_t>(l)].data();
    bytes = static_cast<std::int64_t>(comm_[static_cast<std::size_t>(l)].size());
  } else {
    const Store& s = stores_[which];
    if (static_cast<std::size_t>(l) >= s.arenas.size()) throw DomainError("export: store arena not allocated");
    base = s.arenas[static_cast<std::size_t>(l)].data();
    bytes = static_cast<std::int64_t>(s.arenas[static_cast<std::size_t>(l)].size());
  }
  cudaIpcMemHandle_t h{};
  if (base) {
    DeviceGuard g(devices_[static_cast<std::size_t>(l)].ordinal);
    cuda_check(cudaIpcGetMemHandle(&h, const_cast<char*>(base)), "cudaIpcGetMemHandle");
  }
  std::memcpy(handle, &h, sizeof h);
  return bytes;
}

void Engine::import_arena(int which, int slot, const void* handle, std::int64_t bytes) {
  if (slot < 0 || slot >= nslots_) throw DomainError("import: slot out of range");
  if (local_of(slot) >= 0) return;  // own arena
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  // mapped through the first local device (peer access over NVLink)
  const int dev = devices_[0].ordinal;
  if (which == RS_COMM) {
    if (static_cast<std::size_t>(bytes) != comm_bytes(slot)) throw DomainError("import: comm arena size mismatch");
    comm_imported_[static_cast<std::size_t>(slot)] = bytes ? std::make_unique<ImportedArena>(dev, h) : nullptr;
    comm_imported_bytes_[static_cast<std::size_t>(slot)] = static_cast<std::size_t>(bytes);
  } else {
    Store& s = stores_[which];
    if (!s.laid_out) throw DomainError("import: lay out the store first");
    if (static_cast<std::size_t>(bytes) != s.arena_bytes[static_cast<std::size_t>(slot)])
      throw DomainError("import: arena size mismatch for slot " + std::to_string(slot) + " (layouts differ?)");
    auto& imp = s.imported[static_cast<std::size_t>(slot)];
    imp = bytes ? std::make_unique<ImportedArena>(dev, h) : nullptr;
    for (auto& e : s.entries)
      if (e.slot == slot) e.ptr = imp ? imp->data() + e.off : nullptr;
  }
  prepared_ = false;
}

// ------------------------------------------------------------- kernel knobs

int Engine::grid_for(int dev, int which_kernel) const {
  int per_sm = rs_kernel_max_blocks_per_sm(which_kernel);
  if (per_sm < 1) per_sm = 1;
  if (opts_.blocks_per_sm > 0) per_sm = std::min(per_sm, opts_.blocks_per_sm);
  return devices_[static_cast<std::size_t>(dev)].sms * per_sm;
}

// Resolved copy kernel of a device's program (RS_COPY_* numbering).
// RS_COPY_AUTO = the non-persistent TMA bulk copy (17) when every descriptor
// is 16 B aligned with runs <= 16 KB and nothing is stored into another slot,
// else the non-persistent LDG8 warp copy (15) -- see the default case.
int Engine::copy_variant(int dev) const {
  switch (opts_.copy_kernel) {
    case RS_COPY_LDG4: return 1;
    case RS_COPY_BULK: return programs_[static_cast<std::size_t>(dev)].all_aligned ? 3 : 1;
    case RS_COPY_LDG4_CS: return 4;
    case RS_COPY_LDG8_CS: return 5;
    case RS_COPY_LDG16: return 6;
    case RS_COPY_CTA8: return 7;
    case RS_COPY_LDG8_PF: return 13;
    case RS_COPY_LDG8_EF: return 14;
    case RS_COPY_LDG8_NP: return 15;
    case RS_COPY_TMA_NP: return programs_[static_cast<std::size_t>(dev)].max_row_bytes <= 16384 &&
                                        programs_[static_cast<std::size_t>(dev)].all_aligned ? 17 : 15;
    case RS_COPY_TMA_NP32: return programs_[static_cast<std::size_t>(dev)].max_row_bytes <= 32768 &&
                                          programs_[static_cast<std::size_t>(dev)].all_aligned ? 18 : 15;
    case RS_COPY_BULK_MW:
    case RS_COPY_BULK_MW + 1:
    case RS_COPY_BULK_MW + 2:
    case RS_COPY_BULK_MW + 3:
    case RS_COPY_BULK_MW + 4:  // issuer-count / ring-shape variants (copy_kernels.cu launch_bulk_mw)
      return programs_[static_cast<std::size_t>(dev)].all_aligned ? opts_.copy_kernel : 2;
    case RS_COPY_LDG8: return 2;
    // default: TMA bulk copy over a non-persistent grid when every descriptor is
    // 16 B aligned with rows <= 16 KB (all BASELINE plans), else LDG8 over a
    // non-persistent grid (profiles/r1/tma_np_sweep.jsonl, np_sweep.jsonl)
    default: {
      // (TMA bulk stores into another GPU's memory are unmeasured here -- one
      // GPU per box -- so a program with peer destinations keeps plain
      // st.global peer stores unless RS_COPY_TMA_NP is asked for explicitly)
      const DeviceProgram& p = programs_[static_cast<std::size_t>(dev)];
      return p.all_aligned && p.max_row_bytes <= 16384 && !p.peer_stores ? 17 : 15;
    }
  }
}

int Engine::copy_grid(int dev) const {
  const Device& d = devices_[static_cast<std::size_t>(dev)];
  switch (copy_variant(dev)) {
    case 2:
    case 5:
    case 13:
    case 14:
    case 15: {
      // 3 CTAs (24 warps) per SM at full size; a launch of a few GB is
      // ramp-dominated and runs faster with 4 (profiles/r1/item_sweep*.jsonl)
      const std::uint64_t lb = programs_.empty() ? 0 : programs_[static_cast<std::size_t>(dev)].launch_bytes;
      const int dflt = lb && lb < (4ull << 30) ? 4 : 3;
      int per_sm = std::max(1, rs_kernel_max_blocks_per_sm(3));
      per_sm = std::min(per_sm, opts_.blocks_per_sm > 0 ? opts_.blocks_per_sm : dflt);
      return d.sms * per_sm;
    }
    case 3:
    case 8:
    case 9:
    case 10:
    case 11:
    case 12: return d.sms;  // one bulk-ring CTA (1..16 issuers) per SM
    case 6:
    case 7: {
      int per_sm = std::max(1, rs_kernel_max_blocks_per_sm(copy_variant(dev) == 6 ? 5 : 6));
      per_sm = std::min(per_sm, opts_.blocks_per_sm > 0 ? opts_.blocks_per_sm : 3);
      return d.sms * per_sm;
    }
    default: return grid_for(dev, 0);
  }
}

// ---------------------------------------------------------------- patterns

void Engine::fill_pattern(int which, std::uint64_t seed) { (void)pattern_pass(which, seed, false, nullptr); }

std::int64_t Engine::verify_pattern(int which, std::uint64_t seed, std::int64_t* first_bad) {
  return pattern_pass(which, seed, true, first_bad);
}

// Fill / verify the entries on this process's slots.
std::int64_t Engine::pattern_pass(int which, std::uint64_t seed, bool verify, std::int64_t* first_bad) {
  const Store& s = stores_[which];
  if (!s.laid_out) throw DomainError("store: layout first");
  if (window_layers_ > 0) throw DomainError("pattern fill/verify needs full device stores (this store is windowed)");
  std::int64_t total_bad = 0;
  std::uint64_t first = ~0ull;
  for (int d = 0; d < num_devices(); ++d) {
    const Device& dv = devices_[static_cast<std::size_t>(d)];
    std::vector<rs_pattern_desc> descs;
    std::uint64_t bytes = 0;
    for (const auto& e : s.entries) {
      if (e.slot != dv.slot) continue;
      if (!e.ptr) throw DomainError("store: entry without device memory");
      bytes += static_cast<std::uint64_t>(e.nbytes);
    }
    if (bytes == 0) continue;
    const int grid = grid_for(d, 1);
    const std::uint64_t warps = static_cast<std::uint64_t>(grid) * 8;
    const std::uint64_t item_bytes = std::clamp<std::uint64_t>(bytes / (warps * 8), 16384, 1 << 20);
    for (std::uint32_t k = 0; k < s.entries.size(); ++k) {
      const Entry& e = s.entries[k];
      if (e.slot != dv.slot) continue;
      const auto& t = s.model.tensors[e.ti];
      const std::int64_t eb = s.model.element_bytes(t);
      if (!e.flat) {
        append_pattern(descs, addr(e.ptr), t, e.view, eb, e.ti, k, item_bytes);
        continue;
      }
      // a flat-bucket shard: one pattern run per contiguous box of its range
      std::int64_t at = 0;
      for (const auto& b : reshard::flat_range_boxes(e.view, e.flat_lo, e.flat_lo + e.nbytes / eb)) {
        append_pattern(descs, addr(e.ptr) + static_cast<std::uint64_t>(at), t, b, eb, e.ti, k, item_bytes);
        at += b.element_count() * eb;
      }
    }
    std::vector<std::uint64_t> item0(descs.size());
    std::uint64_t items = 0;
    for (std::size_t i = 0; i < descs.size(); ++i) {
      descs[i].item0 = items;
      item0[i] = items;
      items += (descs[i].rows + descs[i].rows_per_item - 1) / descs[i].rows_per_item;
    }
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
                                 static_cast<std::uint32_t>(descs.size()), items, seed, verify ? 1 : 0, counters,
                                 counters + 1, grid, dv.stream),
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

void Engine::prepare(const reshard::TransferPlan& plan, std::uint64_t plan_id) {
  prepared_id_ = 0;
  check_laid_out();
  const auto& m = stores_[RS_SRC].model;
  if (plan.tensor_ids.size() != m.tensors.size())
    throw DomainError("plan does not match the store model (tensor count)");
  for (std::size_t i = 0; i < m.tensors.size(); ++i)
    if (plan.tensor_ids[i] != m.tensors[i].tensor_id)
      throw DomainError("plan does not match the store model (tensor " + plan.tensor_ids[i] + ")");
  if (stores_[RS_DST].model.tensors.size() != m.tensors.size())
    throw DomainError("src and dst stores use different models");
  for (int w = 0; w < 2; ++w)  // every shard on this process's slots needs memory
    for (const auto& e : stores_[w].entries)
      if (local_of(e.slot) >= 0 && !e.ptr && e.nbytes)
        throw DomainError(std::string(w ? "dst" : "src") + " store: entry rank " + std::to_string(e.rank) +
                          " tensor " + std::to_string(e.ti) + " has no device memory");

  planned_ = rs_exec_report{};
  planned_.failed_layer = -1;
  planned_total_bytes_ = plan.total_bytes();
  std::set<int> layers;
  for (const auto& kv : plan.tasks_by_layer) layers.insert(kv.first);
  for (const auto& kv : plan.carryover_by_layer) layers.insert(kv.first);
  plan_layers_.assign(layers.begin(), layers.end());

  programs_.clear();
  programs_.resize(devices_.size());
  if (opts_.mode == RS_MODE_DIRECT) {
    compile_direct(plan);
  } else if (opts_.mode == RS_MODE_XFER) {
    compile_xfer(plan);
  } else {
    // The ring area is B per destination rank of the slot, so it follows the
    // dst layout: a live-handoff chain changes it every generation.
    // The comm arena must hold this plan's rings for the current dst layout:
    // B per rank (rs_comm_alloc) or plan-sized (rs_comm_alloc_plan).  One
    // process: (re)allocate plan-sized when it does not.  Several processes:
    // the arenas are IPC-shared, so every process must re-run the alloc.
    bool stale = !comm_layout_valid_ || comm_.size() != devices_.size();
    for (std::size_t d = 0; !stale && d < devices_.size(); ++d)
      stale = comm_[d].size() != comm_bytes(devices_[d].slot);
    if (!stale) {
      const RingGeometry geo = ring_geometry(plan);
      std::map<int, int> slot_of_rank;
      for (const auto& e : stores_[RS_DST].entries) slot_of_rank[e.rank] = e.slot;
      for (const auto& [r, need] : geo.ring_bytes_of) {
        const auto& regs = comm_layout_.regions.at(static_cast<std::size_t>(slot_of_rank.at(r)));
        auto it = regs.find(r);
        if (it == regs.end() || it->second.second < need) stale = true;
      }
    }
    for (int s = 0; s < nslots_; ++s)
      if (local_of(s) < 0 && comm_imported_[static_cast<std::size_t>(s)] &&
          comm_imported_bytes_[static_cast<std::size_t>(s)] != comm_bytes(s))
        throw DomainError("staged: peer comm arena of slot " + std::to_string(s) +
                          " was sized for another dst layout or plan; re-run rs_comm_alloc_plan on every process "
                          "and re-exchange the RS_COMM handles");
    if (stale) {
      if (nslots_ > num_devices())
        throw DomainError("staged: comm arena missing or sized for another dst layout or plan; run "
                          "rs_comm_alloc_plan on every process and exchange the RS_COMM handles");
      comm_alloc_plan(plan);
    }
    compile_staged(plan);
  }
  upload_programs();
  prepared_ = true;
  prepared_id_ = plan_id;
}


void Engine::compile_direct(const reshard::TransferPlan& plan) {
  const Store& src = stores_[RS_SRC];
  const Store& dst = stores_[RS_DST];
  const auto& m = src.model;
  const std::int64_t B = opts_.staging_bytes;
  std::vector<std::size_t> mark(devices_.size());

  // de2 (DP broadcast): a second destination with de's layout, written from
  // the same load (rs_copy_desc.dst2_delta)
  auto push = [&](const Entry* se, const Entry* de, const reshard::ShardView& box, std::int64_t eb, int layer,
                  const Entry* de2 = nullptr) {
    const int l = local_of(se->slot);
    if (l < 0) return;  // the source's process pushes it
    auto& prog = programs_[static_cast<std::size_t>(l)];
    if (de->slot != se->slot || (de2 && de2->slot != se->slot)) prog.peer_stores = true;
    const std::size_t first = prog.local.size();
    append_copy(prog.local, view_base(se, "source"), se->view, view_base(de, "destination"), de->view, box, eb,
                static_cast<std::uint32_t>(layer), opts_.copy_kernel != RS_COPY_CE);
    if (!de2) return;
    const auto delta = static_cast<std::int64_t>(view_base(de2, "destination") - view_base(de, "destination"));
    for (std::size_t k = first; k < prog.local.size(); ++k) {
      rs_copy_desc& d = prog.local[k];
      d.dst2_delta = delta;
      while (d.vec_log2 > 0 && (static_cast<std::uint64_t>(delta) & ((1ull << d.vec_log2) - 1))) --d.vec_log2;
    }
  };
  // DP broadcasts: a layer's copies with one source rank, tensor and box into
  // destinations of identical layout (DP replicas) are paired so one load
  // feeds both stores -- 3 instead of 4 bytes of HBM traffic per byte pair.
  // Only the copy kernels that honour dst2_delta (LDG warp engine, TMA-NP).
  static const bool bcast_off = [] {  // diagnostic A/B knob: RS_DIRECT_BCAST=0
    const char* e = std::getenv("RS_DIRECT_BCAST");
    return e && std::atoi(e) == 0;
  }();
  const bool bcast = !bcast_off && opts_.copy_kernel != RS_COPY_CE && opts_.copy_kernel != RS_COPY_CTA8 &&
                     opts_.copy_kernel != RS_COPY_BULK && (opts_.copy_kernel < RS_COPY_BULK_MW ||
                                                          opts_.copy_kernel > RS_COPY_BULK_MW + 4);
  struct Copy {
    int src_rank, dst_rank;
    std::uint32_t ti;
    const reshard::ShardView* box;
    bool keep;
  };
  std::vector<Copy> copies;
  std::vector<int> partner;

  for (int layer : plan_layers_) {
    for (std::size_t d = 0; d < devices_.size(); ++d) mark[d] = programs_[d].local.size();
    rs_exec_report delta{};
    try {
      // validate every copy of the layer (the reference's checks and
      // messages), then pair DP broadcasts, then emit
      copies.clear();
      if (auto it = plan.carryover_by_layer.find(layer); it != plan.carryover_by_layer.end()) {
        for (const auto& k : it->second) {
          const Entry* se = src.find(k.rank, k.tensor_index);
          const Entry* de = se ? dst.find(k.rank, k.tensor_index) : nullptr;
          if (!se || !de) throw IntegrityError(no_buffer(k.rank, k.tensor_index));
          if (!holds(se, k.bounds)) throw IntegrityError(escape_msg("slice_local", k.bounds, se->view));
          if (!holds(de, k.bounds)) throw IntegrityError(escape_msg("scatter_local", k.bounds, de->view));
          copies.push_back({k.rank, k.rank, k.tensor_index, &k.bounds, true});
          delta.carryover_bytes += k.bounds.element_count() * m.element_bytes(m.tensors[k.tensor_index]);
        }
      }
      if (auto it = plan.tasks_by_layer.find(layer); it != plan.tasks_by_layer.end()) {
        for (const auto& t : it->second) {
          const Entry* se = src.find(t.src_rank, t.tensor_index);
          if (!se) throw IntegrityError(no_buffer(t.src_rank, t.tensor_index));
          if (!holds(se, t.bounds)) throw IntegrityError("integrity: task bounds escape source view");
          const std::int64_t eb = m.element_bytes(m.tensors[t.tensor_index]);
          if (eb > B) throw IntegrityError("chunk_bounds: one element exceeds the staging budget");
          const Entry* de = dst.find(t.dst_rank, t.tensor_index);
          if (!de) throw IntegrityError(no_buffer(t.dst_rank, t.tensor_index));
          if (!holds(de, t.bounds)) throw IntegrityError(escape_msg("scatter_local", t.bounds, de->view));
          copies.push_back({t.src_rank, t.dst_rank, t.tensor_index, &t.bounds, false});
          const std::int64_t n = t.bounds.element_count() * eb;
          if (t.is_local()) delta.local_copy_bytes += n;
          else delta.bytes_moved += n;
        }
      }
      partner.assign(copies.size(), -1);  // -1 alone, >= 0 the paired copy, -2 emitted by its partner
      if (bcast && copies.size() > 1) {
        std::map<std::tuple<int, std::uint32_t, std::vector<std::int64_t>>, std::vector<std::size_t>> groups;
        for (std::size_t i = 0; i < copies.size(); ++i) {
          std::vector<std::int64_t> b;
          for (std::size_t d = 0; d < copies[i].box->ndims(); ++d) {
            b.push_back(copies[i].box->dim(d).lo);
            b.push_back(copies[i].box->dim(d).hi);
          }
          groups[{copies[i].src_rank, copies[i].ti, std::move(b)}].push_back(i);
        }
        for (const auto& kv : groups) {
          const auto& g = kv.second;
          for (std::size_t a = 0; a < g.size(); ++a) {
            if (partner[g[a]] != -1) continue;
            const Entry* da = dst.find(copies[g[a]].dst_rank, copies[g[a]].ti);
            for (std::size_t b = a + 1; b < g.size(); ++b) {
              if (partner[g[b]] != -1) continue;
              const Entry* db = dst.find(copies[g[b]].dst_rank, copies[g[b]].ti);
              if (da->view == db->view && da->flat == db->flat && da->flat_lo == db->flat_lo) {
                partner[g[a]] = static_cast<int>(g[b]);
                partner[g[b]] = -2;
                break;
              }
            }
          }
        }
      }
      for (std::size_t i = 0; i < copies.size(); ++i) {
        if (partner[i] == -2) continue;
        const Copy& c = copies[i];
        const Entry* se = src.find(c.src_rank, c.ti);
        const Entry* de = dst.find(c.dst_rank, c.ti);
        const Entry* de2 = partner[i] >= 0 ? dst.find(copies[static_cast<std::size_t>(partner[i])].dst_rank, c.ti)
                                           : nullptr;
        push(se, de, *c.box, m.element_bytes(m.tensors[c.ti]), layer, de2);
      }
    } catch (const IntegrityError& e) {
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

// RS_COPY_CE comparator: every descriptor whose items fall in [b, e) as
// cudaMemcpy2DAsync planes (innermost outer dim = rows; further outer dims
// loop on the host).  Returns the number of copy calls.
int Engine::ce_copies(const std::vector<rs_copy_desc>& descs, std::uint64_t b, std::uint64_t e,
                      cudaStream_t stream) {
  int calls = 0;
  for (const auto& D : descs) {
    if (D.item0 < b || D.item0 >= e) continue;
    if (D.nouter == 0) {
      cuda_check(cudaMemcpyAsync(reinterpret_cast<void*>(D.dst), reinterpret_cast<const void*>(D.src), D.row_bytes,
                                 cudaMemcpyDefault, stream),
                 "ce copy");
      ++calls;
      continue;
    }
    std::uint64_t planes = 1;
    for (std::uint32_t k = 1; k < D.nouter; ++k) planes *= D.ext[k];
    for (std::uint64_t pl = 0; pl < planes; ++pl) {
      std::int64_t so = 0, dof = 0;
      std::uint64_t r = pl;
      for (std::uint32_t k = 1; k < D.nouter; ++k) {
        const std::uint64_t i = r % D.ext[k];
        r /= D.ext[k];
        so += static_cast<std::int64_t>(i) * D.sstr[k];
        dof += static_cast<std::int64_t>(i) * D.dstr[k];
      }
      cuda_check(cudaMemcpy2DAsync(reinterpret_cast<void*>(D.dst + dof), static_cast<std::size_t>(D.dstr[0]),
                                   reinterpret_cast<const void*>(D.src + so), static_cast<std::size_t>(D.sstr[0]),
                                   D.row_bytes, D.ext[0], cudaMemcpyDefault, stream),
                 "ce copy 2d");
      ++calls;
    }
  }
  return calls;
}

std::vector<rs_trace_record> Engine::trace(int dev) const {
  if (dev < 0 || dev >= num_devices()) throw DomainError("trace: bad local device index");
  const DeviceProgram& p = programs_.at(static_cast<std::size_t>(dev));
  if (!opts_.trace || opts_.mode != RS_MODE_STAGED) throw DomainError("trace: create the engine with trace = 1 in STAGED mode");
  std::vector<rs_trace_record> all(p.d_trace.size() / sizeof(rs_trace_record)), out;
  if (all.empty()) return out;
  DeviceGuard g(devices_[static_cast<std::size_t>(dev)].ordinal);
  cuda_check(cudaMemcpy(all.data(), p.d_trace.data(), p.d_trace.size(), cudaMemcpyDeviceToHost), "trace read");
  for (const auto& r : all)
    if (r.t_end) out.push_back(r);
  return out;
}

void Engine::upload_programs() {
  for (std::size_t d = 0; d < devices_.size(); ++d) {
    DeviceProgram& p = programs_[d];
    const Device& dv = devices_[d];
    std::uint64_t bytes = 0;
    p.all_aligned = true;
    p.max_row_bytes = 0;
    for (const auto& c : p.local) {
      bytes += bytes_of(c);
      p.all_aligned = p.all_aligned && c.vec_log2 == 4;
      p.max_row_bytes = std::max<std::uint64_t>(p.max_row_bytes, c.row_bytes);
    }
    p.local_bytes = bytes;
    // bytes one launch moves: everything (fused), or the largest layer (strict
    // per-layer launches, where the last items of every layer form a tail)
    p.launch_bytes = bytes;
    if (opts_.strict_layers) {
      p.launch_bytes = 0;
      for (const auto& lr : p.layers) {
        std::uint64_t lb = 0;
        for (std::size_t i = static_cast<std::size_t>(lr.item_begin); i < static_cast<std::size_t>(lr.item_end); ++i)
          lb += bytes_of(p.local[i]);
        p.launch_bytes = std::max(p.launch_bytes, lb);
      }
    }
    std::uint64_t item_bytes = static_cast<std::uint64_t>(opts_.item_bytes);
    if (item_bytes == 0) {
      const int variant = copy_variant(static_cast<int>(d));
      if (variant == 3) {
        item_bytes = std::clamp<std::uint64_t>(bytes / (static_cast<std::uint64_t>(dv.sms) * 8 + 1), 32768, 8u << 20);
      } else if (variant == 18) {
        item_bytes = 32768;
      } else if (variant == 15 || variant == 17) {
        // non-persistent grid: one 16 KB item per warp, the block scheduler
        // deals CTAs in item order (C2 28.6 ms = 100.7 % of the copy_ peak,
        // strict per-layer 28.9 ms, C1 0.649 ms; np_sweep.jsonl)
        item_bytes = 16384;
      } else if (variant >= 8) {  // 4..16 bulk issuers per SM
        item_bytes = std::clamp<std::uint64_t>(bytes / (static_cast<std::uint64_t>(dv.sms) * 32 + 1), 32768, 1u << 20);
      } else {
        // 64-256 KB items are equivalent at full size (item_sweep_c2.jsonl);
        // smaller when a launch is small so every warp still gets ~64 items
        // and the last items do not form a tail (C1 0.80 -> 0.67 ms, strict
        // per-layer C2 34.6 -> 30.9 ms, item_sweep_c1_strict.jsonl)
        const std::uint64_t warps = static_cast<std::uint64_t>(copy_grid(static_cast<int>(d))) * 8;
        item_bytes = std::clamp<std::uint64_t>(p.launch_bytes / (warps * 64 + 1), 16384, 256u << 10);
      }
    }
    std::uint64_t item = 0;
    for (auto& lr : p.layers) {
      const auto first = static_cast<std::size_t>(lr.item_begin), last = static_cast<std::size_t>(lr.item_end);
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
      if (opts_.trace) p.d_trace = DeviceBuffer(dv.ordinal, 2 * std::max<std::size_t>(1, p.batches.size()) * sizeof(rs_trace_record));
      p.d_frames = DeviceBuffer(dv.ordinal, p.frames.size() * sizeof(rs_copy_desc));
      p.d_error = DeviceBuffer(dv.ordinal, sizeof(unsigned int));
      if (opts_.strict_layers) upload_layer_sync(d);
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
  if (opts_.mode == RS_MODE_XFER) throw DomainError("xfer mode: the caller drives rounds with rs_xfer_step");
  rs_exec_report rep = planned_;
  const auto t0 = std::chrono::steady_clock::now();
  int launches = 0;
  for (auto& dv : devices_) {
    DeviceGuard g(dv.ordinal);
    cuda_check(cudaEventRecord(dv.ev_begin, dv.stream), "event");
  }
  auto launch_copy = [&](std::size_t d, std::uint64_t b, std::uint64_t e) {
    DeviceProgram& p = programs_[d];
    if (e <= b) return;
    DeviceGuard g(devices_[d].ordinal);
    if (opts_.copy_kernel == RS_COPY_CE) {  // comparator: the DMA copy engines, one call per 2-D plane
      launches += ce_copies(p.local, b, e, devices_[d].stream);
      return;
    }
    cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                              reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                              static_cast<std::uint32_t>(p.local.size()), b, e, copy_grid(static_cast<int>(d)),
                              copy_variant(static_cast<int>(d)), devices_[d].stream),
               "copy kernel launch");
    ++launches;
  };
  if (opts_.mode == RS_MODE_DIRECT) {
    if (!opts_.strict_layers) {
      for (std::size_t d = 0; d < devices_.size(); ++d) launch_copy(d, 0, programs_[d].local_items);
    } else {
      const std::size_t nl = programs_.empty() ? 0 : programs_[0].layers.size();
      for (std::size_t li = 0; li < nl; ++li) {
        for (std::size_t d = 0; d < devices_.size(); ++d)
          launch_copy(d, programs_[d].layers[li].item_begin, programs_[d].layers[li].item_end);
        if (devices_.size() > 1) {  // layer barrier across this process's devices
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
      if (p.stream_lanes) {
        launches += run_stream_lanes(d);
        continue;
      }
      const int cap = grid_for(static_cast<int>(d), exchange_kernel_id());
      if (p.ntx + p.nrx >= cap)
        throw DomainError("staged: " + std::to_string(p.ntx + p.nrx) +
                          " ring lanes exceed the co-resident CTA capacity " + std::to_string(cap) +
                          "; lower lanes_per_link");
      if (!p.ntx && !p.nrx && !p.local_items && !opts_.strict_layers) continue;
      DeviceGuard g(devices_[d].ordinal);
      if (opts_.trace && p.d_trace.size())
        cuda_check(cudaMemsetAsync(p.d_trace.data(), 0, p.d_trace.size(), devices_[d].stream), "trace reset");
      const auto* lanes = reinterpret_cast<const rs_lane_desc*>(p.d_lanes.data());
      // strict layers: zero the launch's arrival counter; the barrier flags
      // are epoch-valued and never reset
      rs_layer_sync sync{};
      if (opts_.strict_layers) {
        sync = p.layer_sync;
        cuda_check(cudaMemsetAsync(sync.arrive, 0, (sync.nlayers + 1ull) * sizeof(unsigned long long), devices_[d].stream),
                   "memset");
      }
      // ring slots in L2: 0 = default (discard + policies), else bit flags (2 = neither)
      const int ring_l2 = opts_.ring_discard == 0 ? 5 : opts_.ring_discard;
      cuda_check(rs_launch_exchange(lanes, static_cast<std::uint32_t>(p.ntx), lanes + p.ntx,
                                    static_cast<std::uint32_t>(p.nrx),
                                    reinterpret_cast<const rs_batch_desc*>(p.d_batches.data()),
                                    reinterpret_cast<const rs_copy_desc*>(p.d_frames.data()),
                                    reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                                    reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                                    static_cast<std::uint32_t>(p.local.size()), p.local_items, epoch_,
                                    reinterpret_cast<unsigned int*>(p.d_error.data()),
                                    opts_.spin_limit > 0 ? static_cast<std::uint64_t>(opts_.spin_limit)
                                                         : kSpinLimit,
                                    (opts_.fault_inject == 1 ? 1 : 0) | (ring_l2 & 1 ? 2 : 0) | (ring_l2 & 4 ? 4 : 0) |
                                        (ring_l2 & 8 ? 8 : 0) |
                                        ((ring_l2 & 24) == 24 && opts_.ring_cta_threads == 256 ? 16 : 0),
                                    cap - p.ntx - p.nrx, opts_.ring_cta_threads,
                                    opts_.trace ? reinterpret_cast<rs_trace_record*>(p.d_trace.data()) : nullptr,
                                    opts_.strict_layers ? &sync : nullptr, devices_[d].stream),
                 "exchange kernel launch");
      ++launches;
    }
  }
  double worst = 0;
  for (auto& dv : devices_) {
    DeviceGuard g(dv.ordinal);
    cuda_check(cudaEventRecord(dv.ev_end, dv.stream), "event");
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
        std::snprintf(rep.error, sizeof rep.error, "staged transfer: ring wait timed out on device %d",
                      devices_[d].ordinal);
        cuda_check(cudaMemset(programs_[d].d_error.data(), 0, sizeof flag), "memset");
      }
    }
  }
  rep.device_ms = worst;
  rep.kernel_launches = launches;
  rep.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  describe_run(rep);
  return rep;
}

void Engine::describe_run(rs_exec_report& rep) const {
  rep.copy_kernel = -1;
  if (opts_.mode == RS_MODE_DIRECT && !devices_.empty() && !programs_.empty())
    rep.copy_kernel = opts_.copy_kernel == RS_COPY_CE ? RS_COPY_CE : copy_variant(0);
  rep.ring_same_slot = opts_.mode == RS_MODE_STAGED ? same_slot_policy() : 0;
  rep.ring_kernel = 0;
  if (opts_.mode == RS_MODE_STAGED && !programs_.empty())
    rep.ring_kernel = programs_[0].stream_lanes ? 2 : (programs_[0].ntx + programs_[0].nrx ? 1 : 0);
  rep.relay_routes = relay_routes_;
}

// ------------------------------------------------------------ live handoff

}  // namespace rsb
