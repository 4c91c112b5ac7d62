// Host-store execution (rs_execute_host: H2D / reshard / D2H pipelined by
// layer, optional bounded device window) and the live-handoff Switch step
// (rs_switch: drain -> transfer -> swap, device-timed).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <set>

#include "engine.hpp"
#include "compile.hpp"
#include "engine_internal.hpp"
#include "kernels.h"

namespace rsb {

using namespace detail;

// Drain -> transfer -> swap, the Switch phase of generation.cpp:239-290 with
// each piece executed instead of priced.  The drain is a stream-order wait on
// the caller's iteration-boundary events, so no host thread blocks on the
// training stream and the transfer starts the instant the last one fires.
rs_switch_stats Engine::switch_step(void* const* drain_events, bool swap) {
  if (!prepared_) throw DomainError("switch: prepare the handoff plan first (Prepare phase)");
  rs_switch_stats st{};
  for (std::size_t d = 0; d < devices_.size(); ++d) {
    DeviceGuard g(devices_[d].ordinal);
    cuda_check(cudaEventRecord(devices_[d].ev_call, devices_[d].stream), "event");
    if (drain_events && drain_events[d])
      cuda_check(cudaStreamWaitEvent(devices_[d].stream, static_cast<cudaEvent_t>(drain_events[d]), 0),
                 "drain wait");
  }
  st.exec = run();  // records ev_begin behind the drain waits
  for (auto& dv : devices_) {
    DeviceGuard g(dv.ordinal);
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, dv.ev_call, dv.ev_begin), "elapsed");
    st.drain_ms = std::max(st.drain_ms, static_cast<double>(ms));
  }
  st.transfer_ms = st.exec.device_ms;
  st.transfer_bytes = planned_total_bytes_;
  if (st.exec.ok && swap) {
    const auto t0 = std::chrono::steady_clock::now();
    swap_stores();
    st.swap_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    st.swapped = 1;
  }
  st.pause_ms = st.drain_ms + st.transfer_ms + st.swap_ms;
  return st;
}

void Engine::swap_stores() {
  std::swap(stores_[RS_SRC], stores_[RS_DST]);
  prepared_ = false;  // compiled descriptors point into the old roles
  prepared_id_ = 0;
}

// Host<->device copies of a set of store entries, merged into runs: entries
// that are back to back in the device arena AND in the caller's host buffers
// become one copy (never touching a byte outside the entries), cut into
// <= 256 MiB pieces.  Thousands of per-shard copies cap concurrent H2D + D2H
// at 65 GB/s on a B200 host; merged runs reach 96 GB/s
// (profiles/r1/e2e_probe2.json).
void Engine::copy_runs(const Store& s, const std::vector<std::size_t>& idx, void* const* host, bool to_device) {
  struct Piece {
    char* dev;
    char* hst;
    std::size_t n;
    int local;
  };
  std::vector<Piece> ps;
  ps.reserve(idx.size());
  for (std::size_t k : idx) {
    const Entry& e = s.entries[k];
    if (!e.nbytes) continue;
    ps.push_back({e.ptr, static_cast<char*>(host[k]), static_cast<std::size_t>(e.nbytes), local_of(e.slot)});
  }
  std::sort(ps.begin(), ps.end(), [](const Piece& a, const Piece& b) {
    return a.local != b.local ? a.local < b.local : a.dev < b.dev;
  });
  std::vector<Piece> runs;
  for (const Piece& p : ps) {
    if (!runs.empty()) {
      Piece& r = runs.back();
      if (r.local == p.local && p.dev == r.dev + r.n && p.hst == r.hst + r.n) {
        r.n += p.n;
        continue;
      }
    }
    runs.push_back(p);
  }
  constexpr std::size_t kPiece = 256u << 20;
  for (const Piece& r : runs) {
    const Device& dv = devices_[static_cast<std::size_t>(r.local)];
    DeviceGuard g(dv.ordinal);
    for (std::size_t off = 0; off < r.n; off += kPiece) {
      const std::size_t n = std::min(kPiece, r.n - off);
      if (to_device)
        cuda_check(cudaMemcpyAsync(r.dev + off, r.hst + off, n, cudaMemcpyHostToDevice, dv.h2d), "H2D");
      else
        cuda_check(cudaMemcpyAsync(r.hst + off, r.dev + off, n, cudaMemcpyDeviceToHost, dv.d2h), "D2H");
    }
  }
}

rs_exec_report Engine::run_host(void* const* host_src, void* const* host_dst, int window_layers) {
  (void)window_layers;
  if (!prepared_) throw DomainError("engine: prepare a plan first");
  const auto t0 = std::chrono::steady_clock::now();
  const Store& S = stores_[RS_SRC];
  const Store& D = stores_[RS_DST];
  if (window_layers_ > 0 && opts_.mode != RS_MODE_DIRECT)
    throw DomainError("windowed host-store execution runs in RS_MODE_DIRECT");
  if (opts_.mode != RS_MODE_DIRECT) {
    // staged transfers run as one launch: stage everything in, run, stage out
    for (std::size_t k = 0; k < S.entries.size(); ++k) {
      const Entry& e = S.entries[k];
      const int l = local_of(e.slot);
      if (l < 0) continue;
      const Device& dv = devices_[static_cast<std::size_t>(l)];
      DeviceGuard g(dv.ordinal);
      cuda_check(cudaMemcpyAsync(e.ptr, host_src[k], static_cast<std::size_t>(e.nbytes), cudaMemcpyHostToDevice,
                                 dv.stream), "H2D");
    }
    rs_exec_report rep = run();
    for (std::size_t k = 0; k < D.entries.size(); ++k) {
      const Entry& e = D.entries[k];
      const int l = local_of(e.slot);
      if (l < 0) continue;
      const Device& dv = devices_[static_cast<std::size_t>(l)];
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
  // stream), its destination shards go D2H once every local device finished
  // layer l (d2h stream) -- H2D of l+1, the kernel of l and D2H of l-1
  // overlap and PCIe runs full duplex.  Layers are the plan's
  // (executor.cpp:134-138).
  rs_exec_report rep = planned_;
  const std::size_t nlayers = programs_.empty() ? 0 : programs_[0].layers.size();
  const std::size_t ndev = devices_.size();
  std::map<int, std::size_t> slot_of_layer;
  for (std::size_t li = 0; li < nlayers; ++li) slot_of_layer[programs_[0].layers[li].layer] = li;
  std::vector<std::vector<std::size_t>> src_by_layer(nlayers), dst_by_layer(nlayers);
  for (std::size_t k = 0; k < S.entries.size(); ++k) {
    auto it = slot_of_layer.find(S.model.tensors[S.entries[k].ti].layer);
    if (it != slot_of_layer.end() && local_of(S.entries[k].slot) >= 0) src_by_layer[it->second].push_back(k);
  }
  for (std::size_t k = 0; k < D.entries.size(); ++k) {
    auto it = slot_of_layer.find(D.model.tensors[D.entries[k].ti].layer);
    if (it != slot_of_layer.end() && local_of(D.entries[k].slot) >= 0) dst_by_layer[it->second].push_back(k);
  }
  std::vector<cudaEvent_t> ev_in(nlayers * ndev), ev_done(nlayers * ndev), ev_out(nlayers * ndev);
  for (std::size_t d = 0; d < ndev; ++d) {
    DeviceGuard g(devices_[d].ordinal);
    for (std::size_t li = 0; li < nlayers; ++li) {
      cuda_check(cudaEventCreateWithFlags(&ev_in[li * ndev + d], cudaEventDisableTiming), "event");
      cuda_check(cudaEventCreateWithFlags(&ev_done[li * ndev + d], cudaEventDisableTiming), "event");
      cuda_check(cudaEventCreateWithFlags(&ev_out[li * ndev + d], cudaEventDisableTiming), "event");
    }
    cuda_check(cudaEventRecord(devices_[d].ev_begin, devices_[d].h2d), "event");
  }
  // Windowed stores: layer l reuses the device slot of the last earlier plan
  // layer with the same (l % window); its H2D waits for that layer's D2H.
  std::vector<long> reuse_of(nlayers, -1);
  if (window_layers_ > 0) {
    std::map<int, std::size_t> last_in_slot;
    for (std::size_t li = 0; li < nlayers; ++li) {
      const int w = programs_[0].layers[li].layer % window_layers_;
      if (auto it = last_in_slot.find(w); it != last_in_slot.end()) reuse_of[li] = static_cast<long>(it->second);
      last_in_slot[w] = li;
    }
  }
  // One interleaved enqueue loop (an event must be recorded before a stream
  // waits on it): H2D(l) -> kernel(l) -> D2H(l), three streams per device.
  int launches = 0;
  for (std::size_t li = 0; li < nlayers; ++li) {
    if (reuse_of[li] >= 0)
      for (std::size_t d = 0; d < ndev; ++d) {
        DeviceGuard g(devices_[d].ordinal);
        cuda_check(cudaStreamWaitEvent(devices_[d].h2d, ev_out[static_cast<std::size_t>(reuse_of[li]) * ndev + d], 0),
                   "wait");
      }
    copy_runs(S, src_by_layer[li], host_src, true);
    for (std::size_t d = 0; d < ndev; ++d) {
      DeviceGuard g(devices_[d].ordinal);
      cuda_check(cudaEventRecord(ev_in[li * ndev + d], devices_[d].h2d), "event");
    }
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
                                  copy_grid(static_cast<int>(d)), copy_variant(static_cast<int>(d)),
                                  devices_[d].stream),
                   "copy kernel launch");
        ++launches;
      }
      cuda_check(cudaEventRecord(ev_done[li * ndev + d], devices_[d].stream), "event");
    }
    for (std::size_t d = 0; d < ndev; ++d) {
      DeviceGuard g(devices_[d].ordinal);
      for (std::size_t o = 0; o < ndev; ++o)
        cuda_check(cudaStreamWaitEvent(devices_[d].d2h, ev_done[li * ndev + o], 0), "wait");
    }
    copy_runs(D, dst_by_layer[li], host_dst, false);
    for (std::size_t d = 0; d < ndev; ++d) {
      DeviceGuard g(devices_[d].ordinal);
      cuda_check(cudaEventRecord(ev_out[li * ndev + d], devices_[d].d2h), "event");
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
    cudaEventDestroy(ev_out[i]);
  }
  rep.device_ms = worst;
  rep.kernel_launches = launches;
  rep.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  describe_run(rep);
  return rep;
}

}  // namespace rsb
