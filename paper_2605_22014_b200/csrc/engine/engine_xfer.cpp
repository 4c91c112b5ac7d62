// RS_MODE_XFER: the host-driven point-to-point comparator.
//
// The paper's executor moves every chunk with NCCL isend/irecv between Megatron
// processes (Algorithm 1).  This mode keeps
// that transport but runs our kernels around it: every cross-GPU link
// (src rank -> dst rank on different slots) gets one send buffer on the
// sender and one receive buffer on the receiver, each B / (inbound links of
// the destination rank) bytes -- the staging budget, as in STAGED.  Frames are
// cut with chunk_bounds and packed into per-link batches exactly like the ring
// path; batch r of every link forms round r.  The caller (Python, NCCL) moves
// round r's bytes between rs_xfer_step(pack) and rs_xfer_step(unpack).
// Links are ordered by (src rank, dst rank) on every process, so matching
// send/recv pairs are posted in the same order on both sides.
#include <algorithm>
#include <map>
#include <set>

#include "compile.hpp"
#include "engine.hpp"
#include "engine_internal.hpp"
#include "kernels.h"

namespace rsb {

namespace {

struct Guard {
  int prev = 0;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~Guard() { cudaSetDevice(prev); }
};

std::uint64_t addr_of(const char* p) { return reinterpret_cast<std::uint64_t>(p); }

std::string missing(int rank, std::uint32_t ti) {
  return "shard store: no buffer for rank " + std::to_string(rank) + " tensor " + std::to_string(ti);
}

std::string escapes(const char* who, const reshard::ShardView& b, const reshard::ShardView& owner) {
  return std::string(who) + ": bounds " + b.to_string() + " escape owner view " + owner.to_string();
}

}  // namespace

void Engine::compile_xfer(const reshard::TransferPlan& plan) {
  if (devices_.size() != 1) throw DomainError("xfer mode drives exactly one local device per process");
  const Store& src = stores_[RS_SRC];
  const Store& dst = stores_[RS_DST];
  const auto& m = src.model;
  const std::int64_t B = opts_.staging_bytes;
  const int me = devices_[0].slot;

  struct Frame {
    const Entry* se;
    const Entry* de;
    reshard::ShardView region;
    std::int64_t eb;
    std::uint64_t off;
  };
  struct Link {
    int src_rank, dst_rank, sslot, dslot;
    std::uint64_t slot_bytes = 0;
    std::vector<std::vector<Frame>> batches;
    std::uint64_t fill = 0;
  };
  // cross-GPU links, counted globally (deterministic on every process).  A
  // carryover or local task crosses GPUs too when its rank id is placed on
  // different slots in the two configurations.
  std::map<int, std::set<int>> inbound;
  for (const auto& kv : plan.tasks_by_layer)
    for (const auto& t : kv.second) {
      const Entry* se = src.find(t.src_rank, t.tensor_index);
      const Entry* de = dst.find(t.dst_rank, t.tensor_index);
      if (se && de && se->slot != de->slot) inbound[t.dst_rank].insert(t.src_rank);
    }
  for (const auto& kv : plan.carryover_by_layer)
    for (const auto& k : kv.second) {
      const Entry* se = src.find(k.rank, k.tensor_index);
      const Entry* de = dst.find(k.rank, k.tensor_index);
      if (se && de && se->slot != de->slot) inbound[k.rank].insert(k.rank);
    }
  std::map<std::pair<int, int>, Link> links;

  DeviceProgram& p = programs_[0];
  for (int layer : plan_layers_) {
    const std::size_t mark = p.local.size();
    auto link_marks = std::map<std::pair<int, int>, std::pair<std::size_t, std::uint64_t>>{};
    for (auto& [k, l] : links) link_marks[k] = {l.batches.size(), l.fill};
    std::map<std::pair<int, int>, std::size_t> last_batch_size;
    for (auto& [k, l] : links) last_batch_size[k] = l.batches.empty() ? 0 : l.batches.back().size();
    rs_exec_report delta{};
    // Same GPU: one local copy.  Different GPUs: chunks on link (src, dst).
    auto route = [&](const Entry* se, const Entry* de, const reshard::ShardView& box, std::int64_t eb, int src_rank,
                     int dst_rank) {
      if (se->slot == de->slot) {
        if (se->slot != me) return;
        if (!se->ptr || !de->ptr) throw DomainError("xfer: local shard without device memory");
        append_copy(p.local, addr_of(se->ptr) - static_cast<std::uint64_t>(se->flat_off), se->view,
                    addr_of(de->ptr) - static_cast<std::uint64_t>(de->flat_off), de->view, box, eb,
                    static_cast<std::uint32_t>(layer));
        return;
      }
      const auto key = std::make_pair(src_rank, dst_rank);
      Link& l = links[key];
      if (l.slot_bytes == 0) {
        l.src_rank = src_rank;
        l.dst_rank = dst_rank;
        l.sslot = se->slot;
        l.dslot = de->slot;
        std::uint64_t sb = static_cast<std::uint64_t>(B) / inbound[dst_rank].size();
        l.slot_bytes = sb >= 4096 ? sb / 256 * 256 : sb / 16 * 16;
      }
      if (static_cast<std::uint64_t>(eb) > l.slot_bytes)
        throw IntegrityError("staging: link buffer of " + std::to_string(l.slot_bytes) +
                             " bytes cannot hold one element");
      for (const auto& c : reshard::chunk_bounds(box, static_cast<std::int64_t>(l.slot_bytes), eb)) {
        const std::uint64_t nb = static_cast<std::uint64_t>(c.element_count() * eb);
        std::uint64_t off = (l.fill + 15) / 16 * 16;
        if (l.batches.empty() || off + nb > l.slot_bytes) {
          l.batches.emplace_back();
          off = 0;
        }
        l.batches.back().push_back({se, de, c, eb, off});
        l.fill = off + nb;
      }
    };
    try {
      if (auto it = plan.carryover_by_layer.find(layer); it != plan.carryover_by_layer.end())
        for (const auto& k : it->second) {
          const Entry* se = src.find(k.rank, k.tensor_index);
          const Entry* de = se ? dst.find(k.rank, k.tensor_index) : nullptr;
          if (!se || !de) throw IntegrityError(missing(k.rank, k.tensor_index));
          if (!detail::holds(se, k.bounds)) throw IntegrityError(escapes("slice_local", k.bounds, se->view));
          if (!detail::holds(de, k.bounds)) throw IntegrityError(escapes("scatter_local", k.bounds, de->view));
          const std::int64_t eb = m.element_bytes(m.tensors[k.tensor_index]);
          route(se, de, k.bounds, eb, k.rank, k.rank);
          delta.carryover_bytes += k.bounds.element_count() * eb;
        }
      if (auto it = plan.tasks_by_layer.find(layer); it != plan.tasks_by_layer.end())
        for (const auto& t : it->second) {
          const Entry* se = src.find(t.src_rank, t.tensor_index);
          if (!se) throw IntegrityError(missing(t.src_rank, t.tensor_index));
          if (!detail::holds(se, t.bounds)) throw IntegrityError("integrity: task bounds escape source view");
          const std::int64_t eb = m.element_bytes(m.tensors[t.tensor_index]);
          if (eb > B) throw IntegrityError("chunk_bounds: one element exceeds the staging budget");
          const Entry* de = dst.find(t.dst_rank, t.tensor_index);
          if (!de) throw IntegrityError(missing(t.dst_rank, t.tensor_index));
          if (!detail::holds(de, t.bounds)) throw IntegrityError(escapes("scatter_local", t.bounds, de->view));
          const std::int64_t n = t.bounds.element_count() * eb;
          if (t.is_local()) delta.local_copy_bytes += n;
          else delta.bytes_moved += n;
          route(se, de, t.bounds, eb, t.src_rank, t.dst_rank);
        }
    } catch (const IntegrityError& e) {
      p.local.resize(mark);
      for (auto it = links.begin(); it != links.end();) {
        auto m2 = link_marks.find(it->first);
        if (m2 == link_marks.end()) {
          it = links.erase(it);
          continue;
        }
        it->second.batches.resize(m2->second.first);
        if (!it->second.batches.empty()) it->second.batches.back().resize(last_batch_size[it->first]);
        it->second.fill = m2->second.second;
        ++it;
      }
      planned_.ok = 0;
      planned_.failed_layer = layer;
      std::snprintf(planned_.error, sizeof planned_.error, "%s", e.what());
      break;
    }
    planned_.carryover_bytes += delta.carryover_bytes;
    planned_.local_copy_bytes += delta.local_copy_bytes;
    planned_.bytes_moved += delta.bytes_moved;
    planned_.layers_processed++;
    p.layers.push_back({layer, mark, p.local.size()});
  }
  if (planned_.failed_layer < 0) planned_.ok = 1;

  // rounds, buffers (this process's links only), peak staging per dst rank
  xfer_rounds_ = 0;
  std::map<int, std::int64_t> rx_per_dst;
  std::uint64_t need = 0;
  std::vector<std::pair<std::pair<int, int>, int>> mine;  // (link key, dir)
  for (const auto& [key, l] : links) {
    xfer_rounds_ = std::max<int>(xfer_rounds_, static_cast<int>(l.batches.size()));
    rx_per_dst[l.dst_rank] += static_cast<std::int64_t>(l.slot_bytes);
    if (l.sslot == me) mine.push_back({key, 0});
    if (l.dslot == me) mine.push_back({key, 1});
  }
  for (const auto& kv : rx_per_dst) planned_.peak_staging_bytes = std::max(planned_.peak_staging_bytes, kv.second);
  for (const auto& [key, dir] : mine) need += links.at(key).slot_bytes;
  xfer_buffers_ = DeviceBuffer(devices_[0].ordinal, need);
  xfer_tx_.clear();
  xfer_rx_.clear();
  std::uint64_t off = 0;
  for (const auto& [key, dir] : mine) {
    const Link& l = links.at(key);
    XferLink x;
    x.peer_slot = dir ? l.sslot : l.dslot;
    x.src_rank = l.src_rank;
    x.dst_rank = l.dst_rank;
    x.buf = xfer_buffers_.data() + off;
    x.buf_bytes = l.slot_bytes;
    off += l.slot_bytes;
    x.round_bytes.assign(static_cast<std::size_t>(xfer_rounds_), 0);
    for (std::size_t b = 0; b < l.batches.size(); ++b)
      for (const auto& f : l.batches[b])
        x.round_bytes[b] = std::max<std::uint64_t>(x.round_bytes[b], f.off + static_cast<std::uint64_t>(f.region.element_count() * f.eb));
    (dir ? xfer_rx_ : xfer_tx_).push_back(std::move(x));
  }

  // descriptors: per round, pack (tx) then, separately, unpack (rx)
  xfer_descs_.clear();
  xfer_round_items_.assign(static_cast<std::size_t>(xfer_rounds_), XferRound{});
  std::uint64_t item = 0;
  const std::uint64_t item_bytes = 256u << 10;
  for (int pass = 0; pass < 2; ++pass) {
    for (int r = 0; r < xfer_rounds_; ++r) {
      const std::size_t first = xfer_descs_.size();
      std::size_t tx_i = 0, rx_i = 0;
      for (const auto& [key, dir] : mine) {
        const Link& l = links.at(key);
        XferLink& x = dir ? xfer_rx_[rx_i++] : xfer_tx_[tx_i++];
        if (dir != pass || r >= static_cast<int>(l.batches.size())) continue;
        for (const auto& f : l.batches[static_cast<std::size_t>(r)]) {
          const std::uint64_t b = addr_of(x.buf) + f.off;
          if (pass == 0)
            append_copy(xfer_descs_, addr_of(f.se->ptr) - static_cast<std::uint64_t>(f.se->flat_off), f.se->view, b,
                        f.region, f.region, f.eb, static_cast<std::uint32_t>(r));
          else
            append_copy(xfer_descs_, b, f.region, addr_of(f.de->ptr) - static_cast<std::uint64_t>(f.de->flat_off),
                        f.de->view, f.region, f.eb, static_cast<std::uint32_t>(r));
        }
      }
      const std::uint64_t end = assign_items(xfer_descs_, first, item, item_bytes);
      if (pass == 0) {
        xfer_round_items_[static_cast<std::size_t>(r)].pack_begin = item;
        xfer_round_items_[static_cast<std::size_t>(r)].pack_end = end;
      } else {
        xfer_round_items_[static_cast<std::size_t>(r)].unpack_begin = item;
        xfer_round_items_[static_cast<std::size_t>(r)].unpack_end = end;
      }
      item = end;
    }
  }
  std::vector<std::uint64_t> item0(xfer_descs_.size());
  for (std::size_t i = 0; i < xfer_descs_.size(); ++i) item0[i] = xfer_descs_[i].item0;
  const Device& dv = devices_[0];
  d_xfer_descs_ = DeviceBuffer(dv.ordinal, xfer_descs_.size() * sizeof(rs_copy_desc));
  d_xfer_item0_ = DeviceBuffer(dv.ordinal, item0.size() * sizeof(std::uint64_t));
  d_xfer_descs_.upload(xfer_descs_.data(), xfer_descs_.size() * sizeof(rs_copy_desc), dv.stream);
  d_xfer_item0_.upload(item0.data(), item0.size() * sizeof(std::uint64_t), dv.stream);
  cuda_check(cudaStreamSynchronize(dv.stream), "xfer upload");
}

void* Engine::xfer_stream() const {
  if (!prepared_ || opts_.mode != RS_MODE_XFER) throw DomainError("xfer: prepare a plan in RS_MODE_XFER first");
  return devices_[0].stream;
}

void Engine::xfer_step(int what, int round) {
  if (!prepared_ || opts_.mode != RS_MODE_XFER) throw DomainError("xfer: prepare a plan in RS_MODE_XFER first");
  const bool async = (what & RS_XFER_ASYNC) != 0;  // enqueue only: the caller orders NCCL by events
  what &= ~RS_XFER_ASYNC;
  if (what < 0 || what > 2) throw DomainError("xfer: step must be 0 (local), 1 (pack) or 2 (unpack)");
  const Device& dv = devices_[0];
  Guard g(dv.ordinal);
  if (what == 0) {
    DeviceProgram& p = programs_[0];
    cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                              reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                              static_cast<std::uint32_t>(p.local.size()), 0, p.local_items, copy_grid(0),
                              copy_variant(0), dv.stream),
               "xfer local copies");
  } else {
    if (round < 0 || round >= xfer_rounds_) throw DomainError("xfer: round out of range");
    const XferRound& r = xfer_round_items_[static_cast<std::size_t>(round)];
    // link-buffer frames: 256 KB items, any alignment -> the LDG8 non-persistent kernel
    const std::uint64_t b = what == 1 ? r.pack_begin : r.unpack_begin;
    const std::uint64_t e = what == 1 ? r.pack_end : r.unpack_end;
    cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(d_xfer_descs_.data()),
                              reinterpret_cast<const std::uint64_t*>(d_xfer_item0_.data()),
                              static_cast<std::uint32_t>(xfer_descs_.size()), b, e, copy_grid(0), 15,
                              dv.stream),
               what == 1 ? "xfer pack" : "xfer unpack");
  }
  if (!async) cuda_check(cudaStreamSynchronize(dv.stream), "xfer step");
}

}  // namespace rsb
