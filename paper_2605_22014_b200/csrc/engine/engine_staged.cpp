// STAGED mode: ring geometry, the staging (comm) arena and the compilation
// of a plan into ring lanes / batches / frames for rs_exchange_kernel.
// Bounded staging like the reference's executor (proj/src/executor.cpp:183-206):
// chunk_bounds cuts tasks to the ring slot size, a destination rank's rings
// live in its budget B.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <thread>
#include <limits>
#include <map>
#include <queue>
#include <set>

#include "engine.hpp"
#include "compile.hpp"
#include "engine_internal.hpp"
#include "kernels.h"

namespace rsb {

using namespace detail;

std::size_t Engine::comm_bytes(int slot) const {
  if (comm_layout_valid_) return comm_layout_.slot_bytes.at(static_cast<std::size_t>(slot));
  return make_comm_layout(nullptr).slot_bytes.at(static_cast<std::size_t>(slot));
}

void Engine::comm_alloc() {
  if (!stores_[RS_DST].laid_out) throw DomainError("comm: lay out the dst store first");
  comm_layout_ = make_comm_layout(nullptr);
  comm_layout_valid_ = true;
  alloc_comm_arenas();
}

// Plan-sized rings: each dst rank's region holds exactly its rings (<= B),
// so resident staging is what the rings use, not B per rank.
void Engine::comm_alloc_plan(const reshard::TransferPlan& plan) {
  if (!stores_[RS_DST].laid_out || !stores_[RS_SRC].laid_out) throw DomainError("comm: lay out both stores first");
  const RingGeometry geo = ring_geometry(plan);
  comm_layout_ = make_comm_layout(&geo.ring_bytes_of);
  comm_layout_valid_ = true;
  alloc_comm_arenas();
}

void Engine::alloc_comm_arenas() {
  comm_.clear();
  for (const auto& dv : devices_) {
    const std::size_t n = comm_bytes(dv.slot);
    comm_.emplace_back(dv.ordinal, n);
    DeviceGuard g(dv.ordinal);
    cuda_check(cudaMemset(comm_.back().data(), 0, n), "comm memset");
  }
  prepared_ = false;
}

char* Engine::comm_base(int slot) const {
  const int l = local_of(slot);
  if (l >= 0) return static_cast<std::size_t>(l) < comm_.size() ? comm_[static_cast<std::size_t>(l)].data() : nullptr;
  const auto& imp = comm_imported_[static_cast<std::size_t>(slot)];
  return imp ? imp->data() : nullptr;
}

int Engine::same_slot_policy() const {
  return opts_.ring_same_slot == 0 ? (nslots_ > 1 ? 2 : 1) : opts_.ring_same_slot;
}

bool Engine::ringed(const reshard::TransferTask& t) const {
  if (t.is_local()) return false;
  if (same_slot_policy() == 1) return true;
  const Entry* se = stores_[RS_SRC].find(t.src_rank, t.tensor_index);
  const Entry* de = stores_[RS_DST].find(t.dst_rank, t.tensor_index);
  return !(se && de && se->slot == de->slot);
}

// Ring geometry of a plan (STAGED): lanes per link, slot size and ring bytes
// per destination rank.  Deterministic from the plan and the layouts, so
// every process computes the same rings for every slot.
Engine::RingGeometry Engine::ring_geometry(const reshard::TransferPlan& plan) const {
  const Store& src = stores_[RS_SRC];
  const Store& dst = stores_[RS_DST];
  const std::int64_t B = opts_.staging_bytes;
  const int K = opts_.slots_per_link;
  RingGeometry geo;
  geo.stream = stream_lanes_for(plan);
  std::map<int, int> src_slot, dst_slot;  // rank -> slot
  for (const auto& e : src.entries) src_slot.emplace(e.rank, e.slot);
  for (const auto& e : dst.entries) dst_slot.emplace(e.rank, e.slot);
  auto slot_in = [](const std::map<int, int>& m, int rank) {
    auto it = m.find(rank);
    return it == m.end() ? -1 : it->second;
  };

  // Relay chains for DP broadcasts (reshard::relay_chains): route = distinct
  // (source rank, destination chain); hop 0 of a chain rides the route's
  // lanes, later hops are forwarded by the previous hop's receivers.
  std::map<std::pair<int, std::vector<int>>, int> route_id;
  if (opts_.relay && nslots_ > 1) {
    if (!geo.stream)
      throw DomainError("relay: needs stream lanes (16 B aligned plans, ring_kernel 0 or 2)");
    const auto chains = reshard::relay_chains(
        plan, [&](int r) { return slot_in(src_slot, r); }, [&](int r) { return slot_in(dst_slot, r); });
    for (const auto& ch : chains) {
      const auto& tasks = plan.tasks_by_layer.at(ch.layer);
      std::vector<int> ranks;
      for (std::size_t i : ch.tasks) ranks.push_back(tasks[i].dst_rank);
      const auto key = std::make_pair(tasks[ch.tasks[0]].src_rank, ranks);
      auto it = route_id.find(key);
      if (it == route_id.end()) {
        it = route_id.emplace(key, static_cast<int>(geo.route_chain.size())).first;
        geo.route_chain.push_back(ranks);
      }
      for (std::size_t k = 0; k < ch.tasks.size(); ++k)
        geo.relay_of[{ch.layer, ch.tasks[k]}] = {it->second, static_cast<int>(k)};
    }
  }

  // ring links: bytes, the sender's slot, the receivers' ranks and slots
  struct Link {
    std::uint64_t bytes = 0;
    int tx_slot = 0;
    std::vector<int> rx_ranks;
    int first = -1, last = -1;  // plan-layer index range of its tasks
    std::map<int, std::uint64_t> layer_bytes;  // plan-layer index -> its bytes there
  };
  // plan-layer index of every layer (the order prepare executes them in);
  // from the plan itself: rs_comm_alloc_plan sizes the rings before prepare
  std::map<int, int> layer_index;
  for (const auto& kv : plan.tasks_by_layer) layer_index.emplace(kv.first, 0);
  for (const auto& kv : plan.carryover_by_layer) layer_index.emplace(kv.first, 0);
  {
    int i = 0;
    for (auto& kv : layer_index) kv.second = i++;
  }
  std::map<LaneKey, Link> links;
  for (const auto& [layer, tasks] : plan.tasks_by_layer)
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      const auto& t = tasks[i];
      if (!ringed(t)) continue;
      LaneKey key{t.src_rank, t.dst_rank, -1};
      if (auto it = geo.relay_of.find({layer, i}); it != geo.relay_of.end()) {
        if (it->second.second > 0) continue;  // a forwarded hop: the route's lanes carry it
        key = LaneKey{t.src_rank, t.dst_rank, it->second.first};
      }
      Link& lk = links[key];
      if (lk.rx_ranks.empty()) {
        lk.tx_slot = slot_in(src_slot, t.src_rank);
        lk.rx_ranks = std::get<2>(key) < 0 ? std::vector<int>{t.dst_rank}
                                           : geo.route_chain[static_cast<std::size_t>(std::get<2>(key))];
      }
      lk.bytes += static_cast<std::uint64_t>(t.byte_size);
      const int li = layer_index.count(layer) ? layer_index.at(layer) : 0;
      lk.first = lk.first < 0 ? li : std::min(lk.first, li);
      lk.last = std::max(lk.last, li);
      lk.layer_bytes[li] += static_cast<std::uint64_t>(t.byte_size);
    }
  std::map<int, std::set<LaneKey>> inbound;  // dst rank -> links with a receiver there
  for (const auto& [key, lk] : links)
    for (int r : lk.rx_ranks) inbound[r].insert(key);

  // Lanes per link.  Throughput of a lane is one lane-end CTA's worth of
  // bytes in flight (a 1-warp stream-lane CTA, or an 8-warp classic one), so
  // more lanes is faster (profiles/r1/staged_sweep.jsonl,
  // profiles/r2/stream_lane_share_sweep.jsonl) until the sender + receiver
  // CTAs of the busiest slot stop being co-resident.
  // Automatic choice: lanes proportional to each link's bytes (a link's
  // lanes finish together, so the launch ends when the heaviest link does),
  // scaled so every slot's sender + receiver lanes fit a share of one
  // device's CTA capacity (below), at least one and at most 64 per link (same
  // answer on every process: the plan and the placement are global).  A
  // relay route's lanes have a receiver (forwarder) CTA on every hop.
  auto& lanes_of = geo.lanes_of;
  if (opts_.lanes_per_link > 0) {
    for (const auto& kv : links) lanes_of[kv.first] = opts_.lanes_per_link;
  } else if (!links.empty()) {
    auto touches = [&](const Link& lk, auto&& fn) {  // every CTA-hosting slot of a link, once per CTA
      fn(lk.tx_slot);
      for (int r : lk.rx_ranks) fn(slot_in(dst_slot, r));
    };
    // Share of the co-resident CTAs given to ring lanes; the rest run the
    // local copies (local tasks + carryovers) in the same launch.  Balanced so
    // both finish together: a lane pair (2 CTAs) streams ~10 GB/s of payload,
    // a local-copy CTA ~20 GB/s (profiles/r1/trace_capacity.jsonl), so with
    // r = local / remote bytes the lane CTAs take 1.94 / (2 + r / 2) of 97 %.
    std::uint64_t remote_total = 0, local_total = 0;
    for (const auto& kv : plan.tasks_by_layer)
      for (const auto& t : kv.second) (ringed(t) ? remote_total : local_total) += static_cast<std::uint64_t>(t.byte_size);
    for (const auto& kv : plan.carryover_by_layer)
      for (const auto& k : kv.second) local_total += static_cast<std::uint64_t>(k.byte_size);
    const double r = remote_total ? static_cast<double>(local_total) / static_cast<double>(remote_total) : 0.0;
    // stream lanes: the local copies run as their own launch beside the lane
    // kernel, so the lanes may take (almost) every co-resident CTA slot
    // (strict: the local copies run inside the lane launch, in 1-warp CTAs
    // that move ~2/3 of a lane end's bytes each -- leave them a 1.5 r share:
    // full C2 strict 49.0 ms at 1 / (1 + r), 47.4 ms at this share,
    // profiles/r2/strict_scoped/strict_sweep2.jsonl)
    double frac = geo.stream ? (opts_.strict_layers ? 0.98 * std::clamp(1.0 / (1.0 + 1.5 * r), 0.5, 0.95) : 0.98)
                             : std::clamp(1.94 / (2.0 + 0.5 * r), 0.5, 0.97);
    if (const char* env = std::getenv("RS_RING_CAPACITY_FRAC")) frac = std::atof(env);
    const int capacity = static_cast<int>(lane_capacity(0, geo.stream) * frac);
    // per link (few-link plans, e.g. GPT-2 C1 with 4 links, need more than
    // 32; strict stream lanes give one PP stage's few links the whole share)
    int max_lanes = geo.stream && opts_.strict_layers ? 128 : 64;
    if (const char* env = std::getenv("RS_RING_MAX_LANES")) max_lanes = std::atoi(env);
    // The capacity constraint is per slot; under strict layers it is per
    // (layer, slot): the lane kernel runs layer-scoped roles (a lane end's
    // CTA is needed only over its link's layer range, upload_layer_sync), so
    // links that never share a layer -- the PP stages -- each get the whole
    // lane share instead of splitting it.  Fused, every lane is live at once:
    // one "layer" spanning the plan.
    const bool scoped = geo.stream && opts_.strict_layers;
    const std::size_t nl = scoped ? std::max<std::size_t>(layer_index.size(), 1) : 1;
    auto span = [&](const Link& lk, auto&& fn) {  // the layers (rows) a link's lanes are live in
      if (!scoped) return fn(std::size_t{0});
      for (int li = std::max(lk.first, 0); li <= lk.last; ++li) fn(static_cast<std::size_t>(li));
    };
    const std::size_t ns = static_cast<std::size_t>(nslots_);
    // per-row lane capacity.  Fused: the share above.  Strict: each (layer,
    // slot) splits the launch's CTAs between lane ends and in-launch local
    // copies by that layer's bytes (ring bytes per lane end, local bytes
    // weighted by RS_STRICT_LOCAL_WEIGHT), so a layer without local work
    // (C2's second PP stage) gives the lanes everything; the local-copy
    // roles take what the lanes leave (upload_layer_sync)
    std::vector<int> cap_row(nl * ns, capacity);
    if (scoped) {
      // a local byte weighs 1.5 ring bytes per lane end (strict sweep,
      // profiles/r2/strict_scoped/local_sweep.jsonl: best for C2, C4, C5b)
      double w = 1.5;
      if (const char* env = std::getenv("RS_STRICT_LOCAL_WEIGHT")) w = std::atof(env);
      std::vector<double> ring_row(nl * ns, 0.0), local_row(nl * ns, 0.0);
      for (const auto& [key, lk] : links)
        for (const auto& [li, b] : lk.layer_bytes)
          touches(lk, [&](int sl) { ring_row[static_cast<std::size_t>(li) * ns + static_cast<std::size_t>(sl)] += static_cast<double>(b); });
      auto add_local = [&](int layer, int rank, std::int64_t bytes) {
        const int sl = slot_in(src_slot, rank);
        if (sl < 0 || !layer_index.count(layer)) return;
        local_row[static_cast<std::size_t>(layer_index.at(layer)) * ns + static_cast<std::size_t>(sl)] += static_cast<double>(bytes);
      };
      for (const auto& [layer, tasks] : plan.tasks_by_layer)
        for (const auto& t : tasks)
          if (!ringed(t)) add_local(layer, t.src_rank, t.byte_size);
      for (const auto& [layer, keeps] : plan.carryover_by_layer)
        for (const auto& k : keeps) add_local(layer, k.rank, k.byte_size);
      const double total = 0.98 * lane_capacity(0, geo.stream);
      for (std::size_t row = 0; row < nl * ns; ++row)
        cap_row[row] = ring_row[row] > 0
                           ? std::max(1, static_cast<int>(total * ring_row[row] / (ring_row[row] + w * local_row[row])))
                           : std::numeric_limits<int>::max();  // lanes idle here: no constraint from this row
      if (std::getenv("RS_RING_CAPACITY_FRAC")) std::fill(cap_row.begin(), cap_row.end(), capacity);
    }
    std::vector<double> live_bytes(nl * ns, 0.0);
    for (const auto& [key, lk] : links)
      span(lk, [&](std::size_t li) { touches(lk, [&](int sl) { live_bytes[li * ns + static_cast<std::size_t>(sl)] += static_cast<double>(lk.bytes); }); });
    double scale = std::numeric_limits<double>::max();  // lanes per byte: the tightest row decides
    for (std::size_t row = 0; row < nl * ns; ++row)
      if (live_bytes[row] > 0 && cap_row[row] < std::numeric_limits<int>::max())
        scale = std::min(scale, cap_row[row] / live_bytes[row]);
    if (scale == std::numeric_limits<double>::max()) scale = 0.0;
    std::vector<int> live_lanes(nl * ns, 0);
    for (const auto& [key, lk] : links) {
      const int n = std::clamp(static_cast<int>(scale * static_cast<double>(lk.bytes)), 1, max_lanes);
      lanes_of[key] = n;
      span(lk, [&](std::size_t li) { touches(lk, [&](int sl) { live_lanes[li * ns + static_cast<std::size_t>(sl)] += n; }); });
    }
    // the max(1, .) floor can overshoot a slot with many light links: trim
    // the widest links live there
    for (std::size_t row = 0; row < nl * ns; ++row)
      while (live_lanes[row] > cap_row[row]) {
        const std::size_t li = row / ns;
        const int sl = static_cast<int>(row % ns);
        const LaneKey* widest = nullptr;
        int w = 1;
        for (const auto& [key, lk] : links) {
          bool hit = false;
          touches(lk, [&](int x) { hit = hit || x == sl; });
          if (scoped) hit = hit && static_cast<int>(li) >= lk.first && static_cast<int>(li) <= lk.last;
          if (hit && lanes_of[key] > w) {
            w = lanes_of[key];
            widest = &key;
          }
        }
        if (!widest) break;  // every link at one lane: the launch check reports it
        --lanes_of[*widest];
        const Link& wl = links.at(*widest);
        span(wl, [&](std::size_t l2) { touches(wl, [&](int x) { --live_lanes[l2 * ns + static_cast<std::size_t>(x)]; }); });
      }
    // Flooring leaves up to one lane per link unused: hand the spare CTA
    // slots out one lane at a time to the link with the most bytes per lane
    // whose rows all have room, so the per-lane bytes -- and the lanes'
    // finish times -- come out as even as the capacity allows.
    // (ties go to the smaller link key: every process computes the same
    // geometry, and comm_alloc_plan and prepare agree)
    using Cand = std::pair<double, const LaneKey*>;
    auto later = [](const Cand& a, const Cand& b) {
      return a.first != b.first ? a.first < b.first : *b.second < *a.second;
    };
    std::priority_queue<Cand, std::vector<Cand>, decltype(later)> grow(later);
    for (const auto& [key, lk] : links)
      if (lanes_of[key] < max_lanes) grow.push({static_cast<double>(lk.bytes) / lanes_of[key], &key});
    while (!grow.empty()) {
      const LaneKey* kp = grow.top().second;
      grow.pop();
      const Link& lk = links.at(*kp);
      std::map<int, int> per_slot;  // CTAs one more lane adds to each slot (both ends may share one)
      touches(lk, [&](int sl) { ++per_slot[sl]; });
      bool room = true;
      span(lk, [&](std::size_t li) {
        for (const auto& [sl, c] : per_slot) {
          const std::size_t row = li * ns + static_cast<std::size_t>(sl);
          room = room && static_cast<long long>(live_lanes[row]) + c <= cap_row[row];
        }
      });
      if (!room) continue;  // rows only fill up: this link cannot grow again
      const int n = ++lanes_of[*kp];
      span(lk, [&](std::size_t li) { touches(lk, [&](int sl) { ++live_lanes[li * ns + static_cast<std::size_t>(sl)]; }); });
      if (n < max_lanes) grow.push({static_cast<double>(lk.bytes) / n, kp});
    }
  }
  // Ring slot size per dst rank: B split over its inbound lanes, capped at
  // 128 KiB by default -- B is the budget, not the target footprint.  At
  // 64-128 KiB the rings stay (almost) entirely in L2: DRAM traffic of the
  // exchange kernel = the 2x floor (profiles/r1/ring_traffic/).  With
  // GPU-scope handshakes for same-device lanes, 128-256 KiB slots x K = 2
  // keep the rings small enough to stay largely L2-resident (less HBM
  // traffic than the 4x of a DRAM-resident ring) while a batch is still long
  // against its handshake; 32 KiB slots pay the handshake, >= 1 MiB slots
  // spill to DRAM (profiles/r1/ring_sweep_v3.jsonl).  The kernel adds
  // evict-first / evict-last L2 policies and discards drained slots by
  // default (ring_sweep_v4.jsonl: 15.4 -> 13.1 ms on the C5 slice).
  // stream lanes: 64 KiB slots (4 stage-sized items per batch) keep ~450
  // lanes' rings in L2 (profiles/r2/stream_sweep.jsonl: 128 KiB -> 48 ms, 64 KiB -> 38.7 ms on full C2)
  const std::uint64_t slot_default = geo.stream ? kRingSlotStreamDefault : kRingSlotDefault;
  const std::uint64_t slot_cap = opts_.ring_slot_kib < 0    ? ~0ull
                                 : opts_.ring_slot_kib == 0 ? slot_default
                                                            : static_cast<std::uint64_t>(opts_.ring_slot_kib) << 10;
  auto& inbound_lanes = geo.inbound_lanes;
  for (const auto& [key, lk] : links)
    for (int r : lk.rx_ranks) inbound_lanes[r] += static_cast<std::uint64_t>(lanes_of.at(key));
  // largest element a destination rank receives over rings
  std::map<int, std::uint64_t> need_eb;
  for (const auto& [layer, tasks] : plan.tasks_by_layer)
    for (const auto& t : tasks)
      if (ringed(t)) {
        const auto& m = src.model;
        auto& e = need_eb[t.dst_rank];
        e = std::max<std::uint64_t>(e, static_cast<std::uint64_t>(m.element_bytes(m.tensors[t.tensor_index])));
      }
  auto& slot_bytes_of = geo.slot_bytes_of;
  for (const auto& [d, keys] : inbound) {
    // A tiny budget cannot host K slots on every lane into d: fall back to one
    // lane per link, then to K = 1 (strictly alternating pack / unpack), so
    // the ring path accepts every B the reference's executor accepts (a
    // destination needs room for one element per inbound link).
    int k = K;
    const std::uint64_t need = std::max<std::uint64_t>(need_eb[d], 16);
    auto slot_for = [&]() { return static_cast<std::uint64_t>(B) / (inbound_lanes.at(d) * static_cast<std::uint64_t>(k)); };
    const bool relayed = std::any_of(keys.begin(), keys.end(), [](const LaneKey& x) { return std::get<2>(x) >= 0; });
    if (slot_for() < need) {
      if (relayed)  // one lane per link would change the route's lanes on every hop
        throw DomainError("relay: staging budget " + std::to_string(B) + " B is too small for the relay rings into dst rank " +
                          std::to_string(d) + "; disable relay");
      for (const auto& key : keys)
        if (int& n = lanes_of.at(key); n > 1) {
          inbound_lanes[d] -= static_cast<std::uint64_t>(n - 1);
          n = 1;
        }
    }
    if (slot_for() < need) k = 1;
    geo.k_of[d] = k;
    std::uint64_t sb = std::min(slot_for(), slot_cap);
    if (sb >= 4096) sb = sb / kAlign * kAlign;
    else if (sb >= 16) sb = sb / 16 * 16;
    else if (need_eb[d]) sb = sb / need_eb[d] * need_eb[d];
    if (sb < need_eb[d]) {
      // B / inbound links < one element: no ring geometry fits the budget.
      // The reference executor still succeeds (it needs B >= one element,
      // executor.cpp:183-206), so this destination receives its bytes by
      // direct stores into its shards -- zero staging, the budget holds.
      if (relayed)
        throw DomainError("relay: staging budget " + std::to_string(B) + " B cannot hold a relay ring into dst rank " +
                          std::to_string(d) + "; disable relay");
      geo.direct_dst.insert(d);
      for (const auto& key : keys) lanes_of.erase(key);
      inbound_lanes[d] = 0;
      slot_bytes_of[d] = 0;
      geo.ring_bytes_of[d] = 0;
      continue;
    }
    slot_bytes_of[d] = sb;
    geo.ring_bytes_of[d] = slot_bytes_of[d] * inbound_lanes.at(d) * static_cast<std::uint64_t>(k);
  }
  // a route's rings are alike on every hop (the forwarder stores each batch at
  // the same slot offsets): the smallest slot and depth of its destinations
  for (const auto& chain : geo.route_chain) {
    std::uint64_t sb = ~0ull;
    int k = K;
    for (int r : chain) {
      sb = std::min(sb, slot_bytes_of.at(r));
      k = std::min(k, geo.k_of.at(r));
    }
    geo.route_slot_bytes.push_back(sb);
    geo.route_k.push_back(k);
  }

  return geo;
}

// Comm arena layout over every slot: the dst ranks of a slot in ascending
// order, each with `ring_bytes[rank]` (plan-sized) or B bytes, then the flags.
Engine::CommLayout Engine::make_comm_layout(const std::map<int, std::uint64_t>* ring_bytes) const {
  CommLayout L;
  L.regions.resize(static_cast<std::size_t>(nslots_));
  L.slot_bytes.assign(static_cast<std::size_t>(nslots_), kFlagBytes);
  std::map<int, std::set<int>> ranks_on_slot;
  for (const auto& e : stores_[RS_DST].entries) ranks_on_slot[e.slot].insert(e.rank);
  for (const auto& [slot, ranks] : ranks_on_slot) {
    std::size_t off = 0;
    for (int r : ranks) {
      std::size_t b = static_cast<std::size_t>(opts_.staging_bytes);
      if (ring_bytes) {
        auto it = ring_bytes->find(r);
        b = it == ring_bytes->end() ? 0 : align_up(static_cast<std::size_t>(it->second), kAlign);
      }
      L.regions[static_cast<std::size_t>(slot)][r] = {off, b};
      off += b;
    }
    L.slot_bytes[static_cast<std::size_t>(slot)] = off + kFlagBytes;
  }
  return L;
}

void Engine::compile_staged(const reshard::TransferPlan& plan) {
  const Store& src = stores_[RS_SRC];
  const Store& dst = stores_[RS_DST];
  const auto& m = src.model;
  const std::int64_t B = opts_.staging_bytes;
  const int K = opts_.slots_per_link;

  const RingGeometry geo = ring_geometry(plan);
  relay_routes_ = static_cast<int>(geo.route_chain.size());
  const auto& lanes_of = geo.lanes_of;
  const auto& slot_bytes_of = geo.slot_bytes_of;
  const auto& inbound_lanes = geo.inbound_lanes;
  // each destination rank's region in its slot's comm arena (the layout the
  // arena was allocated with: B per rank, or plan-sized, rs_comm_alloc_plan)
  std::map<int, std::size_t> region_of, region_bytes;
  for (std::size_t sl = 0; sl < comm_layout_.regions.size(); ++sl)
    for (const auto& [r, ob] : comm_layout_.regions[sl]) {
      region_of[r] = ob.first;
      region_bytes[r] = ob.second;
    }

  struct Frame {
    const Entry* se;
    const Entry* de;
    reshard::ShardView region;
    std::int64_t eb;
    std::uint64_t off;
    int layer;
  };
  struct LaneBuild {
    int src_rank, dst_rank, sslot, dslot;
    std::uint64_t slot_bytes;
    int k;  // ring depth of this lane (geo.k_of: K, or 1 for a tiny budget)
    std::vector<std::vector<Frame>> batches;
    std::uint64_t fill = 0;
    int route = -1;   // relay route (hop 0 lanes carry it from the source)
    int hop = 0;      // relay hop: > 0 = fed by the previous hop's receiver (no sender CTA)
    int next = -1;    // lane of the next hop (this lane's receiver forwards into it)
  };
  std::vector<LaneBuild> lanes;
  std::map<LaneKey, int> link_first_lane, link_cursor;

  std::vector<std::size_t> mark(devices_.size());
  std::map<int, std::uint32_t> layer_idx;
  for (std::size_t i = 0; i < plan_layers_.size(); ++i) layer_idx[plan_layers_[i]] = static_cast<std::uint32_t>(i);
  for (int layer : plan_layers_) {
    for (std::size_t d = 0; d < devices_.size(); ++d) mark[d] = programs_[d].local.size();
    // strict layers: a batch never spans two layers (the lanes meet a barrier
    // between them), so every lane opens a fresh batch here
    if (opts_.strict_layers)
      for (auto& lb : lanes) lb.fill = lb.slot_bytes + 1;
    std::vector<std::size_t> lane_mark_batches(lanes.size()), lane_mark_frames(lanes.size());
    std::vector<std::uint64_t> lane_mark_fill(lanes.size());
    for (std::size_t i = 0; i < lanes.size(); ++i) {
      lane_mark_batches[i] = lanes[i].batches.size();
      lane_mark_fill[i] = lanes[i].fill;
      lane_mark_frames[i] = lanes[i].batches.empty() ? 0 : lanes[i].batches.back().size();
    }
    const std::size_t lanes_before = lanes.size();
    rs_exec_report delta{};
    auto local_copy = [&](const Entry* se, const Entry* de, const reshard::ShardView& box, std::int64_t eb) {
      const int l = local_of(se->slot);
      if (l < 0) return;
      append_copy(programs_[static_cast<std::size_t>(l)].local, view_base(se, "source"), se->view,
                  view_base(de, "destination"), de->view, box, eb, static_cast<std::uint32_t>(layer));
    };
    try {
      if (auto it = plan.carryover_by_layer.find(layer); it != plan.carryover_by_layer.end()) {
        for (const auto& k : it->second) {
          const Entry* se = src.find(k.rank, k.tensor_index);
          const Entry* de = se ? dst.find(k.rank, k.tensor_index) : nullptr;
          if (!se || !de) throw IntegrityError(no_buffer(k.rank, k.tensor_index));
          if (!holds(se, k.bounds)) throw IntegrityError(escape_msg("slice_local", k.bounds, se->view));
          if (!holds(de, k.bounds)) throw IntegrityError(escape_msg("scatter_local", k.bounds, de->view));
          const std::int64_t eb = m.element_bytes(m.tensors[k.tensor_index]);
          local_copy(se, de, k.bounds, eb);
          delta.carryover_bytes += k.bounds.element_count() * eb;
        }
      }
      if (auto it = plan.tasks_by_layer.find(layer); it != plan.tasks_by_layer.end()) {
        for (std::size_t ti = 0; ti < it->second.size(); ++ti) {
          const auto& t = it->second[ti];
          const Entry* se = src.find(t.src_rank, t.tensor_index);
          if (!se) throw IntegrityError(no_buffer(t.src_rank, t.tensor_index));
          if (!holds(se, t.bounds)) throw IntegrityError("integrity: task bounds escape source view");
          const std::int64_t eb = m.element_bytes(m.tensors[t.tensor_index]);
          if (eb > B) throw IntegrityError("chunk_bounds: one element exceeds the staging budget");
          const Entry* de = dst.find(t.dst_rank, t.tensor_index);
          if (!de) throw IntegrityError(no_buffer(t.dst_rank, t.tensor_index));
          if (!holds(de, t.bounds)) throw IntegrityError(escape_msg("scatter_local", t.bounds, de->view));
          if (t.is_local()) {
            local_copy(se, de, t.bounds, eb);
            delta.local_copy_bytes += t.bounds.element_count() * eb;
            continue;
          }
          if (!ringed(t) || geo.direct_dst.count(t.dst_rank)) {
            // cross-rank, both ranks on one GPU of a multi-slot job, or a
            // destination whose budget cannot host a ring (ring_geometry)
            local_copy(se, de, t.bounds, eb);
            delta.bytes_moved += t.bounds.element_count() * eb;
            continue;
          }
          // relay chains: hop 0 rides its route's lanes, later hops are
          // forwarded from the previous destination's ring (no frames here)
          int route = -1;
          if (auto r = geo.relay_of.find({layer, ti}); r != geo.relay_of.end()) {
            if (r->second.second > 0) {
              delta.bytes_moved += t.bounds.element_count() * eb;
              continue;
            }
            route = r->second.first;
          }
          const std::uint64_t sb = route < 0 ? slot_bytes_of.at(t.dst_rank)
                                             : geo.route_slot_bytes[static_cast<std::size_t>(route)];
          if (static_cast<std::uint64_t>(eb) > sb)
            throw IntegrityError("staging: ring slot of " + std::to_string(sb) + " bytes cannot hold one element (B=" +
                                 std::to_string(B) + " over " + std::to_string(inbound_lanes.at(t.dst_rank)) +
                                 " inbound links)");
          const auto chunks = reshard::chunk_bounds(t.bounds, static_cast<std::int64_t>(sb), eb);
          const LaneKey lk{t.src_rank, t.dst_rank, route};
          const int P = lanes_of.at(lk);
          if (!link_first_lane.count(lk)) {
            link_first_lane[lk] = static_cast<int>(lanes.size());
            const int k = route < 0 ? geo.k_of.at(t.dst_rank) : geo.route_k[static_cast<std::size_t>(route)];
            for (int p = 0; p < P; ++p) {
              lanes.push_back({t.src_rank, t.dst_rank, se->slot, de->slot, sb, k, {}, 0});
              lanes.back().route = route;
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
      if (dynamic_cast<const DomainError*>(&e)) throw;  // mapping errors are not plan integrity
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

  // Relay hops: a route lane's batches continue along the chain.  Hop h is a
  // copy of the route lane with the same batches and frame offsets whose
  // receiver unpacks into chain[h]'s shards; hop h-1's receiver is its sender.
  for (std::size_t i = 0, n0 = lanes.size(); i < n0; ++i) {
    if (lanes[i].route < 0) continue;
    const auto& chain = geo.route_chain[static_cast<std::size_t>(lanes[i].route)];
    std::size_t prev = i;
    for (std::size_t h = 1; h < chain.size(); ++h) {
      LaneBuild hb = lanes[prev];
      hb.src_rank = chain[h - 1];
      hb.dst_rank = chain[h];
      hb.sslot = lanes[prev].dslot;
      hb.hop = static_cast<int>(h);
      hb.next = -1;
      for (auto& batch : hb.batches)
        for (auto& f : batch) {
          f.de = dst.find(chain[h], f.se->ti);
          if (!f.de || !holds(f.de, f.region))  // the plan's own task for this hop was checked above
            throw IntegrityError("relay: dst rank " + std::to_string(chain[h]) + " has no buffer for a forwarded box");
        }
      hb.dslot = -1;
      for (const auto& e : dst.entries)
        if (e.rank == chain[h]) {
          hb.dslot = e.slot;
          break;
        }
      lanes[prev].next = static_cast<int>(lanes.size());
      prev = lanes.size();
      lanes.push_back(std::move(hb));
    }
  }

  // Ring memory inside the comm arenas (deterministic on every process):
  // a destination rank's lanes take consecutive K-slot rings in its B region;
  // ready flags in the destination slot's flag area, credit flags in the
  // source slot's.
  std::map<int, std::uint64_t> ring_used;  // dst rank -> bytes used in its region
  std::vector<std::size_t> flag_used(static_cast<std::size_t>(nslots_), 0);
  const std::size_t flags_per_lane = align_up(sizeof(std::uint64_t) * static_cast<std::size_t>(K), 64);
  struct LaneAddr {
    std::uint64_t ring_off, ready_off, credit_off;
  };
  std::vector<LaneAddr> where(lanes.size());
  for (std::size_t i = 0; i < lanes.size(); ++i) {
    const auto& lb = lanes[i];
    std::uint64_t& used = ring_used[lb.dst_rank];
    auto reg = region_of.find(lb.dst_rank);
    if (reg == region_of.end())
      throw DomainError("staged: comm arena has no ring region for dst rank " + std::to_string(lb.dst_rank) +
                        "; re-run rs_comm_alloc for this dst layout");
    where[i].ring_off = reg->second + used;
    used += lb.slot_bytes * static_cast<std::uint64_t>(lb.k);
    if (used > region_bytes.at(lb.dst_rank))
      throw DomainError("staged: ring region of dst rank " + std::to_string(lb.dst_rank) + " (" +
                        std::to_string(region_bytes.at(lb.dst_rank)) + " bytes) is smaller than this plan's rings; " +
                        "re-run rs_comm_alloc_plan with this plan");
    auto& fr = flag_used[static_cast<std::size_t>(lb.dslot)];
    auto& fc = flag_used[static_cast<std::size_t>(lb.sslot)];
    if (fr + flags_per_lane > kFlagBytes - kSyncFlagBytes || fc + flags_per_lane > kFlagBytes - kSyncFlagBytes)
      throw DomainError("staged: too many ring lanes for the flag area; lower lanes_per_link");
    where[i].ready_off = fr;
    fr += flags_per_lane;
    where[i].credit_off = fc;
    fc += flags_per_lane;
    planned_.peak_staging_bytes = std::max<std::int64_t>(planned_.peak_staging_bytes, static_cast<std::int64_t>(used));
  }
  auto flag_base = [&](int slot) -> char* {
    char* b = comm_base(slot);
    const std::size_t ring_area = comm_bytes(slot) - kFlagBytes;
    return b ? b + ring_area : nullptr;
  };

  // serialise lanes / batches / frames (global tables, uploaded to every local
  // device).  Lane descriptors and batch offsets first (sequential, cheap),
  // then every lane's frames in parallel into lane-local tables, then one
  // concatenation in lane order -- the same tables a sequential pass builds
  // (a full 7B STAGED plan is ~650 k batches, ~1.3 M frames).
  std::vector<rs_lane_desc> all_lanes(lanes.size());
  std::vector<std::uint8_t> tx_local(lanes.size()), rx_local(lanes.size());
  std::uint64_t nbatch_total = 0;
  for (std::size_t i = 0; i < lanes.size(); ++i) {
    const auto& lb = lanes[i];
    tx_local[i] = local_of(lb.sslot) >= 0;
    rx_local[i] = local_of(lb.dslot) >= 0;
    char* ring = comm_base(lb.dslot);
    char* ready = flag_base(lb.dslot);
    char* credit = flag_base(lb.sslot);
    if ((tx_local[i] || rx_local[i]) && (!ring || !ready || !credit))
      throw DomainError("staged: comm arena of slot " + std::to_string(tx_local[i] ? lb.dslot : lb.sslot) +
                        " not mapped in this process (rs_arena_import RS_COMM)");
    if (rx_local[i] && lb.next >= 0 && !comm_base(lanes[static_cast<std::size_t>(lb.next)].dslot))
      throw DomainError("staged: comm arena of slot " + std::to_string(lanes[static_cast<std::size_t>(lb.next)].dslot) +
                        " not mapped in this process (relay forwarding; rs_arena_import RS_COMM)");
    rs_lane_desc& L = all_lanes[i];
    L = rs_lane_desc{};
    const std::uint64_t ring_addr = ring ? addr(ring) + where[i].ring_off : 0;
    L.slot_base = L.slot_base_rx = ring_addr;
    L.slot_bytes = lb.slot_bytes;
    L.ready_flags = L.ready_flags_rx = ready ? addr(ready) + where[i].ready_off : 0;
    L.credit_flags = L.credit_flags_tx = credit ? addr(credit) + where[i].credit_off : 0;
    L.slots = static_cast<std::uint32_t>(lb.k);
    // GPU-scope synchronisation only when both ends are this process's same
    // slot; every cross-slot lane (another GPU, or another process sharing a
    // GPU through IPC) synchronises at system scope
    L.flags = lb.sslot == lb.dslot ? 0u : RS_LANE_PEER;
    L.batch0 = static_cast<std::uint32_t>(nbatch_total);
    L.nbatches = static_cast<std::uint32_t>(lb.batches.size());
    nbatch_total += lb.batches.size();
    if (lb.next >= 0 && rx_local[i]) {  // relay forwarder: the next hop's ring, as mapped here
      const auto j = static_cast<std::size_t>(lb.next);
      L.fwd_slot_base = addr(comm_base(lanes[j].dslot)) + where[j].ring_off;
      L.fwd_ready_flags = addr(flag_base(lanes[j].dslot)) + where[j].ready_off;
      L.fwd_credit_flags = addr(flag_base(lanes[j].sslot)) + where[j].credit_off;
      L.fwd_flags = lanes[j].sslot == lanes[j].dslot ? 0u : RS_LANE_PEER;
    }
  }
  // hop lanes have no sender CTA: their receiver's predecessor forwards
  for (std::size_t i = 0; i < lanes.size(); ++i)
    if (lanes[i].hop > 0) tx_local[i] = 0;
  std::uint64_t item_div = 32;  // work items per slot (RS_FRAME_ITEMS overrides; diagnostic)
  if (const char* env = std::getenv("RS_FRAME_ITEMS")) item_div = std::max(1, std::atoi(env));
  const bool stream = geo.stream;  // items = one 16 KB shared-memory stage of a stream lane
  std::vector<std::vector<rs_copy_desc>> lane_frames(lanes.size());
  std::vector<std::vector<rs_batch_desc>> lane_batches(lanes.size());
  std::vector<std::uint32_t> lane_npack(lanes.size(), 0);
  // A lane's frames are laid out per role: every pack frame in batch order,
  // then every unpack frame in batch order, so a lane end walks one
  // contiguous frame sequence across batch boundaries (the stream lanes
  // prefetch the next descriptor while the current one moves).
  auto build_lane = [&](std::size_t i) {
    const auto& lb = lanes[i];
    const std::uint64_t ring_addr = all_lanes[i].slot_base;
    auto& frames = lane_frames[i];
    auto& batches = lane_batches[i];
    batches.reserve(lb.batches.size());
    std::vector<rs_copy_desc> unpack;
    // work items inside a batch: ~32 per slot so all 8 warps of the lane's
    // CTA share even a small (L2-resident) slot
    const std::uint64_t frame_item =
        stream ? 16384 : std::clamp<std::uint64_t>(lb.slot_bytes / item_div, 2048, 65536);
    for (std::size_t b = 0; b < lb.batches.size(); ++b) {
      const std::uint64_t slot_addr = ring_addr + (b % static_cast<std::size_t>(lb.k)) * lb.slot_bytes;
      rs_batch_desc Bd{};
      Bd.pack0 = static_cast<std::uint32_t>(frames.size());
      if (tx_local[i])
        for (const auto& f : lb.batches[b])
          append_copy(frames, addr(f.se->ptr) - static_cast<std::uint64_t>(f.se->flat_off), f.se->view, slot_addr + f.off,
                      f.region, f.region, f.eb,
                      static_cast<std::uint32_t>(f.layer));
      for (const auto& f : lb.batches[b]) {
        const std::uint64_t n = static_cast<std::uint64_t>(f.region.element_count() * f.eb);
        Bd.bytes += n;
        Bd.extent = std::max(Bd.extent, f.off + n);
      }
      Bd.layer = lb.batches[b].empty() ? 0u : static_cast<std::uint32_t>(lb.batches[b].front().layer);
      Bd.layer_idx = lb.batches[b].empty() ? 0u : layer_idx.at(lb.batches[b].front().layer);
      Bd.npack = static_cast<std::uint32_t>(frames.size()) - Bd.pack0;
      Bd.pack_items = static_cast<std::uint32_t>(assign_items(frames, Bd.pack0, 0, frame_item));
      Bd.unpack0 = static_cast<std::uint32_t>(unpack.size());  // rebased below
      if (rx_local[i])
        for (const auto& f : lb.batches[b])
          append_copy(unpack, slot_addr + f.off, f.region, view_base(f.de, "destination"), f.de->view, f.region,
                      f.eb, static_cast<std::uint32_t>(f.layer));
      Bd.nunpack = static_cast<std::uint32_t>(unpack.size()) - Bd.unpack0;
      Bd.unpack_items = static_cast<std::uint32_t>(assign_items(unpack, Bd.unpack0, 0, frame_item));
      batches.push_back(Bd);
    }
    const auto npack = static_cast<std::uint32_t>(frames.size());
    for (auto& Bd : batches) Bd.unpack0 += npack;
    frames.insert(frames.end(), unpack.begin(), unpack.end());
    lane_npack[i] = npack;
  };
  const unsigned nthreads = std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency()));
  if (nthreads <= 1 || lanes.size() < 8) {
    for (std::size_t i = 0; i < lanes.size(); ++i) build_lane(i);
  } else {
    std::vector<std::exception_ptr> errors(nthreads);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nthreads; ++t)
      pool.emplace_back([&, t] {
        try {
          for (std::size_t i = t; i < lanes.size(); i += nthreads) build_lane(i);
        } catch (...) {
          errors[t] = std::current_exception();
        }
      });
    for (auto& th : pool) th.join();
    for (auto& e : errors)
      if (e) std::rethrow_exception(e);
  }
  std::vector<rs_batch_desc> batches;
  std::vector<rs_copy_desc> frames;
  {
    std::size_t nf = 0;
    for (const auto& v : lane_frames) nf += v.size();
    frames.reserve(nf);
    batches.reserve(nbatch_total);
    for (std::size_t i = 0; i < lanes.size(); ++i) {
      const auto off = static_cast<std::uint32_t>(frames.size());
      all_lanes[i].tx_frame0 = off;
      all_lanes[i].tx_nframes = lane_npack[i];
      all_lanes[i].rx_frame0 = off + lane_npack[i];
      all_lanes[i].rx_nframes = static_cast<std::uint32_t>(lane_frames[i].size()) - lane_npack[i];
      for (auto Bd : lane_batches[i]) {
        Bd.pack0 += off;
        Bd.unpack0 += off;
        batches.push_back(Bd);
      }
      frames.insert(frames.end(), lane_frames[i].begin(), lane_frames[i].end());
      std::vector<rs_copy_desc>().swap(lane_frames[i]);
    }
  }
  for (std::size_t d = 0; d < devices_.size(); ++d) {
    DeviceProgram& p = programs_[d];
    const int slot = devices_[d].slot;
    if (d + 1 == devices_.size()) {
      p.batches = std::move(batches);
      p.frames = std::move(frames);
    } else {
      p.batches = batches;
      p.frames = frames;
    }
    p.lanes.clear();
    for (std::size_t i = 0; i < lanes.size(); ++i)
      if (lanes[i].sslot == slot && lanes[i].hop == 0) p.lanes.push_back(all_lanes[i]);
    p.ntx = static_cast<int>(p.lanes.size());
    for (std::size_t i = 0; i < lanes.size(); ++i)
      if (lanes[i].dslot == slot) p.lanes.push_back(all_lanes[i]);
    p.nrx = static_cast<int>(p.lanes.size()) - p.ntx;
    // stream lanes need every frame this device touches to be bulk-copyable:
    // 16 B aligned runs of <= one 16 KB stage (the slot-side layout and the
    // flag protocol are the same for both lane kernels, so processes may differ)
    // (strict: every slot launches -- its CTAs meet every layer barrier, and
    // its local copies run inside the lane launch)
    p.stream_lanes = stream && (!p.lanes.empty() || opts_.strict_layers);
    auto bulk_ok = [](const rs_copy_desc& f) {
      return f.vec_log2 == 4 && f.row_bytes <= 16384 && f.rows_per_item * f.row_bytes <= 16384;
    };
    // the plan was bulk-copy eligible (stream_lanes_for), so only a
    // caller-bound shard buffer off a 16 B boundary fails here; every process
    // must run the geometry it computed, so this cannot fall back
    const bool frames_ok = std::all_of(p.frames.begin(), p.frames.end(), bulk_ok);
    const bool local_ok = !opts_.strict_layers || std::all_of(p.local.begin(), p.local.end(), [](const rs_copy_desc& f) {
      return f.vec_log2 == 4 && f.row_bytes <= 16384;  // (items are assigned at upload: 16 KB)
    });
    if (p.stream_lanes && !(frames_ok && local_ok))
      throw DomainError("staged: stream lanes need 16 B aligned shard buffers (rs_store_bind); "
                        "use ring_kernel = 1 (classic lanes) for this job");
  }
}

// Stream lanes (TMA bulk copies) run a plan when the options allow them and
// every ringed task is bulk-copyable on both sides: 16 B aligned runs and
// strides with the engine's 256 B-aligned shard arenas and 16 B-aligned slot
// offsets.  Decided from the plan and the layouts alone, so every process of
// a job makes the same choice (the ring geometry depends on it).
bool Engine::stream_lanes_for(const reshard::TransferPlan& plan) const {
  if (opts_.mode != RS_MODE_STAGED || opts_.ring_kernel == 1) return false;
  if (opts_.ring_discard & 8) return false;  // the warp-specialised control-warp design is classic only
  const Store& src = stores_[RS_SRC];
  const Store& dst = stores_[RS_DST];
  const auto& m = src.model;
  std::vector<rs_copy_desc> scratch;
  for (const auto& kv : plan.tasks_by_layer)
    for (const auto& t : kv.second) {
      if (!ringed(t)) continue;
      const Entry* se = src.find(t.src_rank, t.tensor_index);
      const Entry* de = dst.find(t.dst_rank, t.tensor_index);
      if (!se || !de) continue;  // an integrity failure: reported by compile_staged
      const std::int64_t eb = m.element_bytes(m.tensors[t.tensor_index]);
      scratch.clear();
      // (bases 0 - flat_off: a flat-bucket shard's view origin keeps its alignment)
      append_copy(scratch, static_cast<std::uint64_t>(-se->flat_off), se->view, 0, t.bounds, t.bounds, eb, 0);
      append_copy(scratch, 0, t.bounds, static_cast<std::uint64_t>(-de->flat_off), de->view, t.bounds, eb, 0);
      for (const auto& d : scratch)
        if (d.vec_log2 != 4 || d.row_bytes > 16384) return false;
    }
  if (opts_.strict_layers) {
    // strict: the lane launch also runs the local tasks + carryovers through
    // its shared-memory stages, so they must be bulk-copyable too
    auto local_ok = [&](std::uint32_t ti, int src_rank, int dst_rank, const reshard::ShardView& box) {
      const Entry* se = src.find(src_rank, ti);
      const Entry* de = dst.find(dst_rank, ti);
      if (!se || !de) return true;  // an integrity failure: reported by compile_staged
      scratch.clear();
      append_copy(scratch, static_cast<std::uint64_t>(-se->flat_off), se->view,
                  static_cast<std::uint64_t>(-de->flat_off), de->view, box, m.element_bytes(m.tensors[ti]), 0);
      for (const auto& d : scratch)
        if (d.vec_log2 != 4 || d.row_bytes > 16384) return false;
      return true;
    };
    for (const auto& kv : plan.tasks_by_layer)
      for (const auto& t : kv.second)
        if (!ringed(t) && !local_ok(t.tensor_index, t.src_rank, t.dst_rank, t.bounds)) return false;
    for (const auto& kv : plan.carryover_by_layer)
      for (const auto& k : kv.second)
        if (!local_ok(k.tensor_index, k.rank, k.rank, k.bounds)) return false;
  }
  return true;
}

int Engine::lane_capacity(int dev, bool stream) const {
  if (stream)
    return devices_[static_cast<std::size_t>(dev)].sms *
           std::max(1, stream_max_blocks_per_sm(opts_.ring_stages));
  return grid_for(dev, exchange_kernel_id());
}

// Stream lanes: the lane kernel on the device stream (launched first, so its
// CTAs -- which wait on each other -- are all resident), the local copies as
// a TMA / LDG copy launch on the aux stream beside it, joined before ev_end.
int Engine::run_stream_lanes(std::size_t d) {
  DeviceProgram& p = programs_[d];
  Device& dv = devices_[d];
  const int cap = lane_capacity(static_cast<int>(d), true);
  // strict: layer-scoped roles, so only the lane CTAs active in one layer
  // (plus one local-copy CTA) must be co-resident
  const int resident = opts_.strict_layers ? p.strict_max_active : p.ntx + p.nrx;
  if (resident > cap || (opts_.strict_layers && resident >= cap))
    throw DomainError("staged: " + std::to_string(resident) + " stream lanes" +
                      (opts_.strict_layers ? " active in one layer" : "") + " exceed the co-resident CTA capacity " +
                      std::to_string(cap) + (opts_.strict_layers ? " (strict: one CTA must stay for the local copies)" : "") +
                      "; lower lanes_per_link");
  DeviceGuard g(dv.ordinal);
  int launches = 0;
  if (opts_.trace && p.d_trace.size())
    cuda_check(cudaMemsetAsync(p.d_trace.data(), 0, p.d_trace.size(), dv.stream), "trace reset");
  const int ring_l2 = opts_.ring_discard == 0 ? 5 : opts_.ring_discard;
  static const int stream_flags = [] {  // diagnostics: RS_STREAM_FLAGS (64 = register stores), RS_STREAM_PROF
    const char* e = std::getenv("RS_STREAM_FLAGS");
    return e ? std::atoi(e) : 0;
  }();
  static const bool prof_on = std::getenv("RS_STREAM_PROF") != nullptr;
  DeviceBuffer prof;
  if (prof_on && p.ntx + p.nrx) {
    prof = DeviceBuffer(dv.ordinal, 64ull * static_cast<std::size_t>(p.ntx + p.nrx));
    cuda_check(cudaMemsetAsync(prof.data(), 0, prof.size(), dv.stream), "memset");
  }
  const bool strict = opts_.strict_layers != 0;
  rs_layer_sync sync{};
  if (strict) {  // zero the launch's arrival counter; the barrier flags are epoch-valued
    sync = p.layer_sync;
    cuda_check(cudaMemsetAsync(sync.arrive, 0, (sync.nlayers + 1ull) * sizeof(unsigned long long), dv.stream),
               "memset");
  }
  if (p.ntx + p.nrx || strict) {
    const auto* lanes = reinterpret_cast<const rs_lane_desc*>(p.d_lanes.data());
    cuda_check(rs_launch_stream_exchange(lanes, static_cast<std::uint32_t>(p.ntx), lanes + p.ntx,
                                         static_cast<std::uint32_t>(p.nrx),
                                         reinterpret_cast<const rs_batch_desc*>(p.d_batches.data()),
                                         reinterpret_cast<const rs_copy_desc*>(p.d_frames.data()), epoch_,
                                         reinterpret_cast<unsigned int*>(p.d_error.data()),
                                         opts_.spin_limit > 0 ? static_cast<std::uint64_t>(opts_.spin_limit) : kSpinLimit,
                                         (opts_.fault_inject == 1 ? 1 : 0) | (ring_l2 & 1 ? 2 : 0) | stream_flags,
                                         opts_.ring_stages,
                                         opts_.trace ? reinterpret_cast<rs_trace_record*>(p.d_trace.data()) : nullptr,
                                         prof.size() ? reinterpret_cast<unsigned long long*>(prof.data()) : nullptr,
                                         reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                                         reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                                         static_cast<std::uint32_t>(p.local.size()),
                                         strict ? p.strict_local_ctas : cap - p.ntx - p.nrx,
                                         strict ? &sync : nullptr, dv.stream),
               "stream lane kernel launch");
    ++launches;
    if (prof.size()) {  // diagnostic summary on stderr: mean cycles per phase, senders / receivers
      std::vector<unsigned long long> h(prof.size() / 8);
      cuda_check(cudaMemcpyAsync(h.data(), prof.data(), prof.size(), cudaMemcpyDeviceToHost, dv.stream), "prof");
      cuda_check(cudaStreamSynchronize(dv.stream), "prof");
      double acc[2][9] = {};
      int n[2] = {0, 0};
      for (std::size_t i = 0; i < h.size() / 8; ++i) {
        const int role = h[8 * i + 6] ? 0 : 1;
        ++n[role];
        for (int k = 0; k < 8; ++k) acc[role][k] += static_cast<double>(h[8 * i + k]);
        acc[role][1] -= static_cast<double>(h[8 * i + 1]);
        acc[role][1] += static_cast<double>(h[8 * i + 1] & 0xffffffffull);
        acc[role][8] += static_cast<double>(h[8 * i + 1] >> 32);
      }
      for (int role = 0; role < 2; ++role)
        if (n[role])
          std::fprintf(stderr,
                       "[stream prof] %s lanes=%d total=%.0f load_loop=%.0f reuse_wait=%.0f store_issue=%.0f "
                       "publish_wait=%.0f idle=%.0f items=%.0f land_latency_per_item=%.0f (cycles, mean per lane)\n",
                       role ? "rx" : "tx", n[role], acc[role][0] / n[role], acc[role][8] / n[role],
                       acc[role][1] / n[role], acc[role][2] / n[role], acc[role][3] / n[role], acc[role][4] / n[role],
                       acc[role][5] / n[role], acc[role][7] / std::max(1.0, acc[role][5]));
    }
  }
  static const int local_after = [] {  // diagnostic: 1 = local copies after the lanes, same stream
    const char* e = std::getenv("RS_STREAM_LOCAL_AFTER");
    return e ? std::atoi(e) : 0;
  }();
  if (strict) return launches;  // the local copies ran inside the lane launch
  if (p.local_items && local_after) {
    cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                              reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                              static_cast<std::uint32_t>(p.local.size()), 0, p.local_items,
                              copy_grid(static_cast<int>(d)), copy_variant(static_cast<int>(d)), dv.stream),
               "local copy launch");
    return launches + 1;
  }
  if (p.local_items) {
    cuda_check(cudaStreamWaitEvent(dv.aux, dv.ev_begin, 0), "wait");
    cuda_check(rs_launch_copy(reinterpret_cast<const rs_copy_desc*>(p.d_local.data()),
                              reinterpret_cast<const std::uint64_t*>(p.d_item0.data()),
                              static_cast<std::uint32_t>(p.local.size()), 0, p.local_items,
                              copy_grid(static_cast<int>(d)), copy_variant(static_cast<int>(d)), dv.aux),
               "local copy launch");
    ++launches;
    cuda_check(cudaEventRecord(dv.ev_aux, dv.aux), "event");
    cuda_check(cudaStreamWaitEvent(dv.stream, dv.ev_aux, 0), "wait");
  }
  return launches;
}

char* Engine::layer_done_flag(int slot) const {
  char* b = comm_base(slot);
  return b ? b + comm_bytes(slot) - kSyncFlagBytes : nullptr;
}

// STAGED strict layers: the barrier state of one local device -- arrival
// counters (one per layer) and the role ticket, a release flag, the address
// (as mapped in this process) of every slot's layer-done flag, the local-copy
// item end of every plan layer, and for stream lanes the layer-scoped roles:
// each lane end is active from its first batch's layer to its last's; roles
// are dealt by ticket in that order after the local-copy CTAs (active in
// every layer), and barrier l expects the CTAs active in l.  Deadlock-free
// when the lane ends active in any one layer plus the local-copy CTAs fit the
// co-resident capacity: a role starts only after every role of an earlier
// first layer has started, and a role whose last layer is done exits.
void Engine::upload_layer_sync(std::size_t d) {
  DeviceProgram& p = programs_[d];
  const Device& dv = devices_[d];
  const std::size_t nl = p.layers.size();
  const std::size_t ns = nslots_ > 1 ? static_cast<std::size_t>(nslots_) : 0;
  const bool scoped = p.stream_lanes;
  std::vector<std::uint32_t> expect, local_n, roles, local_roles;
  p.strict_max_active = 0;
  p.strict_local_ctas = 0;
  if (scoped) {
    const int nlanes = p.ntx + p.nrx;
    std::vector<int> first(static_cast<std::size_t>(nlanes), -1), last(static_cast<std::size_t>(nlanes), -1);
    std::vector<int> active(nl + 1, 0);
    for (int i = 0; i < nlanes; ++i) {
      const rs_lane_desc& L = p.lanes[static_cast<std::size_t>(i)];
      if (!L.nbatches) continue;  // exits at once: never arrives
      int lo = static_cast<int>(nl), hi = -1;
      for (std::uint32_t b = 0; b < L.nbatches; ++b) {
        const int li = static_cast<int>(p.batches[L.batch0 + b].layer_idx);
        lo = std::min(lo, li);
        hi = std::max(hi, li);
      }
      if (static_cast<int>(p.batches[L.batch0].layer_idx) != lo)
        throw IntegrityError("staged strict: a lane's batches are not in layer order");
      first[static_cast<std::size_t>(i)] = lo;
      last[static_cast<std::size_t>(i)] = hi;
      for (int li = lo; li <= hi; ++li) ++active[static_cast<std::size_t>(li)];
    }
    p.strict_max_active = *std::max_element(active.begin(), active.end());
    const int cap = lane_capacity(static_cast<int>(d), true);
    // Local-copy roles: layer l's local items are shared by n[l] CTAs --
    // every CTA slot its lane ends leave (at least one, so each barrier has
    // an arrival on this GPU).  Local slot j works in the layers with
    // n > j; each maximal run of such layers is one role (a CTA that exits
    // after the run), so exactly n[l] local roles are live in layer l and
    // lanes + local roles never exceed the co-resident capacity.
    std::vector<std::uint32_t> n(nl);
    for (std::size_t li = 0; li < nl; ++li) n[li] = static_cast<std::uint32_t>(std::max(1, cap - active[li]));
    std::vector<std::pair<int, std::uint32_t>> order_all;  // (sort key, role)
    const std::uint32_t m = *std::max_element(n.begin(), n.end());
    for (std::uint32_t jj = 0; jj < m; ++jj)
      for (std::size_t li = 0; li < nl;) {
        if (n[li] <= jj) {
          ++li;
          continue;
        }
        std::size_t l1 = li;
        while (l1 + 1 < nl && n[l1 + 1] > jj) ++l1;
        const auto q = static_cast<std::uint32_t>(local_roles.size() / 2);
        local_roles.push_back(jj);
        local_roles.push_back(static_cast<std::uint32_t>(li) | static_cast<std::uint32_t>(l1) << 16);
        order_all.push_back({2 * static_cast<int>(li), static_cast<std::uint32_t>(nlanes) + q});
        li = l1 + 1;
      }
    p.strict_local_ctas = static_cast<int>(local_roles.size() / 2);
    expect.resize(nl);
    for (std::size_t li = 0; li < nl; ++li) expect[li] = static_cast<std::uint32_t>(active[li]) + n[li];
    local_n = n;
    // local roles and lane ends in first-layer order (local first on ties)
    for (int i = 0; i < nlanes; ++i) {
      const int f = first[static_cast<std::size_t>(i)];
      order_all.push_back({f < 0 ? 1 << 30 : 2 * f + 1, static_cast<std::uint32_t>(i)});
    }
    std::stable_sort(order_all.begin(), order_all.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& [k, role] : order_all) roles.push_back(role);
  }
  const std::size_t n32 = expect.size() + local_n.size() + roles.size() + local_roles.size();
  std::vector<std::uint64_t> words(nl + 2 + ns + nl + (n32 + 1) / 2, 0);
  for (std::size_t s = 0; s < ns; ++s) {
    char* f = layer_done_flag(static_cast<int>(s));
    if (!f)
      throw DomainError("staged strict_layers: comm arena of slot " + std::to_string(s) +
                        " not mapped in this process (rs_arena_import RS_COMM on every process)");
    words[nl + 2 + s] = addr(f);
  }
  for (std::size_t li = 0; li < nl; ++li) words[nl + 2 + ns + li] = p.layers[li].item_end;
  auto* tail = reinterpret_cast<std::uint32_t*>(words.data() + nl + 2 + ns + nl);
  std::copy(expect.begin(), expect.end(), tail);
  std::copy(local_n.begin(), local_n.end(), tail + expect.size());
  std::copy(roles.begin(), roles.end(), tail + expect.size() + local_n.size());
  std::copy(local_roles.begin(), local_roles.end(), tail + expect.size() + local_n.size() + roles.size());
  DeviceGuard g(dv.ordinal);
  p.d_sync = DeviceBuffer(dv.ordinal, words.size() * sizeof(std::uint64_t));
  p.d_sync.upload(words.data(), words.size() * sizeof(std::uint64_t), dv.stream);
  auto* base = reinterpret_cast<std::uint64_t*>(p.d_sync.data());
  p.layer_sync = rs_layer_sync{};
  p.layer_sync.nlayers = static_cast<std::uint32_t>(nl);
  p.layer_sync.nslots = static_cast<std::uint32_t>(ns);
  p.layer_sync.arrive = reinterpret_cast<unsigned long long*>(base);
  p.layer_sync.tickets = reinterpret_cast<unsigned long long*>(base + nl);
  p.layer_sync.release = base + nl + 1;
  p.layer_sync.done_self = ns ? reinterpret_cast<std::uint64_t*>(layer_done_flag(dv.slot)) : nullptr;
  p.layer_sync.done_all = reinterpret_cast<const std::uint64_t* const*>(base + nl + 2);
  p.layer_sync.local_layer_end = base + nl + 2 + ns;
  const auto* tail_dev = reinterpret_cast<const std::uint32_t*>(base + nl + 2 + ns + nl);
  p.layer_sync.expect = scoped ? tail_dev : nullptr;
  p.layer_sync.local_n = scoped ? tail_dev + expect.size() : nullptr;
  p.layer_sync.roles = scoped ? tail_dev + expect.size() + local_n.size() : nullptr;
  p.layer_sync.local_roles = scoped ? tail_dev + expect.size() + local_n.size() + roles.size() : nullptr;
}

}  // namespace rsb
