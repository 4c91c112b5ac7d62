// Relay chains for DP broadcasts (forwarding).
//
// The reference planner sources every region a destination rank did not hold
// itself from the dp-0 owner in C_old (planner.cpp:154-171).  When C_new adds
// DP replicas (BASELINE config 5b, TP2PP2 -> TP2PP2DP2), the same box of the
// same tensor leaves one source GPU once per replica: the source's NVLink
// egress doubles (47.2 GB from one GPU for iota C5b) while the new GPUs' links
// idle.  A relay chain serves the replicas in turn instead:
//   src -> d0 -> d1 -> ... -> d(n-1)
// d0's ring receiver stores each drained batch into its own shard AND into
// the d0 -> d1 ring (the bytes are already in its shared memory), so every
// GPU sends each byte at most once and the hops overlap batch by batch.
// The plan is unchanged -- the same tasks, the same destination bytes; only
// which GPU a task's bytes leave from changes (execution detail, like the
// reference's SPEC.md:192 leaving routing to the transport).
//
// Grouping: remote tasks (source and destination on different slots) of one
// layer with the same source rank, tensor and bounds.  One member per
// distinct destination slot joins the candidate chain; a group with fewer than
// two candidates stays point-to-point.  Groups are decided greedily, largest
// first: the chain orders its members by the egress their slots already
// carry (least loaded first -- the last member forwards nothing), and a group
// is chained only when that lowers the highest egress among the slots
// involved; otherwise it stays a star from the source.  Deterministic in the
// plan and the placement, so every process of a job derives the same chains.
#include <algorithm>
#include <map>
#include <stdexcept>
#include <tuple>

#include "reshard_b200/reshard.hpp"

namespace reshard {

std::vector<RelayChain> relay_chains(const TransferPlan& plan, const std::function<int(int)>& src_slot,
                                     const std::function<int(int)>& dst_slot) {
  using Key = std::tuple<int, int, std::uint32_t, std::vector<std::int64_t>>;  // layer, src, tensor, bounds
  struct Group {
    std::vector<std::size_t> members;  // task indices within the layer
    std::int64_t bytes = 0;
  };
  std::map<Key, Group> groups;
  std::map<int, std::int64_t> egress;  // slot -> bytes it sends
  for (const auto& [layer, tasks] : plan.tasks_by_layer)
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      const TransferTask& t = tasks[i];
      if (t.is_local() || src_slot(t.src_rank) == dst_slot(t.dst_rank)) continue;
      std::vector<std::int64_t> b;
      b.reserve(2 * t.bounds.ndims());
      for (std::size_t d = 0; d < t.bounds.ndims(); ++d) {
        b.push_back(t.bounds.dim(d).lo);
        b.push_back(t.bounds.dim(d).hi);
      }
      Group& g = groups[Key{layer, t.src_rank, t.tensor_index, std::move(b)}];
      g.members.push_back(i);
      g.bytes = t.byte_size;
    }

  struct Candidate {
    const Key* key;
    const Group* group;
    std::vector<std::size_t> chain;  // one member per distinct destination slot
  };
  std::vector<Candidate> cands;
  for (const auto& [key, g] : groups) {
    const auto& tasks = plan.tasks_by_layer.at(std::get<0>(key));
    std::map<int, std::size_t> by_slot;  // first member (lowest dst rank) per destination slot
    for (std::size_t i : g.members) {
      const int s = dst_slot(tasks[i].dst_rank);
      auto it = by_slot.find(s);
      if (it == by_slot.end() || tasks[i].dst_rank < tasks[it->second].dst_rank) by_slot[s] = i;
    }
    const int s = src_slot(std::get<1>(key));
    if (by_slot.size() < 2) {  // point-to-point only
      egress[s] += g.bytes * static_cast<std::int64_t>(g.members.size());
      continue;
    }
    // members sharing a candidate's slot (several ranks on one GPU) stay direct from the source
    egress[s] += g.bytes * static_cast<std::int64_t>(g.members.size() - by_slot.size());
    Candidate c{&key, &g, {}};
    for (const auto& kv : by_slot) c.chain.push_back(kv.second);
    cands.push_back(std::move(c));
  }
  std::stable_sort(cands.begin(), cands.end(),
                   [](const Candidate& a, const Candidate& b) { return a.group->bytes > b.group->bytes; });

  std::vector<RelayChain> out;
  for (auto& c : cands) {
    const int layer = std::get<0>(*c.key);
    const auto& tasks = plan.tasks_by_layer.at(layer);
    const int s = src_slot(std::get<1>(*c.key));
    const std::int64_t b = c.group->bytes;
    const std::int64_t n = static_cast<std::int64_t>(c.chain.size());
    auto slot_of = [&](std::size_t i) { return dst_slot(tasks[i].dst_rank); };
    std::stable_sort(c.chain.begin(), c.chain.end(), [&](std::size_t x, std::size_t y) {
      const std::int64_t ex = egress[slot_of(x)], ey = egress[slot_of(y)];
      return ex != ey ? ex < ey : slot_of(x) < slot_of(y);
    });
    std::int64_t star = egress[s] + n * b;
    std::int64_t chain = egress[s] + b;
    for (std::size_t k = 0; k < c.chain.size(); ++k) {
      const std::int64_t e = egress[slot_of(c.chain[k])];
      star = std::max(star, e);
      chain = std::max(chain, e + (k + 1 < c.chain.size() ? b : 0));
    }
    if (chain >= star) {
      egress[s] += n * b;
      continue;
    }
    egress[s] += b;
    for (std::size_t k = 0; k + 1 < c.chain.size(); ++k) egress[slot_of(c.chain[k])] += b;
    out.push_back({layer, std::move(c.chain)});
  }
  std::sort(out.begin(), out.end(), [](const RelayChain& a, const RelayChain& b) {
    return a.layer != b.layer ? a.layer < b.layer : a.tasks < b.tasks;
  });
  return out;
}

}  // namespace reshard
