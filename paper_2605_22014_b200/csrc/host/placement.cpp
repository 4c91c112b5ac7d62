// Placement-aware destination rank ordering.
//
// The rank list of a ParallelConfig is semantic: position i of the list gets
// coordinate (tp, dp, pp) = (i % tp, (i / tp) % dp, i / (tp*dp))
// (parallel_config.cpp:19-71), and the planner lets a destination rank source
// every region it already held itself (planner.cpp:139-152: carryover or a
// local task) while everything else crosses a link from the dp-0 owner
// (planner.cpp:154-171).  Which GPU ids fill which positions of C_new therefore
// decides how many bytes cross NVLink and how they pile up per GPU.  The
// reference fixes the list (SPEC.md:192 leaves routing to the simulator);
// choose_placement searches it.
//
// Decomposition.  With balance_sources off, the tasks generated for position p
// depend only on p and the rank id g placed there (the self-held test looks up
// g in C_old; the source of a non-held region is C_old's dp-0 owner).  G
// cyclic probe lists list_k[p] = cand[(p + k) % G] cover every (p, g) pair
// once, so G planner calls give the per-(p, g) traffic F[p][g][u] (bytes from
// GPU u), local-task and carryover bytes.  A placement's roofline is then
//   t = max_g max(max(out_g, in_g) / NVLink, (out_g + in_g + 2 local_g + 2 carry_g) / HBM)
// (SURVEY.md §8(d)), one rank per GPU.  Exhaustive over injective assignments
// when the count is small (8 of 8: 40320), else best-improvement local search
// (swap two positions / replace one with an unused candidate) from the given
// list.  The chosen list is re-planned for real and scored from that plan, so
// the reported numbers never rely on the decomposition.
#include <algorithm>
#include <cmath>
#include <map>
#include <stdexcept>
#include <unordered_map>

#include "reshard_b200/reshard.hpp"

namespace reshard {

namespace {

struct Score {
  double t = 0;  // seconds
  std::int64_t remote = 0, local = 0, carry = 0, max_link = 0;
};

bool better(const Score& a, const Score& b) {
  const double tol = 1e-12 * std::max(a.t, b.t);
  if (a.t < b.t - tol) return true;
  if (a.t > b.t + tol) return false;
  return a.remote < b.remote;
}

struct Gpus {
  std::vector<int> ids;                 // dense index -> rank id (GPU)
  std::unordered_map<int, int> index;   // rank id -> dense index
  int of(int id) {
    auto it = index.find(id);
    if (it != index.end()) return it->second;
    index[id] = static_cast<int>(ids.size());
    ids.push_back(id);
    return static_cast<int>(ids.size()) - 1;
  }
};

Score finish(const std::vector<std::int64_t>& out, const std::vector<std::int64_t>& in,
             const std::vector<std::int64_t>& hbm, std::int64_t remote, std::int64_t local, std::int64_t carry,
             const PlacementOptions& o) {
  Score s;
  s.remote = remote;
  s.local = local;
  s.carry = carry;
  for (std::size_t u = 0; u < out.size(); ++u) {
    const std::int64_t link = std::max(out[u], in[u]);
    s.max_link = std::max(s.max_link, link);
    s.t = std::max({s.t, static_cast<double>(link) / (o.nvlink_gbs * 1e9),
                    static_cast<double>(hbm[u]) / (o.hbm_gbs * 1e9)});
  }
  return s;
}

Score score_plan(const TransferPlan& plan, Gpus& gpus, const PlacementOptions& o) {
  std::map<int, std::int64_t> out, in, hbm;
  std::int64_t remote = 0, local = 0, carry = 0;
  for (const auto& kv : plan.tasks_by_layer)
    for (const auto& t : kv.second) {
      if (t.is_local()) {
        hbm[t.dst_rank] += 2 * t.byte_size;
        local += t.byte_size;
      } else {
        out[t.src_rank] += t.byte_size;
        in[t.dst_rank] += t.byte_size;
        hbm[t.src_rank] += t.byte_size;
        hbm[t.dst_rank] += t.byte_size;
        remote += t.byte_size;
      }
    }
  for (const auto& kv : plan.carryover_by_layer)
    for (const auto& k : kv.second) {
      hbm[k.rank] += 2 * k.byte_size;
      carry += k.byte_size;
    }
  for (auto* m : {&out, &in, &hbm})
    for (const auto& kv : *m) gpus.of(kv.first);
  const std::size_t U = gpus.ids.size();
  std::vector<std::int64_t> vo(U, 0), vi(U, 0), vh(U, 0);
  for (const auto& kv : out) vo[static_cast<std::size_t>(gpus.of(kv.first))] = kv.second;
  for (const auto& kv : in) vi[static_cast<std::size_t>(gpus.of(kv.first))] = kv.second;
  for (const auto& kv : hbm) vh[static_cast<std::size_t>(gpus.of(kv.first))] = kv.second;
  return finish(vo, vi, vh, remote, local, carry, o);
}

}  // namespace

PlacementResult choose_placement(const ParallelConfig& c_old, const ParallelConfig& c_new, const ModelSpec& model,
                                 const std::vector<int>& candidates, const PlacementOptions& opts) {
  if (opts.nvlink_gbs <= 0 || opts.hbm_gbs <= 0) throw std::invalid_argument("placement: bandwidths must be > 0");
  const int P = c_new.world_size();
  const int G = static_cast<int>(candidates.size());
  if (G < P) throw std::invalid_argument("placement: fewer candidate ranks than positions in the new config");
  {
    std::vector<int> c = candidates;
    std::sort(c.begin(), c.end());
    if (std::adjacent_find(c.begin(), c.end()) != c.end())
      throw std::invalid_argument("placement: duplicate candidate rank");
    if (!c.empty() && c.front() < 0) throw std::invalid_argument("placement: negative candidate rank");
  }
  if (auto v = validate_config(c_new, model); !v.empty())
    throw std::invalid_argument("placement: invalid destination config: " + v.front());

  Gpus gpus;
  for (int r : c_old.ranks()) gpus.of(r);
  for (int r : candidates) gpus.of(r);
  const std::size_t U = gpus.ids.size();
  if (static_cast<double>(P) * G * static_cast<double>(U) > 64e6)
    throw std::invalid_argument("placement: problem too large for the dense traffic table");

  // F[(p * G + c) * U + u]: bytes position p needs from GPU u when candidate c sits at p
  std::vector<std::int64_t> F(static_cast<std::size_t>(P) * G * U, 0);
  std::vector<std::int64_t> loc(static_cast<std::size_t>(P) * G, 0), car(static_cast<std::size_t>(P) * G, 0);
  std::unordered_map<int, int> cand_index;
  for (int c = 0; c < G; ++c) cand_index[candidates[static_cast<std::size_t>(c)]] = c;
  PlanOptions popt;
  popt.balance_sources = opts.balance_sources;
  for (int k = 0; k < G; ++k) {
    std::vector<int> list(static_cast<std::size_t>(P));
    for (int p = 0; p < P; ++p) list[static_cast<std::size_t>(p)] = candidates[static_cast<std::size_t>((p + k) % G)];
    const ParallelConfig probe =
        ParallelConfig(c_new.generation_id(), c_new.tp(), c_new.pp(), c_new.dp(), list, c_new.layer_assignment())
            .with_distributed_optimizer(c_new.distributed_optimizer());
    const TransferPlan plan = compute_transfer_plan(c_old, probe, model, popt);
    auto cell = [&](int rank) {
      const int p = probe.index_of(rank);
      return static_cast<std::size_t>(p) * G + static_cast<std::size_t>(cand_index.at(rank));
    };
    for (const auto& kv : plan.tasks_by_layer)
      for (const auto& t : kv.second) {
        const std::size_t pc = cell(t.dst_rank);
        if (t.is_local()) loc[pc] += t.byte_size;
        else F[pc * U + static_cast<std::size_t>(gpus.of(t.src_rank))] += t.byte_size;
      }
    for (const auto& kv : plan.carryover_by_layer)
      for (const auto& c : kv.second) car[cell(c.rank)] += c.byte_size;
  }

  // incremental state of a (partial) assignment
  std::vector<std::int64_t> out(U, 0), in(U, 0), hbm(U, 0);
  std::int64_t remote = 0, local = 0, carry = 0;
  auto apply = [&](int p, int c, int sign) {
    const std::size_t pc = static_cast<std::size_t>(p) * G + static_cast<std::size_t>(c);
    const std::size_t g = static_cast<std::size_t>(gpus.of(candidates[static_cast<std::size_t>(c)]));
    const std::int64_t* row = &F[pc * U];
    for (std::size_t u = 0; u < U; ++u) {
      const std::int64_t b = row[u] * sign;
      if (!b) continue;
      out[u] += b;
      hbm[u] += b;
      in[g] += b;
      hbm[g] += b;
      remote += b;
    }
    hbm[g] += 2 * (loc[pc] + car[pc]) * sign;
    local += loc[pc] * sign;
    carry += car[pc] * sign;
  };

  PlacementResult res;
  std::vector<int> assign(static_cast<std::size_t>(P), -1), best_assign;
  Score best;
  bool have = false;
  double count = 1;
  for (int p = 0; p < P; ++p) count *= static_cast<double>(G - p);
  res.exhaustive = count <= static_cast<double>(opts.exhaustive_limit);
  if (res.exhaustive) {
    std::vector<char> used(static_cast<std::size_t>(G), 0);
    auto dfs = [&](auto&& self, int p) -> void {
      if (p == P) {
        ++res.evaluated;
        const Score s = finish(out, in, hbm, remote, local, carry, opts);
        if (!have || better(s, best)) {
          best = s;
          best_assign = assign;
          have = true;
        }
        return;
      }
      for (int c = 0; c < G; ++c) {
        if (used[static_cast<std::size_t>(c)]) continue;
        used[static_cast<std::size_t>(c)] = 1;
        assign[static_cast<std::size_t>(p)] = c;
        apply(p, c, +1);
        self(self, p + 1);
        apply(p, c, -1);
        used[static_cast<std::size_t>(c)] = 0;
      }
    };
    dfs(dfs, 0);
  } else {
    // start from the given list where it is drawn from the candidates
    std::vector<char> used(static_cast<std::size_t>(G), 0);
    for (int p = 0; p < P; ++p) {
      auto it = cand_index.find(c_new.ranks()[static_cast<std::size_t>(p)]);
      if (it != cand_index.end() && !used[static_cast<std::size_t>(it->second)]) {
        assign[static_cast<std::size_t>(p)] = it->second;
        used[static_cast<std::size_t>(it->second)] = 1;
      }
    }
    for (int p = 0, c = 0; p < P; ++p)
      if (assign[static_cast<std::size_t>(p)] < 0) {
        while (used[static_cast<std::size_t>(c)]) ++c;
        assign[static_cast<std::size_t>(p)] = c;
        used[static_cast<std::size_t>(c)] = 1;
      }
    for (int p = 0; p < P; ++p) apply(p, assign[static_cast<std::size_t>(p)], +1);
    best = finish(out, in, hbm, remote, local, carry, opts);
    for (bool improved = true; improved;) {
      improved = false;
      Score move_best = best;
      int mp = -1, mq = -1, mc = -1;
      for (int p = 0; p < P; ++p) {
        const int cp = assign[static_cast<std::size_t>(p)];
        for (int q = p + 1; q < P; ++q) {  // swap positions p and q
          const int cq = assign[static_cast<std::size_t>(q)];
          apply(p, cp, -1); apply(q, cq, -1); apply(p, cq, +1); apply(q, cp, +1);
          ++res.evaluated;
          const Score s = finish(out, in, hbm, remote, local, carry, opts);
          if (better(s, move_best)) { move_best = s; mp = p; mq = q; mc = -1; }
          apply(p, cq, -1); apply(q, cp, -1); apply(p, cp, +1); apply(q, cq, +1);
        }
        for (int c = 0; c < G; ++c) {  // replace p's rank with an unused candidate
          if (used[static_cast<std::size_t>(c)]) continue;
          apply(p, cp, -1); apply(p, c, +1);
          ++res.evaluated;
          const Score s = finish(out, in, hbm, remote, local, carry, opts);
          if (better(s, move_best)) { move_best = s; mp = p; mq = -1; mc = c; }
          apply(p, c, -1); apply(p, cp, +1);
        }
      }
      if (mp >= 0) {
        improved = true;
        best = move_best;
        const int cp = assign[static_cast<std::size_t>(mp)];
        if (mq >= 0) {
          const int cq = assign[static_cast<std::size_t>(mq)];
          apply(mp, cp, -1); apply(mq, cq, -1); apply(mp, cq, +1); apply(mq, cp, +1);
          std::swap(assign[static_cast<std::size_t>(mp)], assign[static_cast<std::size_t>(mq)]);
        } else {
          apply(mp, cp, -1); apply(mp, mc, +1);
          used[static_cast<std::size_t>(cp)] = 0;
          used[static_cast<std::size_t>(mc)] = 1;
          assign[static_cast<std::size_t>(mp)] = mc;
        }
      }
    }
    best_assign = assign;
  }

  res.ranks.resize(static_cast<std::size_t>(P));
  for (int p = 0; p < P; ++p)
    res.ranks[static_cast<std::size_t>(p)] = candidates[static_cast<std::size_t>(best_assign[static_cast<std::size_t>(p)])];
  // Score the chosen and the given lists from real plans.
  const ParallelConfig chosen =
      ParallelConfig(c_new.generation_id(), c_new.tp(), c_new.pp(), c_new.dp(), res.ranks, c_new.layer_assignment())
          .with_distributed_optimizer(c_new.distributed_optimizer());
  const Score sc = score_plan(compute_transfer_plan(c_old, chosen, model, popt), gpus, opts);
  const Score sg = score_plan(compute_transfer_plan(c_old, c_new, model, popt), gpus, opts);
  if (!opts.balance_sources && (sc.remote != best.remote || sc.local != best.local || sc.carry != best.carry))
    throw std::logic_error("placement: decomposed traffic disagrees with the re-planned placement");
  res.roofline_s = sc.t;
  res.remote_bytes = sc.remote;
  res.local_bytes = sc.local;
  res.carryover_bytes = sc.carry;
  res.max_link_bytes = sc.max_link;
  res.given_roofline_s = sg.t;
  res.given_remote_bytes = sg.remote;
  res.given_local_bytes = sg.local;
  res.given_carryover_bytes = sg.carry;
  res.given_max_link_bytes = sg.max_link;
  // never worse than the list the caller already has
  if (better(sg, sc) && std::all_of(c_new.ranks().begin(), c_new.ranks().end(),
                                    [&](int r) { return cand_index.count(r) != 0; })) {
    res.ranks = c_new.ranks();
    res.roofline_s = sg.t;
    res.remote_bytes = sg.remote;
    res.local_bytes = sg.local;
    res.carryover_bytes = sg.carry;
    res.max_link_bytes = sg.max_link;
  }
  return res;
}

}  // namespace reshard
