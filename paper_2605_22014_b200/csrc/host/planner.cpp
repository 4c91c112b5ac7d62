// Metadata-only transfer planner and its exact completeness check.
//
// compute_transfer_plan follows proj/src/planner.cpp:57-192 decision for
// decision (tile each destination view by the old TP block partition;
// self-held regions become carryovers when the local linear layout is
// unchanged (planner.cpp:31-42) or local tasks otherwise; other regions are
// sourced from the dp-index-0 replica, lowest rank id for replicated tensors,
// optional round-robin balance_sources), so write_plan output is
// byte-identical to the reference's.
//
// verify_plan reports the same violations with the same messages as the
// reference's brute-force oracle (planner.cpp:194-303), but counts coverage on
// a coordinate-compressed grid of cells instead of per element.
#include <algorithm>
#include <map>
#include <stdexcept>

#include "reshard_b200/reshard.hpp"

namespace reshard {

namespace {

// Row-major linear offset of `p` (the region origin) inside `owner`, and
// whether every non-degenerate axis of `region` has the same stride in both
// owners -- the "layout unchanged" test of planner.cpp:31-42.
bool same_local_layout(const ShardView& owner_old, const ShardView& owner_new,
                       const ShardView& region) {
  const std::size_t nd = region.ndims();
  std::int64_t stride_old = 1, stride_new = 1, off_old = 0, off_new = 0;
  bool strides_match = true;
  for (std::size_t k = nd; k-- > 0;) {
    off_old += (region.dim(k).lo - owner_old.dim(k).lo) * stride_old;
    off_new += (region.dim(k).lo - owner_new.dim(k).lo) * stride_new;
    if (region.dim(k).length() > 1 && stride_old != stride_new) strides_match = false;
    stride_old *= owner_old.dim(k).length();
    stride_new *= owner_new.dim(k).length();
  }
  return off_old == off_new && strides_match;
}

// Local layout of a held region: the owner block and the flat offset of its
// first held element (flat-bucket shards hold a sub-range of the block).
bool same_local_layout_flat(const ShardView& block_old, std::int64_t lo_old, const ShardView& block_new,
                            std::int64_t lo_new, const ShardView& region) {
  return block_old == block_new && lo_old == lo_new && same_local_layout(block_old, block_new, region);
}

// Extension: a DP-sharded tensor where either config uses
// Megatron's flat buckets.  What each rank holds is a list of boxes
// (held_boxes); every destination box is tiled by every source box of the
// old TP blocks: DP-sharded sources are unique per element, replicated
// sources come from dp index 0 (the reference's choice, planner.cpp:154-171).
// Self-held boxes become carryovers when the block and the flat offset are
// unchanged, local tasks otherwise.
void plan_flat_buckets(TransferPlan& plan, const ModelSpec& model, std::uint32_t ti, const ParallelConfig& c_old,
                       const ParallelConfig& c_new, std::int64_t& pairs) {
  const TensorSpec& t = model.tensors[ti];
  const std::int64_t ebytes = model.element_bytes(t);
  const int s_old = c_old.stage_of_layer(t.layer), s_new = c_new.stage_of_layer(t.layer);
  const bool old_sharded = c_old.distributed_optimizer();
  auto pos_rank = [](const ParallelConfig& c, int tp_i, int dp_i, int s) {
    return c.ranks()[static_cast<std::size_t>(tp_i + c.tp() * (dp_i + c.dp() * s))];
  };
  auto flat_lo = [&](const ParallelConfig& c, int rank) -> std::int64_t {
    auto r = bucket_range(model, ti, c, rank);
    return r ? r->first : 0;
  };
  // source holders in (tp, dp) order: every dp index when the old state is
  // DP-sharded, else dp 0 only.  A tensor without a TP axis is held whole by
  // every TP index, but each TP index's buckets cut it at different places
  // (the other tensors' TP-local sizes differ), so it is sourced from TP
  // index 0's holders only
  struct Source {
    int rank, tp_i, dp_i;
    std::vector<ShardView> boxes;
  };
  std::vector<Source> sources;
  for (int otp = 0; otp < (t.tp_shard_axis ? c_old.tp() : 1); ++otp)
    for (int odp = 0; odp < (old_sharded ? c_old.dp() : 1); ++odp) {
      const int r = pos_rank(c_old, otp, odp, s_old);
      auto boxes = held_boxes(model, ti, c_old, r);
      if (!boxes.empty()) sources.push_back({r, otp, odp, std::move(boxes)});
    }
  for (int dtp = 0; dtp < c_new.tp(); ++dtp)
    for (int ddp = 0; ddp < c_new.dp(); ++ddp) {
      const int dst = pos_rank(c_new, dtp, ddp, s_new);
      const auto dst_boxes = held_boxes(model, ti, c_new, dst);
      if (dst_boxes.empty()) continue;
      const auto v_dst = view(t, c_new, dst);
      const std::int64_t lo_dst = flat_lo(c_new, dst);
      // the destination's own old holding of this tensor, if any
      std::optional<ShardView> v_held;
      int held_tp = -1, held_dp = -1;
      std::int64_t lo_held = 0;
      if (c_old.contains(dst)) {
        const RankCoord oc = c_old.coord_of(dst);
        if (oc.pp == s_old) {
          v_held = view(t, c_old, dst);
          held_tp = oc.tp;
          held_dp = oc.dp;
          lo_held = flat_lo(c_old, dst);
        }
      }
      for (const ShardView& db : dst_boxes)
        for (const Source& src : sources)
          for (const ShardView& sb : src.boxes) {
            ++pairs;
            auto region = intersect(db, sb);
            if (!region) continue;
            const std::int64_t bytes = region->element_count() * ebytes;
            const bool self = v_held && held_tp == src.tp_i && (!old_sharded || held_dp == src.dp_i);
            if (self) {
              if (same_local_layout_flat(*v_held, lo_held, *v_dst, lo_dst, *region))
                plan.carryover_by_layer[t.layer].push_back({ti, t.layer, dst, *region, bytes});
              else
                plan.tasks_by_layer[t.layer].push_back({ti, t.layer, dst, dst, *region, bytes});
              continue;
            }
            plan.tasks_by_layer[t.layer].push_back({ti, t.layer, src.rank, dst, *region, bytes});
          }
    }
}

}  // namespace

TransferPlan compute_transfer_plan(const ParallelConfig& c_old, const ParallelConfig& c_new,
                                   const ModelSpec& model, const PlanOptions& options,
                                   PlannerStats* stats) {
  if (c_old.generation_id() == c_new.generation_id())
    throw std::invalid_argument("compute_transfer_plan: identical generation ids");
  if (auto v = validate_config(c_old, model); !v.empty())
    throw std::invalid_argument("compute_transfer_plan: invalid source config: " + v.front());
  if (auto v = validate_config(c_new, model); !v.empty())
    throw std::invalid_argument("compute_transfer_plan: invalid destination config: " + v.front());

  TransferPlan plan;
  plan.src_config_gen = c_old.generation_id();
  plan.dst_config_gen = c_new.generation_id();
  plan.tensor_ids.reserve(model.tensors.size());

  const int tp_old = c_old.tp(), dp_old = c_old.dp(), tp_new = c_new.tp(), dp_new = c_new.dp();
  std::int64_t pairs = 0, round_robin = 0;

  struct OldBlock {
    int tp_index;
    Interval iv;
  };
  std::vector<OldBlock> old_blocks;

  for (std::uint32_t ti = 0; ti < model.tensors.size(); ++ti) {
    const TensorSpec& t = model.tensors[ti];
    plan.tensor_ids.push_back(t.tensor_id);
    const std::int64_t ebytes = model.element_bytes(t);
    const int s_old = c_old.stage_of_layer(t.layer);
    const int s_new = c_new.stage_of_layer(t.layer);
    const bool sharded = t.tp_shard_axis.has_value();
    const std::size_t axis = sharded ? static_cast<std::size_t>(*t.tp_shard_axis) : 0;
    const std::int64_t axis_len = sharded ? t.shape[axis] : 0;

    // position -> rank within one stage; positions are tp + tp*(dp + dp*stage)
    auto old_rank = [&](int tp_i, int dp_i) {
      return c_old.ranks()[static_cast<std::size_t>(tp_i + tp_old * (dp_i + dp_old * s_old))];
    };
    auto new_rank = [&](int tp_i, int dp_i) {
      return c_new.ranks()[static_cast<std::size_t>(tp_i + tp_new * (dp_i + dp_new * s_new))];
    };

    old_blocks.clear();
    if (sharded) {
      for (int i = 0; i < tp_old; ++i)
        if (auto b = tp_block(axis_len, tp_old, i)) old_blocks.push_back({i, *b});
    } else {
      old_blocks.push_back({-1, {0, 1}});
    }

    if (t.dp_shard_axis && (c_old.flat_buckets() || c_new.flat_buckets())) {
      plan_flat_buckets(plan, model, ti, c_old, c_new, pairs);
      continue;
    }

    // Extension (distributed optimizer): DP-sharded views split the TP block
    // into dp ceil chunks along dp_shard_axis.  Sources that are DP-sharded
    // are unique per (tp, dp) coordinate, so the destination view is tiled by
    // (old TP block x old DP chunk); replicated sources keep the reference's
    // dp0 / round-robin choice.  Without dp sharding this is exactly the
    // reference loop (same order, same pairs_checked).
    const bool dp_old_sharded = c_old.distributed_optimizer() && t.dp_shard_axis.has_value();
    const bool dp_new_sharded = c_new.distributed_optimizer() && t.dp_shard_axis.has_value();
    const std::size_t daxis = t.dp_shard_axis ? static_cast<std::size_t>(*t.dp_shard_axis) : 0;

    const ShardView full = ShardView::full(t.shape);
    auto old_view = [&](int tp_i, int dp_i) -> std::optional<ShardView> {
      ShardView v = full;
      if (sharded) {
        auto b = tp_block(axis_len, tp_old, tp_i);
        if (!b) return std::nullopt;
        v.raw(axis) = *b;
      }
      if (dp_old_sharded) {
        auto c = dp_chunk(v.dim(daxis), dp_old, dp_i);
        if (!c) return std::nullopt;
        v.raw(daxis) = *c;
      }
      return v;
    };
    for (int dtp = 0; dtp < tp_new; ++dtp) {
      ShardView v_dst_tp = full;
      if (sharded) {
        auto b = tp_block(axis_len, tp_new, dtp);
        if (!b) continue;
        v_dst_tp.raw(axis) = *b;
      }
      for (int ddp = 0; ddp < dp_new; ++ddp) {
        ShardView v_dst = v_dst_tp;
        if (dp_new_sharded) {
          auto c = dp_chunk(v_dst.dim(daxis), dp_new, ddp);
          if (!c) continue;  // short axis: this dp index owns nothing
          v_dst.raw(daxis) = *c;
        }
        const int dst = new_rank(dtp, ddp);

        // The destination's own old view of this tensor, if it had one.
        bool held_before = false;  // dst sat on the tensor's old stage
        int held_tp = -1, held_dp = -1;
        std::optional<ShardView> v_held;
        if (c_old.contains(dst)) {
          const RankCoord oc = c_old.coord_of(dst);
          if (oc.pp == s_old) {
            held_before = true;
            held_tp = oc.tp;
            held_dp = oc.dp;
            v_held = old_view(oc.tp, oc.dp);
          }
        }

        for (const OldBlock& ob : old_blocks) {
          ShardView region_tp = v_dst;
          if (sharded) {
            Interval& iv = region_tp.raw(axis);
            iv.lo = std::max(v_dst.dim(axis).lo, ob.iv.lo);
            iv.hi = std::min(v_dst.dim(axis).hi, ob.iv.hi);
            if (iv.lo >= iv.hi) {
              ++pairs;
              continue;
            }
          }
          const int dp_sources = dp_old_sharded ? dp_old : 1;
          for (int sdp = 0; sdp < dp_sources; ++sdp) {
            ++pairs;
            ShardView region = region_tp;
            if (dp_old_sharded) {
              auto src_view = old_view(sharded ? ob.tp_index : 0, sdp);
              if (!src_view) continue;
              Interval& iv = region.raw(daxis);
              iv.lo = std::max(region_tp.dim(daxis).lo, src_view->dim(daxis).lo);
              iv.hi = std::min(region_tp.dim(daxis).hi, src_view->dim(daxis).hi);
              if (iv.lo >= iv.hi) continue;
            }
            const std::int64_t bytes = region.element_count() * ebytes;

            const bool self = held_before && (!sharded || held_tp == ob.tp_index) &&
                              (!dp_old_sharded || held_dp == sdp) && v_held.has_value();
            if (self) {
              if (same_local_layout(*v_held, v_dst, region))
                plan.carryover_by_layer[t.layer].push_back({ti, t.layer, dst, region, bytes});
              else
                plan.tasks_by_layer[t.layer].push_back({ti, t.layer, dst, dst, region, bytes});
              continue;
            }

            int src;
            if (dp_old_sharded) {
              // the dp group's holder (lowest rank id if replicated over TP)
              src = old_rank(sharded ? ob.tp_index : 0, sdp);
              if (!sharded)
                for (int k = 1; k < tp_old; ++k) src = std::min(src, old_rank(k, sdp));
            } else {
              const int src_dp = options.balance_sources ? static_cast<int>(round_robin++ % dp_old) : 0;
              if (sharded) {
                src = old_rank(ob.tp_index, src_dp);
              } else {
                src = old_rank(0, src_dp);
                for (int k = 1; k < tp_old; ++k) src = std::min(src, old_rank(k, src_dp));
              }
            }
            plan.tasks_by_layer[t.layer].push_back({ti, t.layer, src, dst, region, bytes});
          }
        }
      }
    }
  }
  if (stats) stats->pairs_checked = pairs;
  return plan;
}

namespace {

// Exact cover counting over the cells of a compressed grid: every axis is cut
// at every box bound, so each cell is either fully inside or fully outside
// each box.  Returns {elements with cover 0, elements with cover > 1}.
std::pair<std::int64_t, std::int64_t> cover_counts(const ShardView& domain,
                                                   const std::vector<ShardView>& boxes) {
  const std::size_t nd = domain.ndims();
  std::vector<std::vector<std::int64_t>> cuts(nd);
  for (std::size_t k = 0; k < nd; ++k) {
    auto& c = cuts[k];
    c.push_back(domain.dim(k).lo);
    c.push_back(domain.dim(k).hi);
    for (const auto& b : boxes) {
      c.push_back(b.dim(k).lo);
      c.push_back(b.dim(k).hi);
    }
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
  }
  std::vector<std::size_t> seg(nd);
  std::size_t cells = 1;
  for (std::size_t k = 0; k < nd; ++k) {
    seg[k] = cuts[k].size() - 1;
    cells *= seg[k];
  }
  std::vector<std::uint16_t> cover(cells, 0);
  // Mark each box's cell range.
  std::vector<std::size_t> lo(nd), hi(nd), idx(nd);
  for (const auto& b : boxes) {
    for (std::size_t k = 0; k < nd; ++k) {
      lo[k] = static_cast<std::size_t>(std::lower_bound(cuts[k].begin(), cuts[k].end(), b.dim(k).lo) - cuts[k].begin());
      hi[k] = static_cast<std::size_t>(std::lower_bound(cuts[k].begin(), cuts[k].end(), b.dim(k).hi) - cuts[k].begin());
      idx[k] = lo[k];
    }
    while (true) {
      std::size_t flat = 0;
      for (std::size_t k = 0; k < nd; ++k) flat = flat * seg[k] + idx[k];
      if (cover[flat] < 0xffff) ++cover[flat];
      std::size_t k = nd;
      while (k-- > 0) {
        if (++idx[k] < hi[k]) break;
        idx[k] = lo[k];
      }
      if (k == static_cast<std::size_t>(-1)) break;
    }
  }
  std::int64_t gaps = 0, overlaps = 0;
  std::fill(idx.begin(), idx.end(), 0);
  for (std::size_t flat = 0; flat < cells; ++flat) {
    std::size_t rem = flat;
    std::int64_t vol = 1;
    for (std::size_t k = nd; k-- > 0;) {
      const std::size_t i = rem % seg[k];
      rem /= seg[k];
      vol *= cuts[k][i + 1] - cuts[k][i];
    }
    if (cover[flat] == 0) gaps += vol;
    else if (cover[flat] > 1) overlaps += vol;
  }
  return {gaps, overlaps};
}

}  // namespace

std::vector<std::string> verify_plan(const TransferPlan& plan, const ParallelConfig& c_old,
                                     const ParallelConfig& c_new, const ModelSpec& model) {
  std::vector<std::string> out;
  auto complain = [&](std::string msg) {
    if (out.size() < 64) out.push_back(std::move(msg));
  };

  std::vector<int> to_model(plan.tensor_ids.size(), -1);
  for (std::size_t pi = 0; pi < plan.tensor_ids.size(); ++pi) {
    for (std::size_t mi = 0; mi < model.tensors.size(); ++mi)
      if (model.tensors[mi].tensor_id == plan.tensor_ids[pi]) to_model[pi] = static_cast<int>(mi);
    if (to_model[pi] < 0) complain("plan references unknown tensor " + plan.tensor_ids[pi]);
  }

  // does the union of `held` contain `region` (held boxes are disjoint)?
  auto inside = [](const std::vector<ShardView>& held, const ShardView& region) {
    if (held.size() == 1) return held.front().contains(region);
    std::int64_t n = 0;
    for (const auto& h : held)
      if (auto x = intersect(h, region)) n += x->element_count();
    return n == region.element_count();
  };
  std::vector<ShardView> marked, part;
  for (std::size_t mi = 0; mi < model.tensors.size(); ++mi) {
    const TensorSpec& t = model.tensors[mi];
    const auto ti = static_cast<std::uint32_t>(mi);
    // what every rank holds: its view, or the boxes of its flat-bucket range
    std::map<int, std::vector<ShardView>> dst_held, src_held;
    for (const auto& [r, v] : owners(t, c_new)) dst_held[r] = held_boxes(model, ti, c_new, r);
    for (const auto& [r, v] : owners(t, c_old)) src_held[r] = held_boxes(model, ti, c_old, r);
    const auto tasks = plan.tasks_by_layer.find(t.layer);
    const auto keeps = plan.carryover_by_layer.find(t.layer);

    for (const auto& [dst, held] : dst_held) {
      if (held.empty()) continue;  // an empty flat-bucket range
      marked.clear();
      auto mark = [&](const ShardView& region, const char* what) {
        if (!inside(held, region)) {
          complain(std::string(what) + " for tensor " + t.tensor_id + " rank " +
                   std::to_string(dst) + " escapes destination view");
          return;
        }
        marked.push_back(region);
      };
      if (tasks != plan.tasks_by_layer.end()) {
        for (const auto& task : tasks->second) {
          if (task.dst_rank != dst || to_model.at(task.tensor_index) != static_cast<int>(mi)) continue;
          if (task.bounds.element_count() <= 0 || task.byte_size <= 0) {
            complain("empty task for tensor " + t.tensor_id);
            continue;
          }
          auto s = src_held.find(task.src_rank);
          if (s == src_held.end() || s->second.empty())
            complain("task source rank " + std::to_string(task.src_rank) + " owns nothing of tensor " +
                     t.tensor_id);
          else if (!inside(s->second, task.bounds))
            complain("task bounds escape source view for tensor " + t.tensor_id + " src " +
                     std::to_string(task.src_rank));
          mark(task.bounds, "task");
        }
      }
      if (keeps != plan.carryover_by_layer.end()) {
        for (const auto& k : keeps->second) {
          if (k.rank != dst || to_model.at(k.tensor_index) != static_cast<int>(mi)) continue;
          auto s = src_held.find(k.rank);
          if (s == src_held.end() || !inside(s->second, k.bounds))
            complain("carryover not resident in old view for tensor " + t.tensor_id + " rank " +
                     std::to_string(k.rank));
          mark(k.bounds, "carryover");
        }
      }
      std::int64_t gaps = 0, overlaps = 0;
      for (const auto& h : held) {  // held boxes are disjoint: count each on its own
        part.clear();
        for (const auto& m : marked)
          if (auto x = intersect(h, m)) part.push_back(*x);
        const auto [g, o] = cover_counts(h, part);
        gaps += g;
        overlaps += o;
      }
      if (gaps)
        complain("coverage gap: tensor " + t.tensor_id + " rank " + std::to_string(dst) + " missing " +
                 std::to_string(gaps) + " elements");
      if (overlaps)
        complain("coverage overlap: tensor " + t.tensor_id + " rank " + std::to_string(dst) + " has " +
                 std::to_string(overlaps) + " doubly-covered elements");
    }
  }
  return out;
}

std::vector<ShardView> chunk_bounds(const ShardView& bounds, std::int64_t max_bytes,
                                    std::int64_t bytes_per_element) {
  std::vector<ShardView> out;
  const std::int64_t total = bounds.element_count() * bytes_per_element;
  if (total <= max_bytes) {
    out.push_back(bounds);
    return out;
  }
  if (bytes_per_element > max_bytes)
    throw std::invalid_argument("chunk_bounds: one element exceeds the staging budget");
  std::size_t d = 0;
  while (d < bounds.ndims() && bounds.dim(d).length() <= 1) ++d;
  if (d == bounds.ndims()) throw std::logic_error("chunk_bounds: single-element region over budget");
  const std::int64_t unit = total / bounds.dim(d).length();
  const std::int64_t step = std::max<std::int64_t>(1, max_bytes / std::max<std::int64_t>(unit, 1));
  for (std::int64_t lo = bounds.dim(d).lo; lo < bounds.dim(d).hi; lo += step) {
    ShardView piece = bounds;
    piece.raw(d) = {lo, std::min(lo + step, bounds.dim(d).hi)};
    if (piece.element_count() * bytes_per_element <= max_bytes) {
      out.push_back(piece);
    } else {
      auto sub = chunk_bounds(piece, max_bytes, bytes_per_element);
      out.insert(out.end(), sub.begin(), sub.end());
    }
  }
  return out;
}

}  // namespace reshard
