// extern "C" boundary of libreshard_b200.so (include/rs_reshard.h).
// Exceptions never cross it: std::invalid_argument / DomainError -> RS_EDOMAIN,
// IntegrityError / plan parse errors -> RS_EINTEGRITY, SystemError (CUDA) ->
// RS_ESYSTEM; the message is kept per thread for rs_last_error().
#include <algorithm>
#include <atomic>
#include <cstring>
#include <memory>
#include <set>
#include <sstream>
#include <string>

#include "engine/engine.hpp"
#include "reshard_b200/reshard.hpp"
#include "rs_reshard.h"

struct rs_plan {
  reshard::ModelSpec model;
  reshard::TransferPlan plan;
  std::int64_t pairs_checked = 0;
  // process-unique identity: an engine skips recompiling the plan it already holds
  std::uint64_t id = next_id();
  static std::uint64_t next_id() {
    static std::atomic<std::uint64_t> counter{0};
    return ++counter;
  }
};

struct rs_engine {
  explicit rs_engine(const rs_engine_options& o) : impl(o) {}
  rsb::Engine impl;
};

namespace {

thread_local std::string g_error;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_error.clear();
    return RS_OK;
  } catch (const rsb::SystemError& e) {
    g_error = e.what();
    return RS_ESYSTEM;
  } catch (const rsb::IntegrityError& e) {
    g_error = e.what();
    return RS_EINTEGRITY;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return RS_EDOMAIN;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return RS_EDOMAIN;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return RS_ESYSTEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return RS_EINTEGRITY;
  }
}

reshard::ParallelConfig to_config(const rs_config* c, int num_layers) {
  if (!c) throw std::invalid_argument("null config");
  if (c->num_ranks < 0 || (c->num_ranks > 0 && !c->ranks)) throw std::invalid_argument("config: bad rank list");
  std::vector<int> ranks(c->ranks, c->ranks + c->num_ranks);
  std::vector<int> stages = c->layer_stage ? std::vector<int>(c->layer_stage, c->layer_stage + num_layers)
                                           : reshard::ParallelConfig::default_layer_assignment(num_layers, c->pp);
  if (c->distributed_optimizer < 0 || c->distributed_optimizer > 2)
    throw std::invalid_argument("config: distributed_optimizer must be 0 (off), 1 (dim chunks) or 2 (flat buckets)");
  if (c->dist_opt_bucket_elems < 0) throw std::invalid_argument("config: negative dist_opt_bucket_elems");
  auto cfg = reshard::ParallelConfig(c->generation_id, c->tp, c->pp, c->dp, std::move(ranks), std::move(stages))
                 .with_distributed_optimizer(c->distributed_optimizer != 0);
  return c->distributed_optimizer == 2 ? cfg.with_flat_buckets(c->dist_opt_bucket_elems) : cfg;
}

// Copies s into buf (truncating); *needed is the full size incl. the NUL.
void put_text(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
}

}  // namespace

extern "C" {

const char* rs_last_error(void) { return g_error.c_str(); }
const char* rs_version(void) { return "reshard_b200 0.1 (sm_100a)"; }

int rs_validate_config(const char* model_spec, const rs_config* cfg, char* buf, size_t cap, size_t* needed,
                       int32_t* num_violations) {
  return guarded([&] {
    auto m = reshard::ModelSpec::parse(model_spec ? model_spec : "");
    auto v = reshard::validate_config(to_config(cfg, m.num_layers), m);
    std::string s;
    for (auto& x : v) s += x + "\n";
    if (num_violations) *num_violations = static_cast<int32_t>(v.size());
    put_text(s, buf, cap, needed);
  });
}

int rs_view(const char* model_spec, const rs_config* cfg, int32_t tensor_index, int32_t rank, int64_t* lo,
            int64_t* hi, int32_t* present) {
  return guarded([&] {
    auto m = reshard::ModelSpec::parse(model_spec ? model_spec : "");
    if (tensor_index < 0 || tensor_index >= static_cast<int32_t>(m.tensors.size()))
      throw std::invalid_argument("tensor index out of range");
    auto v = reshard::view(m.tensors[static_cast<std::size_t>(tensor_index)], to_config(cfg, m.num_layers), rank);
    *present = v.has_value();
    if (v)
      for (std::size_t i = 0; i < v->ndims(); ++i) {
        lo[i] = v->dim(i).lo;
        hi[i] = v->dim(i).hi;
      }
  });
}

int rs_view_range(const char* model_spec, const rs_config* cfg, int32_t tensor_index, int32_t rank, int64_t* lo,
                  int64_t* hi, int32_t* flat) {
  return guarded([&] {
    if (!lo || !hi || !flat) throw std::invalid_argument("null argument");
    auto m = reshard::ModelSpec::parse(model_spec ? model_spec : "");
    if (tensor_index < 0 || tensor_index >= static_cast<int32_t>(m.tensors.size()))
      throw std::invalid_argument("tensor index out of range");
    const auto c = to_config(cfg, m.num_layers);
    const auto ti = static_cast<std::uint32_t>(tensor_index);
    auto r = reshard::bucket_range(m, ti, c, rank);
    *flat = r.has_value();
    *lo = r ? r->first : 0;
    *hi = r ? r->second : 0;
    if (!r)
      if (auto v = reshard::view(m.tensors[ti], c, rank)) *hi = v->element_count();
  });
}

int rs_plan_compute(const char* model_spec, const rs_config* c_old, const rs_config* c_new,
                    const rs_plan_options* opts, rs_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<rs_plan>();
    p->model = reshard::ModelSpec::parse(model_spec ? model_spec : "");
    if (auto v = p->model.validate(); !v.empty()) throw std::invalid_argument("model: " + v.front());
    reshard::PlanOptions o;
    o.balance_sources = opts && opts->balance_sources;
    reshard::PlannerStats st;
    p->plan = reshard::compute_transfer_plan(to_config(c_old, p->model.num_layers),
                                             to_config(c_new, p->model.num_layers), p->model, o, &st);
    p->pairs_checked = st.pairs_checked;
    *out = p.release();
  });
}

int rs_plan_read(const char* model_spec, const char* plan_text, rs_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<rs_plan>();
    p->model = reshard::ModelSpec::parse(model_spec ? model_spec : "");
    std::istringstream is(plan_text ? plan_text : "");
    reshard::TransferPlan parsed = reshard::read_plan(is);
    // read_plan interns ids in appearance order; re-index by name against the
    // model so store lookups use model tensor indices (SURVEY.md §8c caveat)
    std::vector<std::uint32_t> remap(parsed.tensor_ids.size(), 0);
    for (std::size_t pi = 0; pi < parsed.tensor_ids.size(); ++pi) {
      bool found = false;
      for (std::size_t mi = 0; mi < p->model.tensors.size(); ++mi)
        if (p->model.tensors[mi].tensor_id == parsed.tensor_ids[pi]) {
          remap[pi] = static_cast<std::uint32_t>(mi);
          found = true;
        }
      if (!found) throw std::invalid_argument("plan references unknown tensor " + parsed.tensor_ids[pi]);
    }
    p->plan = parsed;
    p->plan.tensor_ids.clear();
    for (const auto& t : p->model.tensors) p->plan.tensor_ids.push_back(t.tensor_id);
    for (auto& kv : p->plan.tasks_by_layer)
      for (auto& t : kv.second) t.tensor_index = remap[t.tensor_index];
    for (auto& kv : p->plan.carryover_by_layer)
      for (auto& k : kv.second) k.tensor_index = remap[k.tensor_index];
    *out = p.release();
  });
}

int rs_plan_write(const rs_plan* plan, char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    if (!plan) throw std::invalid_argument("null plan");
    std::ostringstream os;
    reshard::write_plan(os, plan->plan);
    put_text(os.str(), buf, cap, needed);
  });
}

int rs_plan_summary(const rs_plan* plan, rs_plan_summary_t* out) {
  return guarded([&] {
    if (!plan || !out) throw std::invalid_argument("null argument");
    const auto s = reshard::plan_cost_summary(plan->plan);
    *out = rs_plan_summary_t{};
    out->total_bytes = s.total_bytes;
    out->max_link_bytes = s.max_link_bytes;
    out->task_count = s.task_count;
    out->pairs_checked = plan->pairs_checked;
    out->num_tensors = static_cast<int32_t>(plan->plan.tensor_ids.size());
    std::set<int> layers;
    for (const auto& kv : plan->plan.tasks_by_layer) {
      layers.insert(kv.first);
      for (const auto& t : kv.second) (t.is_local() ? out->local_bytes : out->remote_bytes) += t.byte_size;
    }
    for (const auto& kv : plan->plan.carryover_by_layer) {
      layers.insert(kv.first);
      for (const auto& k : kv.second) {
        out->carryover_bytes += k.byte_size;
        out->carryover_count++;
      }
    }
    out->num_layers_with_work = static_cast<int32_t>(layers.size());
  });
}

int rs_plan_verify(const rs_plan* plan, const rs_config* c_old, const rs_config* c_new, char* buf, size_t cap,
                   size_t* needed, int32_t* num_violations) {
  return guarded([&] {
    if (!plan) throw std::invalid_argument("null plan");
    const int L = plan->model.num_layers;
    auto v = reshard::verify_plan(plan->plan, to_config(c_old, L), to_config(c_new, L), plan->model);
    std::string s;
    for (auto& x : v) s += x + "\n";
    if (num_violations) *num_violations = static_cast<int32_t>(v.size());
    put_text(s, buf, cap, needed);
  });
}

void rs_plan_destroy(rs_plan* plan) { delete plan; }

int rs_chunk_bounds(int32_t ndims, const int64_t* lo, const int64_t* hi, int64_t max_bytes, int64_t bpe,
                    int64_t* out_lo, int64_t* out_hi, int64_t cap, int64_t* count) {
  return guarded([&] {
    std::vector<reshard::Interval> b;
    for (int32_t i = 0; i < ndims; ++i) b.push_back({lo[i], hi[i]});
    auto pieces = reshard::chunk_bounds(reshard::ShardView(b), max_bytes, bpe);
    *count = static_cast<int64_t>(pieces.size());
    for (std::size_t p = 0; p < pieces.size() && static_cast<int64_t>(p) < cap; ++p)
      for (int32_t i = 0; i < ndims; ++i) {
        out_lo[p * static_cast<std::size_t>(ndims) + static_cast<std::size_t>(i)] = pieces[p].dim(static_cast<std::size_t>(i)).lo;
        out_hi[p * static_cast<std::size_t>(ndims) + static_cast<std::size_t>(i)] = pieces[p].dim(static_cast<std::size_t>(i)).hi;
      }
  });
}

int rs_engine_create(const rs_engine_options* opts, rs_engine** out) {
  return guarded([&] {
    if (!opts || !out) throw std::invalid_argument("null argument");
    *out = new rs_engine(*opts);
  });
}

void rs_engine_destroy(rs_engine* e) { delete e; }

int rs_store_layout(rs_engine* e, int32_t which, const char* model_spec, const rs_config* cfg,
                    const int32_t* rank_device) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    auto m = reshard::ModelSpec::parse(model_spec ? model_spec : "");
    auto c = to_config(cfg, m.num_layers);
    std::vector<int> rd(static_cast<std::size_t>(c.world_size()), 0);
    if (rank_device)
      for (std::size_t i = 0; i < rd.size(); ++i) rd[i] = rank_device[i];
    e->impl.layout(which, m, c, rd);
  });
}

int rs_store_alloc(rs_engine* e, int32_t which) {
  return guarded([&] { e->impl.alloc(which); });
}

int rs_store_free(rs_engine* e, int32_t which) {
  return guarded([&] { e->impl.free_store(which); });
}

int rs_store_bind(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index, void* dptr, int64_t nbytes) {
  return guarded([&] { e->impl.bind(which, rank, static_cast<std::uint32_t>(tensor_index), dptr, nbytes); });
}

int rs_store_ptr(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index, void** dptr, int64_t* nbytes) {
  return guarded([&] {
    const rsb::Entry* en = e->impl.store(which).find(rank, static_cast<std::uint32_t>(tensor_index));
    if (!en) throw std::invalid_argument("shard store: no buffer for rank " + std::to_string(rank) + " tensor " +
                                         std::to_string(tensor_index));
    *dptr = en->ptr;
    *nbytes = en->nbytes;
  });
}

int rs_store_bytes(rs_engine* e, int32_t which, int64_t* total) {
  return guarded([&] { *total = e->impl.store(which).total_bytes(); });
}

int rs_store_entries(rs_engine* e, int32_t which, int32_t* tensor_index, int32_t* rank, int64_t* nbytes,
                     int64_t cap, int64_t* count) {
  return guarded([&] {
    const auto& entries = e->impl.store(which).entries;
    *count = static_cast<int64_t>(entries.size());
    for (std::size_t k = 0; k < entries.size() && static_cast<int64_t>(k) < cap; ++k) {
      tensor_index[k] = static_cast<int32_t>(entries[k].ti);
      rank[k] = entries[k].rank;
      nbytes[k] = entries[k].nbytes;
    }
  });
}

int rs_store_read(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index, int64_t offset, int64_t nbytes,
                  void* host) {
  return guarded([&] {
    const rsb::Entry* en = e->impl.store(which).find(rank, static_cast<std::uint32_t>(tensor_index));
    if (!en || !en->ptr) throw std::invalid_argument("store read: no such entry");
    if (offset < 0 || nbytes < 0 || offset + nbytes > en->nbytes) throw std::invalid_argument("store read: out of range");
    rsb::cuda_check(cudaMemcpy(host, en->ptr + offset, static_cast<std::size_t>(nbytes), cudaMemcpyDeviceToHost),
                    "store read");
  });
}

int rs_store_write(rs_engine* e, int32_t which, int32_t rank, int32_t tensor_index, int64_t offset, int64_t nbytes,
                   const void* host) {
  return guarded([&] {
    const rsb::Entry* en = e->impl.store(which).find(rank, static_cast<std::uint32_t>(tensor_index));
    if (!en || !en->ptr) throw std::invalid_argument("store write: no such entry");
    if (offset < 0 || nbytes < 0 || offset + nbytes > en->nbytes) throw std::invalid_argument("store write: out of range");
    rsb::cuda_check(cudaMemcpy(en->ptr + offset, host, static_cast<std::size_t>(nbytes), cudaMemcpyHostToDevice),
                    "store write");
  });
}

int rs_fill_pattern(rs_engine* e, int32_t which, uint64_t seed) {
  return guarded([&] { e->impl.fill_pattern(which, seed); });
}

int rs_verify_pattern(rs_engine* e, int32_t which, uint64_t seed, int64_t* mismatches, int64_t* first_bad_entry) {
  return guarded([&] {
    std::int64_t first = -1;
    *mismatches = e->impl.verify_pattern(which, seed, &first);
    if (first_bad_entry) *first_bad_entry = first;
  });
}

int rs_prepare(rs_engine* e, const rs_plan* plan) {
  return guarded([&] {
    if (!e || !plan) throw std::invalid_argument("null argument");
    e->impl.prepare(plan->plan, plan->id);
  });
}

int rs_run(rs_engine* e, rs_exec_report* report) {
  return guarded([&] {
    *report = e->impl.run();
    if (!report->ok) throw rsb::IntegrityError(report->error);
  });
}

int rs_execute(rs_engine* e, const rs_plan* plan, rs_exec_report* report) {
  return guarded([&] {
    if (!e->impl.prepared_for(plan->id)) e->impl.prepare(plan->plan, plan->id);
    *report = e->impl.run();
    if (!report->ok) throw rsb::IntegrityError(report->error);
  });
}

int rs_execute_host(rs_engine* e, const rs_plan* plan, void* const* host_src, void* const* host_dst,
                    int32_t window_layers, rs_exec_report* report) {
  return guarded([&] {
    if (!e || !plan || !host_src || !host_dst) throw std::invalid_argument("null argument");
    if (window_layers > 0 && e->impl.window_layers() != window_layers) e->impl.set_window(window_layers);
    if (!e->impl.prepared_for(plan->id)) e->impl.prepare(plan->plan, plan->id);
    *report = e->impl.run_host(host_src, host_dst, window_layers);
    if (!report->ok) throw rsb::IntegrityError(report->error);
  });
}

int rs_switch(rs_engine* e, const rs_plan* plan, void* const* drain_events, int32_t swap,
              rs_switch_stats* stats) {
  return guarded([&] {
    if (!e || !plan || !stats) throw std::invalid_argument("null argument");
    if (!e->impl.prepared_for(plan->id)) e->impl.prepare(plan->plan, plan->id);
    *stats = e->impl.switch_step(drain_events, swap != 0);
    if (!stats->exec.ok) throw rsb::IntegrityError(stats->exec.error);
  });
}

int rs_store_swap(rs_engine* e) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null argument");
    e->impl.swap_stores();
  });
}

}  // extern "C"

extern "C" {

int rs_host_alloc(size_t bytes, void** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    rsb::cuda_check(cudaHostAlloc(out, bytes, cudaHostAllocPortable), "cudaHostAlloc");
  });
}

int rs_host_free(void* p) {
  return guarded([&] { rsb::cuda_check(cudaFreeHost(p), "cudaFreeHost"); });
}

}  // extern "C"

extern "C" {

int rs_comm_alloc(rs_engine* e) {
  return guarded([&] { e->impl.comm_alloc(); });
}

int rs_comm_alloc_plan(rs_engine* e, const rs_plan* plan) {
  return guarded([&] {
    if (!e || !plan) throw std::invalid_argument("bad argument");
    e->impl.comm_alloc_plan(plan->plan);
  });
}

int rs_arena_export(rs_engine* e, int32_t which, int32_t slot, void* handle, int64_t* arena_bytes) {
  return guarded([&] {
    if (!handle || !arena_bytes) throw std::invalid_argument("null argument");
    *arena_bytes = e->impl.export_arena(which, slot, handle);
  });
}

int rs_arena_import(rs_engine* e, int32_t which, int32_t slot, const void* handle, int64_t arena_bytes) {
  return guarded([&] {
    if (!handle) throw std::invalid_argument("null argument");
    e->impl.import_arena(which, slot, handle, arena_bytes);
  });
}

int rs_plan_traffic_ex(const rs_plan* plan, const rs_config* c_old, const int32_t* slot_old, const rs_config* c_new,
                       const int32_t* slot_new, int32_t nslots, int32_t flags, int64_t* out) {
  return guarded([&] {
    if (!plan || !out || nslots < 1) throw std::invalid_argument("bad argument");
    if (flags & ~RS_TRAFFIC_RELAY) throw std::invalid_argument("plan traffic: unknown flags");
    const int L = plan->model.num_layers;
    const auto co = to_config(c_old, L), cn = to_config(c_new, L);
    auto slot_in = [&](const reshard::ParallelConfig& c, const int32_t* slots, int rank) {
      const int s = slots ? slots[c.index_of(rank)] : c.index_of(rank);
      if (s < 0 || s >= nslots) throw std::invalid_argument("slot out of range");
      return s;
    };
    auto src_slot = [&](int r) { return slot_in(co, slot_old, r); };
    auto dst_slot = [&](int r) { return slot_in(cn, slot_new, r); };
    // relay chains (extension): hop k of a chain leaves from the previous
    // destination's slot instead of the source's
    std::map<std::pair<int, std::size_t>, int> sender_slot;  // (layer, task index) -> slot it leaves from
    if (flags & RS_TRAFFIC_RELAY)
      for (const auto& ch : reshard::relay_chains(plan->plan, src_slot, dst_slot)) {
        const auto& tasks = plan->plan.tasks_by_layer.at(ch.layer);
        for (std::size_t k = 1; k < ch.tasks.size(); ++k)
          sender_slot[{ch.layer, ch.tasks[k]}] = dst_slot(tasks[ch.tasks[k - 1]].dst_rank);
      }
    std::fill(out, out + 4 * nslots, 0);
    for (const auto& [layer, tasks] : plan->plan.tasks_by_layer)
      for (std::size_t i = 0; i < tasks.size(); ++i) {
        const auto& t = tasks[i];
        const auto d = static_cast<std::size_t>(dst_slot(t.dst_rank));
        auto it = sender_slot.find({layer, i});
        const auto s = static_cast<std::size_t>(it == sender_slot.end() ? src_slot(t.src_rank) : it->second);
        if (t.is_local() || s == d) {
          out[4 * d + 2] += t.byte_size;  // moved inside one GPU
        } else {
          out[4 * s + 0] += t.byte_size;  // egress
          out[4 * d + 1] += t.byte_size;  // ingress
        }
      }
    for (const auto& kv : plan->plan.carryover_by_layer)
      for (const auto& k : kv.second) out[4 * static_cast<std::size_t>(dst_slot(k.rank)) + 3] += k.byte_size;
  });
}

int rs_plan_traffic(const rs_plan* plan, const rs_config* c_old, const int32_t* slot_old, const rs_config* c_new,
                    const int32_t* slot_new, int32_t nslots, int64_t* out) {
  return rs_plan_traffic_ex(plan, c_old, slot_old, c_new, slot_new, nslots, 0, out);
}

int rs_plan_placement(const char* model_spec, const rs_config* c_old, const rs_config* c_new,
                      const int32_t* candidates, int32_t ncand, const rs_placement_options* opts,
                      int32_t* ranks_out, rs_placement_result* out) {
  return guarded([&] {
    if (!candidates || ncand < 1 || !ranks_out || !out) throw std::invalid_argument("bad argument");
    auto m = reshard::ModelSpec::parse(model_spec ? model_spec : "");
    const auto co = to_config(c_old, m.num_layers), cn = to_config(c_new, m.num_layers);
    reshard::PlacementOptions po;
    if (opts) {
      if (opts->nvlink_gbs < 0 || opts->hbm_gbs < 0 || opts->exhaustive_limit < 0)
        throw std::invalid_argument("placement: negative option");
      if (opts->nvlink_gbs > 0) po.nvlink_gbs = opts->nvlink_gbs;
      if (opts->hbm_gbs > 0) po.hbm_gbs = opts->hbm_gbs;
      if (opts->exhaustive_limit > 0) po.exhaustive_limit = opts->exhaustive_limit;
      po.balance_sources = opts->balance_sources != 0;
    }
    const auto r = reshard::choose_placement(co, cn, m, std::vector<int>(candidates, candidates + ncand), po);
    std::copy(r.ranks.begin(), r.ranks.end(), ranks_out);
    *out = rs_placement_result{};
    out->roofline_ms = r.roofline_s * 1e3;
    out->given_roofline_ms = r.given_roofline_s * 1e3;
    out->remote_bytes = r.remote_bytes;
    out->local_bytes = r.local_bytes;
    out->carryover_bytes = r.carryover_bytes;
    out->max_link_bytes = r.max_link_bytes;
    out->given_remote_bytes = r.given_remote_bytes;
    out->given_local_bytes = r.given_local_bytes;
    out->given_carryover_bytes = r.given_carryover_bytes;
    out->given_max_link_bytes = r.given_max_link_bytes;
    out->evaluated = r.evaluated;
    out->exhaustive = r.exhaustive;
  });
}

}  // extern "C"

extern "C" {

int rs_trace_read(rs_engine* e, int32_t device, rs_trace_record_t* out, int64_t cap, int64_t* count) {
  return guarded([&] {
    if (!e || !count || cap < 0 || (cap > 0 && !out)) throw std::invalid_argument("bad argument");
    static_assert(sizeof(rs_trace_record_t) == sizeof(rs_trace_record), "trace record layout");
    const auto recs = e->impl.trace(device);
    *count = static_cast<int64_t>(recs.size());
    const std::size_t n = std::min<std::size_t>(recs.size(), static_cast<std::size_t>(cap));
    if (n) std::memcpy(out, recs.data(), n * sizeof(rs_trace_record));
  });
}

int rs_xfer_info(rs_engine* e, int32_t* rounds, int32_t* ntx, int32_t* nrx) {
  return guarded([&] {
    *rounds = e->impl.xfer_rounds();
    *ntx = static_cast<int32_t>(e->impl.xfer_links(0).size());
    *nrx = static_cast<int32_t>(e->impl.xfer_links(1).size());
  });
}

int rs_xfer_link(rs_engine* e, int32_t dir, int32_t index, int32_t* peer_slot, int32_t* src_rank, int32_t* dst_rank,
                 void** buffer, int64_t* buffer_bytes, int64_t* round_bytes) {
  return guarded([&] {
    const auto& links = e->impl.xfer_links(dir ? 1 : 0);
    if (index < 0 || index >= static_cast<int32_t>(links.size())) throw std::invalid_argument("xfer: link index");
    const auto& l = links[static_cast<std::size_t>(index)];
    *peer_slot = l.peer_slot;
    *src_rank = l.src_rank;
    *dst_rank = l.dst_rank;
    *buffer = l.buf;
    *buffer_bytes = static_cast<int64_t>(l.buf_bytes);
    if (round_bytes)
      for (std::size_t r = 0; r < l.round_bytes.size(); ++r) round_bytes[r] = static_cast<int64_t>(l.round_bytes[r]);
  });
}

int rs_xfer_step(rs_engine* e, int32_t what, int32_t round) {
  return guarded([&] { e->impl.xfer_step(what, round); });
}

int rs_xfer_stream(rs_engine* e, void** stream) {
  return guarded([&] { *stream = e->impl.xfer_stream(); });
}

}  // extern "C"
