// ref_harness.cpp -- TEST INFRASTRUCTURE. A thin C ABI over the UNMODIFIED
// reference sources (/root/reference/proj/src/{parallel_config,topology,
// transfer_plan,planner,shard_store,transport,executor}.cpp), compiled by
// oracle/Makefile into oracle/_ref/libreshard_ref.so.  It exposes the same
// entry points as oracle/oracle.c (prefix ref_ instead of orc_) so tests can
// pin the C restatement against the reference itself, and bench.py can time
// the reference's own execute_plan as the CPU arm.
//
// Nothing here re-implements the reference algorithm; it only parses the
// shared spec text, calls reshard::compute_transfer_plan / verify_plan /
// write_plan / read_plan / execute_plan, and fills source stores with the
// reference's pattern (ShardStore::pattern_byte, one hash per element for
// speed; bytes identical to ShardStore::fill_pattern).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "reshard/executor.hpp"
#include "reshard/planner.hpp"
#include "reshard/shard_store.hpp"
#include "reshard/topology.hpp"
#include "reshard/transfer_plan.hpp"
#include "reshard/transport.hpp"

using namespace reshard;

extern "C" {
struct ref_config {
  uint64_t gen;
  int32_t tp, pp, dp, nranks;
  const int32_t* ranks;
  const int32_t* layer_stage;
  int32_t distributed_optimizer;  // product extension: the reference cannot express it
  int32_t reserved;
};

struct ref_report {
  int32_t ok;
  int32_t failed_layer;
  int64_t peak_staging_bytes;
  int64_t bytes_moved;
  int64_t local_copy_bytes;
  int32_t layers_processed;
  int32_t pad;
  double seconds;
  char error[512];
};
}

namespace {

ModelSpec parse_spec(const char* text) {
  ModelSpec m;
  std::istringstream is(text);
  std::string line;
  bool have_model = false;
  int64_t uniform = -1;
  while (std::getline(is, line)) {
    auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    std::istringstream ls(line);
    std::string kind;
    if (!(ls >> kind)) continue;
    if (kind == "model") {
      std::string k1, k2;
      ls >> m.name >> k1 >> m.num_layers >> k2 >> m.bytes_per_element;
      have_model = true;
    } else if (kind == "tensor") {
      TensorSpec t;
      std::string shape, axis, role;
      int64_t bpe = 0;
      ls >> t.tensor_id >> t.layer >> shape >> axis >> role >> bpe;
      if (!ls) throw std::runtime_error("spec parse: bad tensor line");
      std::stringstream ss(shape);
      std::string d;
      while (std::getline(ss, d, ',')) t.shape.push_back(std::stoll(d));
      if (axis != "-") t.tp_shard_axis = std::stoi(axis);
      t.role = role == "m1"   ? TensorRole::kOptimizerMoment1
               : role == "m2" ? TensorRole::kOptimizerMoment2
                              : TensorRole::kParameter;
      if (uniform < 0) uniform = bpe;
      if (bpe != uniform)
        throw std::runtime_error("reference ModelSpec holds one bytes_per_element; split the spec by dtype");
      m.tensors.push_back(std::move(t));
    } else {
      throw std::runtime_error("spec parse: unknown record " + kind);
    }
  }
  if (!have_model) throw std::runtime_error("spec parse: missing model record");
  if (uniform > 0) m.bytes_per_element = uniform;
  return m;
}

ParallelConfig make_config(const ref_config* c, int num_layers) {
  std::vector<int> ranks(c->ranks, c->ranks + c->nranks);
  std::vector<int> stages;
  if (c->layer_stage)
    stages.assign(c->layer_stage, c->layer_stage + num_layers);
  else
    stages = ParallelConfig::default_layer_assignment(num_layers, c->pp);
  return ParallelConfig(c->gen, c->tp, c->pp, c->dp, std::move(ranks), std::move(stages));
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Walks a view's rows; fn(global_row_start, row_len, byte_offset_in_buffer).
template <typename Fn>
void for_rows(const TensorSpec& t, const ShardView& v, int64_t bpe, Fn&& fn) {
  const size_t nd = t.shape.size();
  std::vector<int64_t> gs(nd, 1);
  for (int i = int(nd) - 2; i >= 0; --i) gs[i] = gs[i + 1] * t.shape[i + 1];
  std::vector<int64_t> p(nd);
  for (size_t i = 0; i < nd; ++i) p[i] = v.dim(i).lo;
  const int64_t row = v.dim(nd - 1).length();
  int64_t off = 0;
  while (true) {
    int64_t g = 0;
    for (size_t i = 0; i < nd; ++i) g += p[i] * gs[i];
    fn(g, row, off);
    off += row * bpe;
    int d = int(nd) - 2;
    while (d >= 0) {
      if (++p[d] < v.dim(d).hi) break;
      p[d] = v.dim(d).lo;
      --d;
    }
    if (d < 0) break;
  }
}

struct Handle {
  ModelSpec model;
  ShardStore store;
  std::vector<std::vector<std::pair<int, ShardStore::Entry*>>> entries;  // [ti] -> ascending rank
};

void index_store(Handle& h, const ParallelConfig& c) {
  h.entries.assign(h.model.tensors.size(), {});
  for (uint32_t ti = 0; ti < h.model.tensors.size(); ++ti)
    for (auto& [rank, v] : owners(h.model.tensors[ti], c))
      h.entries[ti].push_back({rank, &h.store.at(rank, ti)});
}

// Fill every entry with the reference pattern; threads split tensors.
void fast_fill(Handle& h, uint64_t seed, int nthreads) {
  auto work = [&](int tid) {
    for (uint32_t ti = tid; ti < h.entries.size(); ti += nthreads) {
      const auto& t = h.model.tensors[ti];
      const int64_t bpe = h.model.bytes_per_element;
      const uint64_t base = seed ^ (0x1000003ULL * ti);
      for (auto& [rank, e] : h.entries[ti]) {
        uint8_t* buf = e->bytes.data();
        for_rows(t, e->view, bpe, [&](int64_t g, int64_t n, int64_t off) {
          uint8_t* o = buf + off;
          for (int64_t j = 0; j < n; ++j) {
            uint64_t x = splitmix64(base ^ uint64_t(g + j));
            for (int64_t b = 0; b < bpe; ++b) *o++ = uint8_t(x >> ((b % 8) * 8));
          }
        });
      }
    }
  };
  std::vector<std::thread> ts;
  for (int i = 1; i < nthreads; ++i) ts.emplace_back(work, i);
  work(0);
  for (auto& t : ts) t.join();
}

// Count destination elements that differ from the analytic pattern.
int64_t pattern_mismatches(Handle& h, uint64_t seed, int nthreads) {
  std::vector<int64_t> bad(nthreads, 0);
  auto work = [&](int tid) {
    for (uint32_t ti = tid; ti < h.entries.size(); ti += nthreads) {
      const auto& t = h.model.tensors[ti];
      const int64_t bpe = h.model.bytes_per_element;
      const uint64_t base = seed ^ (0x1000003ULL * ti);
      for (auto& [rank, e] : h.entries[ti]) {
        const uint8_t* buf = e->bytes.data();
        for_rows(t, e->view, bpe, [&](int64_t g, int64_t n, int64_t off) {
          const uint8_t* o = buf + off;
          for (int64_t j = 0; j < n; ++j) {
            uint64_t x = splitmix64(base ^ uint64_t(g + j));
            bool ok = true;
            for (int64_t b = 0; b < bpe; ++b) ok &= o[b] == uint8_t(x >> ((b % 8) * 8));
            bad[tid] += !ok;
            o += bpe;
          }
        });
      }
    }
  };
  std::vector<std::thread> ts;
  for (int i = 1; i < nthreads; ++i) ts.emplace_back(work, i);
  work(0);
  for (auto& t : ts) t.join();
  int64_t n = 0;
  for (auto b : bad) n += b;
  return n;
}

TransferPlan reindexed(const std::string& text, const ModelSpec& m) {
  std::istringstream is(text);
  TransferPlan parsed = read_plan(is);
  // read_plan interns ids in appearance order; execute_plan indexes stores by
  // model tensor index (SURVEY §8c caveat) -- remap by name.
  std::vector<uint32_t> remap(parsed.tensor_ids.size(), 0);
  for (size_t pi = 0; pi < parsed.tensor_ids.size(); ++pi)
    for (size_t mi = 0; mi < m.tensors.size(); ++mi)
      if (m.tensors[mi].tensor_id == parsed.tensor_ids[pi]) remap[pi] = uint32_t(mi);
  TransferPlan out = parsed;
  out.tensor_ids.clear();
  for (auto& t : m.tensors) out.tensor_ids.push_back(t.tensor_id);
  for (auto& [layer, tasks] : out.tasks_by_layer)
    for (auto& t : tasks) t.tensor_index = remap[t.tensor_index];
  for (auto& [layer, keeps] : out.carryover_by_layer)
    for (auto& k : keeps) k.tensor_index = remap[k.tensor_index];
  return out;
}

void fill_report(ref_report* r, const ExecutionReport& e, double secs) {
  r->ok = e.ok;
  r->failed_layer = e.failed_layer ? *e.failed_layer : -1;
  r->peak_staging_bytes = e.peak_staging_bytes;
  r->bytes_moved = e.bytes_moved;
  r->local_copy_bytes = e.local_copy_bytes;
  r->layers_processed = e.layers_processed;
  r->seconds = secs;
  std::snprintf(r->error, sizeof r->error, "%s", e.error.c_str());
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

int ref_plan_text(const char* spec, const ref_config* o, const ref_config* n, int balance,
                  char** out, int64_t* pairs) {
  try {
    ModelSpec m = parse_spec(spec);
    PlanOptions opt;
    opt.balance_sources = balance != 0;
    PlannerStats st;
    TransferPlan p = compute_transfer_plan(make_config(o, m.num_layers),
                                           make_config(n, m.num_layers), m, opt, &st);
    std::ostringstream os;
    write_plan(os, p);
    *out = dup(os.str());
    if (pairs) *pairs = st.pairs_checked;
    return 0;
  } catch (const std::exception& e) {
    *out = dup(e.what());
    return 1;
  }
}

int ref_verify_plan(const char* spec, const ref_config* o, const ref_config* n,
                    const char* plan_text, char** out) {
  try {
    ModelSpec m = parse_spec(spec);
    std::istringstream is(plan_text);
    TransferPlan p = read_plan(is);
    auto v = verify_plan(p, make_config(o, m.num_layers), make_config(n, m.num_layers), m);
    std::string s;
    for (auto& x : v) s += x + "\n";
    *out = dup(s);
    return 0;
  } catch (const std::exception& e) {
    *out = dup(e.what());
    return 1;
  }
}

// Fill a source store with the pattern, run the reference execute_plan over a
// LoopbackTransport, return the destination store (ti-major, rank-ascending).
void* ref_execute(const char* spec, const ref_config* o, const ref_config* n,
                  const char* plan_text, uint64_t seed, int64_t staging, ref_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  rep->failed_layer = -1;
  try {
    auto* src = new Handle;
    src->model = parse_spec(spec);
    ParallelConfig co = make_config(o, src->model.num_layers);
    ParallelConfig cn = make_config(n, src->model.num_layers);
    src->store = ShardStore::allocate(src->model, co);
    index_store(*src, co);
    fast_fill(*src, seed, 1);
    auto* dst = new Handle;
    dst->model = src->model;
    dst->store = ShardStore::allocate(dst->model, cn);
    index_store(*dst, cn);
    TransferPlan plan = reindexed(plan_text, src->model);
    LoopbackTransport lb;
    auto t0 = std::chrono::steady_clock::now();
    ExecutionReport r = execute_plan(plan, src->store, dst->store, lb, staging,
                                     src->model.bytes_per_element);
    auto t1 = std::chrono::steady_clock::now();
    fill_report(rep, r, std::chrono::duration<double>(t1 - t0).count());
    delete src;
    return dst;
  } catch (const std::exception& e) {
    std::snprintf(rep->error, sizeof rep->error, "%s", e.what());
    return nullptr;
  }
}

// A pattern store for a config (the analytic expected state when built on C_new).
void* ref_store_pattern(const char* spec, const ref_config* c, uint64_t seed, int fill) {
  try {
    auto* h = new Handle;
    h->model = parse_spec(spec);
    ParallelConfig cc = make_config(c, h->model.num_layers);
    h->store = ShardStore::allocate(h->model, cc);
    index_store(*h, cc);
    if (fill) h->store.fill_pattern(h->model, seed);  // the reference's own fill
    return h;
  } catch (const std::exception&) {
    return nullptr;
  }
}

int ref_store_count(void* s, int ti) {
  auto* h = static_cast<Handle*>(s);
  return (h && ti < int(h->entries.size())) ? int(h->entries[ti].size()) : 0;
}

int ref_store_entry(void* s, int ti, int k, int* rank, uint8_t** bytes, int64_t* n) {
  auto* h = static_cast<Handle*>(s);
  if (!h || ti >= int(h->entries.size()) || k >= int(h->entries[ti].size())) return 1;
  *rank = h->entries[ti][k].first;
  *bytes = h->entries[ti][k].second->bytes.data();
  *n = int64_t(h->entries[ti][k].second->bytes.size());
  return 0;
}

void ref_store_free(void* s) { delete static_cast<Handle*>(s); }

uint8_t ref_pattern_byte(uint32_t ti, int64_t element, int64_t b, uint64_t seed) {
  return ShardStore::pattern_byte(ti, element, b, seed);
}

// The CPU arm.  ref_bench_setup plans and fills once; every ref_bench_step
// times the reference's execute_plan over the same stores.  With nthreads > 1
// the plan's layers are dealt round-robin to threads, each running the
// reference execute_plan on its layer subset with its own LoopbackTransport
// (layers touch disjoint buffers; ShardStore lookups are read-only map finds).
struct Bench {
  Handle src, dst;
  TransferPlan plan;
  int64_t plan_bytes = 0;
};

void* ref_bench_setup(const char* spec, const ref_config* o, const ref_config* n, uint64_t seed,
                      int nthreads, int64_t* plan_bytes, ref_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  rep->failed_layer = -1;
  try {
    auto* b = new Bench;
    b->src.model = parse_spec(spec);
    b->dst.model = b->src.model;
    ParallelConfig co = make_config(o, b->src.model.num_layers);
    ParallelConfig cn = make_config(n, b->src.model.num_layers);
    b->plan = compute_transfer_plan(co, cn, b->src.model);
    b->plan_bytes = b->plan.total_bytes();
    *plan_bytes = b->plan_bytes;
    b->src.store = ShardStore::allocate(b->src.model, co);
    index_store(b->src, co);
    fast_fill(b->src, seed, nthreads > 0 ? nthreads : 1);
    b->dst.store = ShardStore::allocate(b->dst.model, cn);
    index_store(b->dst, cn);
    return b;
  } catch (const std::exception& e) {
    std::snprintf(rep->error, sizeof rep->error, "%s", e.what());
    return nullptr;
  }
}

int ref_bench_step(void* h, int64_t staging, int nthreads, ref_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  rep->failed_layer = -1;
  auto* b = static_cast<Bench*>(h);
  if (nthreads < 1) nthreads = 1;
  std::vector<TransferPlan> parts(nthreads);
  std::vector<int> layers;
  for (auto& [l, t] : b->plan.tasks_by_layer) layers.push_back(l);
  for (auto& [l, c] : b->plan.carryover_by_layer)
    if (!b->plan.tasks_by_layer.count(l)) layers.push_back(l);
  int k = 0;
  for (int l : layers) {
    auto& p = parts[k++ % nthreads];
    p.tensor_ids = b->plan.tensor_ids;
    if (b->plan.tasks_by_layer.count(l)) p.tasks_by_layer[l] = b->plan.tasks_by_layer.at(l);
    if (b->plan.carryover_by_layer.count(l)) p.carryover_by_layer[l] = b->plan.carryover_by_layer.at(l);
  }
  std::vector<ExecutionReport> reps(nthreads);
  auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::thread> ts;
    for (int i = 0; i < nthreads; ++i)
      ts.emplace_back([&, i] {
        LoopbackTransport lb;
        reps[i] = execute_plan(parts[i], b->src.store, b->dst.store, lb, staging,
                               b->src.model.bytes_per_element);
      });
    for (auto& t : ts) t.join();
  }
  auto t1 = std::chrono::steady_clock::now();
  ExecutionReport all;
  all.ok = true;
  for (auto& r : reps) {
    all.ok = all.ok && r.ok;
    if (!r.ok && all.error.empty()) { all.error = r.error; all.failed_layer = r.failed_layer; }
    all.peak_staging_bytes = std::max(all.peak_staging_bytes, r.peak_staging_bytes);
    all.bytes_moved += r.bytes_moved;
    all.local_copy_bytes += r.local_copy_bytes;
    all.layers_processed += r.layers_processed;
  }
  fill_report(rep, all, std::chrono::duration<double>(t1 - t0).count());
  return all.ok ? 0 : 1;
}

int64_t ref_bench_check(void* h, uint64_t seed, int nthreads) {
  return pattern_mismatches(static_cast<Bench*>(h)->dst, seed, nthreads > 0 ? nthreads : 1);
}

void ref_bench_free(void* h) { delete static_cast<Bench*>(h); }

}  // extern "C"
