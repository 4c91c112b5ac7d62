// Transfer-plan aggregates and the plan text format.
//
// Observable behaviour follows the reference (proj/src/transfer_plan.cpp):
// total_bytes counts local tasks too, per_link_bytes only cross-rank ones
// (:13-45); the text is a "plan src_gen=<g> dst_gen=<g>" header, one
// "task <tensor> <layer> <src> <dst> <lo:hi,...> <bytes>[ local]" record per
// task, then one "keep <tensor> <layer> <rank> <lo:hi,...> <bytes>" record per
// carryover region (:73-141), so golden plan files diff byte for byte.
// Reading interns tensor ids in order of first appearance (:94-101); rs_plan_read
// re-indexes them against the model by name.
//
// The implementation is this repo's own: records are built as strings with
// the shared field writers and parsed with the shared record-line reader
// (records.hpp, also behind ModelSpec::parse), dispatching on the record kind.
#include <istream>
#include <iterator>
#include <numeric>
#include <ostream>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "records.hpp"
#include "reshard_b200/reshard.hpp"

namespace reshard {

namespace {

template <class F>
void for_each_task(const TransferPlan& plan, F&& f) {
  for (const auto& [layer, tasks] : plan.tasks_by_layer)
    for (const auto& t : tasks) f(t);
}

}  // namespace

std::int64_t TransferPlan::total_bytes() const {
  std::int64_t n = 0;
  for_each_task(*this, [&](const TransferTask& t) { n += t.byte_size; });
  return n;
}

std::int64_t TransferPlan::task_count() const {
  return std::accumulate(tasks_by_layer.begin(), tasks_by_layer.end(), std::int64_t{0},
                         [](std::int64_t n, const auto& kv) { return n + static_cast<std::int64_t>(kv.second.size()); });
}

std::map<LinkKey, std::int64_t> TransferPlan::per_link_bytes() const {
  std::map<LinkKey, std::int64_t> links;
  for_each_task(*this, [&](const TransferTask& t) {
    if (t.src_rank != t.dst_rank) links[{t.src_rank, t.dst_rank}] += t.byte_size;
  });
  return links;
}

PlanCostSummary plan_cost_summary(const TransferPlan& plan) {
  PlanCostSummary s;
  s.total_bytes = plan.total_bytes();
  s.task_count = plan.task_count();
  const auto links = plan.per_link_bytes();
  for (const auto& [link, bytes] : links) s.max_link_bytes = std::max(s.max_link_bytes, bytes);
  return s;
}

// ------------------------------------------------------------------ writing

void write_plan(std::ostream& os, const TransferPlan& plan) {
  using records::put;
  std::string rec = "plan src_gen=";
  put(rec, static_cast<std::int64_t>(plan.src_config_gen));
  put(rec, " dst_gen=");
  put(rec, static_cast<std::int64_t>(plan.dst_config_gen));
  rec.push_back('\n');
  os << rec;
  for_each_task(plan, [&](const TransferTask& t) {
    rec.assign("task ");
    put(rec, plan.tensor_id(t.tensor_index));
    for (std::int64_t v : {std::int64_t{t.layer}, std::int64_t{t.src_rank}, std::int64_t{t.dst_rank}}) {
      rec.push_back(' ');
      put(rec, v);
    }
    rec.push_back(' ');
    records::put_box(rec, t.bounds);
    rec.push_back(' ');
    put(rec, t.byte_size);
    if (t.src_rank == t.dst_rank) put(rec, " local");
    rec.push_back('\n');
    os << rec;
  });
  for (const auto& [layer, keeps] : plan.carryover_by_layer)
    for (const auto& k : keeps) {
      rec.assign("keep ");
      put(rec, plan.tensor_id(k.tensor_index));
      rec.push_back(' ');
      put(rec, std::int64_t{k.layer});
      rec.push_back(' ');
      put(rec, std::int64_t{k.rank});
      rec.push_back(' ');
      records::put_box(rec, k.bounds);
      rec.push_back(' ');
      put(rec, k.byte_size);
      rec.push_back('\n');
      os << rec;
    }
}

// ------------------------------------------------------------------ reading

namespace {

using PlanLine = records::Line<std::runtime_error>;

// Accumulates a plan record by record.
class PlanReader {
 public:
  void record(PlanLine& in) {
    const std::string_view kind = in.kind();
    if (kind == "plan") header(in);
    else if (kind == "task") task(in);
    else if (kind == "keep") keep(in);
    else in.fail("unknown record '" + std::string(kind) + "'");
  }
  TransferPlan take() { return std::move(plan_); }

 private:
  // tensor ids get indices in order of first appearance
  std::uint32_t tensor(std::string_view id) {
    auto [it, fresh] = ids_.try_emplace(std::string(id), static_cast<std::uint32_t>(plan_.tensor_ids.size()));
    if (fresh) plan_.tensor_ids.emplace_back(id);
    return it->second;
  }
  // "plan key=value ..." -- src_gen / dst_gen; other fields are ignored
  void header(PlanLine& in) {
    while (auto f = in.maybe_word()) {
      const auto eq = f->find('=');
      if (eq == std::string_view::npos) continue;
      const std::string_view key = f->substr(0, eq), val = f->substr(eq + 1);
      std::uint64_t* gen = key == "src_gen" ? &plan_.src_config_gen : key == "dst_gen" ? &plan_.dst_config_gen : nullptr;
      if (!gen) continue;
      const auto [end, ec] = std::from_chars(val.data(), val.data() + val.size(), *gen);
      if (ec != std::errc() || end != val.data() + val.size()) in.fail("bad generation '" + std::string(*f) + "'");
    }
  }
  void task(PlanLine& in) {
    TransferTask t;
    t.tensor_index = tensor(in.word("tensor id"));
    t.layer = in.number<int>("layer");
    t.src_rank = in.number<int>("source rank");
    t.dst_rank = in.number<int>("destination rank");
    t.bounds = in.box("bounds");
    t.byte_size = in.number<std::int64_t>("byte size");
    (void)in.maybe_word();  // optional "local": locality is src == dst
    plan_.tasks_by_layer[t.layer].push_back(t);
  }
  void keep(PlanLine& in) {
    CarryoverRegion k;
    k.tensor_index = tensor(in.word("tensor id"));
    k.layer = in.number<int>("layer");
    k.rank = in.number<int>("rank");
    k.bounds = in.box("bounds");
    k.byte_size = in.number<std::int64_t>("byte size");
    plan_.carryover_by_layer[k.layer].push_back(k);
  }

  TransferPlan plan_;
  std::unordered_map<std::string, std::uint32_t> ids_;
};

}  // namespace

TransferPlan read_plan(std::istream& is) {
  const std::string text{std::istreambuf_iterator<char>(is), std::istreambuf_iterator<char>()};
  PlanReader reader;
  records::for_each_line(text, false, [&](std::string_view line, int lineno) {
    PlanLine in(line, "plan parse", lineno);
    if (!in.blank()) reader.record(in);
  });
  return reader.take();
}

}  // namespace reshard
