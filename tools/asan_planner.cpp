// asan_planner.cpp -- the host planner (csrc/host/*.cpp) built standalone with
// AddressSanitizer + UndefinedBehaviorSanitizer: reads
// "spec_file tp0 pp0 dp0 tp1 pp1 dp1 balance" lines from stdin, and for each
// computes the plan, verifies it, round-trips write_plan / read_plan, chunks
// every task at 4 KiB and runs the placement search.  Prints one summary
// line; any sanitizer finding aborts with a report.
#include <fstream>
#include <iostream>
#include <numeric>
#include <sstream>

#include "reshard_b200/reshard.hpp"

using namespace reshard;

static ParallelConfig iota(std::uint64_t gen, int tp, int pp, int dp, int layers) {
  std::vector<int> r(static_cast<std::size_t>(tp * pp * dp));
  std::iota(r.begin(), r.end(), 0);
  return ParallelConfig(gen, tp, pp, dp, r, ParallelConfig::default_layer_assignment(layers, pp));
}

int main() {
  std::string path;
  int tp0, pp0, dp0, tp1, pp1, dp1, bal;
  long plans = 0, tasks = 0, chunks = 0, violations = 0;
  while (std::cin >> path >> tp0 >> pp0 >> dp0 >> tp1 >> pp1 >> dp1 >> bal) {
    std::ifstream f(path);
    std::stringstream ss;
    ss << f.rdbuf();
    const ModelSpec m = ModelSpec::parse(ss.str());
    const ParallelConfig co = iota(1, tp0, pp0, dp0, m.num_layers), cn = iota(2, tp1, pp1, dp1, m.num_layers);
    if (!validate_config(co, m).empty() || !validate_config(cn, m).empty()) continue;
    PlanOptions o;
    o.balance_sources = bal != 0;
    const TransferPlan p = compute_transfer_plan(co, cn, m, o);
    violations += static_cast<long>(verify_plan(p, co, cn, m).size());
    std::stringstream text;
    write_plan(text, p);
    const TransferPlan q = read_plan(text);
    if (q.task_count() != p.task_count()) return 3;
    for (const auto& kv : p.tasks_by_layer)
      for (const auto& t : kv.second) chunks += static_cast<long>(chunk_bounds(t.bounds, 4096, m.element_bytes(m.tensors[t.tensor_index])).size());
    std::vector<int> cand(static_cast<std::size_t>(std::max(co.world_size(), cn.world_size())));
    std::iota(cand.begin(), cand.end(), 0);
    (void)choose_placement(co, cn, m, cand);
    ++plans;
    tasks += p.task_count();
  }
  std::cout << "{\"plans\": " << plans << ", \"tasks\": " << tasks << ", \"chunks\": " << chunks
            << ", \"violations\": " << violations << "}" << std::endl;
  return violations == 0 ? 0 : 2;
}
