// cpp_api_example.cpp -- a C++ caller written against the reference's planning
// API (the way GenerationMachine::run_switch calls it, proj/src/generation.cpp:242),
// compiled against include/reshard_b200/reshard.hpp and linked to
// libreshard_b200.so instead of the reference's sources.  Plans a resize,
// checks it, prints the plan text (write_plan) and a JSON summary line.
//
//   g++ -std=c++20 -Iinclude tools/cpp_api_example.cpp -Lpaper_2605_22014_b200 \
//       -lreshard_b200 -Wl,-rpath,paper_2605_22014_b200 -o cpp_api_example
//   ./cpp_api_example spec.txt tp0 pp0 dp0 tp1 pp1 dp1 plan_out.txt
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <numeric>
#include <sstream>
#include <stdexcept>

#include "reshard_b200/reshard.hpp"

using namespace reshard;

static ParallelConfig iota(std::uint64_t gen, int tp, int pp, int dp, int num_layers) {
  std::vector<int> ranks(static_cast<std::size_t>(tp * pp * dp));
  std::iota(ranks.begin(), ranks.end(), 0);
  return ParallelConfig(gen, tp, pp, dp, ranks, ParallelConfig::default_layer_assignment(num_layers, pp));
}

int main(int argc, char** argv) {
  if (argc != 9) {
    std::fprintf(stderr, "usage: %s spec tp0 pp0 dp0 tp1 pp1 dp1 plan_out\n", argv[0]);
    return 1;
  }
  std::ifstream in(argv[1]);
  std::stringstream text;
  text << in.rdbuf();
  const ModelSpec model = ModelSpec::parse(text.str());
  const ParallelConfig c_old = iota(1, std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]), model.num_layers);
  const ParallelConfig c_new = iota(2, std::atoi(argv[5]), std::atoi(argv[6]), std::atoi(argv[7]), model.num_layers);

  // the reference's error behaviour: identical generation ids throw
  bool threw = false;
  try {
    compute_transfer_plan(c_old, c_old, model);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  // validate_config returns violations, never throws
  const ParallelConfig bad(3, 3, 1, 1, {0, 1, 1}, ParallelConfig::default_layer_assignment(model.num_layers, 1));
  const auto bad_violations = validate_config(bad, model);

  PlannerStats stats;
  const TransferPlan plan = compute_transfer_plan(c_old, c_new, model, PlanOptions{}, &stats);
  const auto violations = verify_plan(plan, c_old, c_new, model);
  const PlanCostSummary cost = plan_cost_summary(plan);
  std::ofstream out(argv[8]);
  write_plan(out, plan);
  out.close();
  // read_plan round trip
  std::ifstream back(argv[8]);
  const TransferPlan again = read_plan(back);
  // chunk_bounds of the first remote task at 1 MiB
  std::size_t chunks = 0;
  for (const auto& kv : plan.tasks_by_layer) {
    for (const auto& t : kv.second)
      if (!t.is_local()) {
        chunks = chunk_bounds(t.bounds, 1 << 20, model.element_bytes(model.tensors[t.tensor_index])).size();
        break;
      }
    if (chunks) break;
  }
  std::printf(
      "{\"identical_gen_throws\": %s, \"bad_config_violations\": %zu, \"violations\": %zu, "
      "\"total_bytes\": %lld, \"max_link_bytes\": %lld, \"task_count\": %lld, \"pairs_checked\": %lld, "
      "\"reread_task_count\": %lld, \"first_remote_task_chunks_1MiB\": %zu}\n",
      threw ? "true" : "false", bad_violations.size(), violations.size(), static_cast<long long>(cost.total_bytes),
      static_cast<long long>(cost.max_link_bytes), static_cast<long long>(cost.task_count),
      static_cast<long long>(stats.pairs_checked), static_cast<long long>(again.task_count()), chunks);
  return violations.empty() && threw && !bad_violations.empty() ? 0 : 2;
}
