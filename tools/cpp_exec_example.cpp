// cpp_exec_example.cpp -- a caller written against the reference's execution
// API (proj/include/reshard/{executor,shard_store,transport,planner}.hpp, the
// shape of its executor tests and SPEC.md:514 cmd_verify), compiled against
// include/reshard/*.hpp and linked to libreshard_b200.so: the plan runs on
// the B200 engine.
//
//   ./cpp_exec_example spec.txt old.cfg new.cfg staging_bytes bpe direct|staged dst.bin
//
// A .cfg file is one line: "gen tp pp dp r0,r1,... stage0,stage1,...|-".
// Prints one JSON line (the ExecutionReport + transport counters) and writes
// the destination store as "ti:rank:" + bytes records in (tensor, rank) order
// (the golden digest format of tests/golden).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "reshard/executor.hpp"
#include "reshard/planner.hpp"
#include "reshard/shard_store.hpp"
#include "reshard/transport.hpp"

using namespace reshard;

static std::vector<int> ints(const std::string& s) {
  std::vector<int> v;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) v.push_back(std::stoi(tok));
  return v;
}

static ParallelConfig read_config(const char* path, int num_layers) {
  std::ifstream in(path);
  std::uint64_t gen;
  int tp, pp, dp;
  std::string ranks, stages;
  in >> gen >> tp >> pp >> dp >> ranks >> stages;
  return ParallelConfig(gen, tp, pp, dp, ints(ranks),
                        stages == "-" ? ParallelConfig::default_layer_assignment(num_layers, pp) : ints(stages));
}

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: %s spec old.cfg new.cfg staging_bytes bpe direct|staged dst.bin\n", argv[0]);
    return 1;
  }
  std::ifstream sin(argv[1]);
  std::stringstream text;
  text << sin.rdbuf();
  const ModelSpec model = ModelSpec::parse(text.str());
  const ParallelConfig c_old = read_config(argv[2], model.num_layers);
  const ParallelConfig c_new = read_config(argv[3], model.num_layers);
  const std::int64_t staging = std::atoll(argv[4]), bpe = std::atoll(argv[5]);

  const TransferPlan plan = compute_transfer_plan(c_old, c_new, model);
  ShardStore src = ShardStore::allocate(model, c_old);
  ShardStore dst = ShardStore::allocate(model, c_new);
  src.fill_pattern(model, 42);

  DeviceTransport device(std::string(argv[6]) == "direct" ? DeviceTransport::Mode::kDirect
                                                          : DeviceTransport::Mode::kStaged);
  RecordingTransport rec(device);
  const ExecutionReport rep = execute_plan(plan, src, dst, rec, staging, bpe);

  std::int64_t pattern_bad = 0;  // spot-check the reference pattern on the first destination shard
  for (std::uint32_t ti = 0; ti < model.tensors.size() && !pattern_bad; ++ti)
    for (int r : c_new.ranks())
      if (dst.has(r, ti) && rep.ok) {
        const auto& e = dst.at(r, ti);
        if (e.view.ndims() == 1) {  // 1-D: global element = lo + i
          for (std::int64_t i = 0; i < e.view.element_count(); ++i)
            for (std::int64_t b = 0; b < bpe; ++b)
              pattern_bad += e.bytes[static_cast<std::size_t>(i * bpe + b)] !=
                             ShardStore::pattern_byte(ti, e.view.dim(0).lo + i, b, 42);
        }
        break;
      }

  std::ofstream out(argv[7], std::ios::binary);
  for (std::uint32_t ti = 0; ti < model.tensors.size(); ++ti)
    for (int r : [&] { auto v = c_new.ranks(); std::sort(v.begin(), v.end()); return v; }())
      if (dst.has(r, ti)) {
        const std::string head = std::to_string(ti) + ":" + std::to_string(r) + ":";
        out.write(head.data(), static_cast<std::streamsize>(head.size()));
        const auto& b = dst.at(r, ti).bytes;
        out.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
      }
  std::int64_t event_bytes = 0;
  for (const auto& e : rec.events()) event_bytes += e.bytes;
  std::printf("{\"ok\": %s, \"error\": \"%s\", \"failed_layer\": %d, \"peak_staging_bytes\": %lld, "
              "\"bytes_moved\": %lld, \"local_copy_bytes\": %lld, \"layers_processed\": %d, \"events\": %zu, "
              "\"event_bytes\": %lld, \"bytes_sent\": %lld, \"pattern_bad\": %lld}\n",
              rep.ok ? "true" : "false", rep.error.c_str(), rep.failed_layer ? *rep.failed_layer : -1,
              static_cast<long long>(rep.peak_staging_bytes), static_cast<long long>(rep.bytes_moved),
              static_cast<long long>(rep.local_copy_bytes), rep.layers_processed, rec.events().size(),
              static_cast<long long>(event_bytes), static_cast<long long>(rec.bytes_sent()),
              static_cast<long long>(pattern_bad));
  return 0;
}
