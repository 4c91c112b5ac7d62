#!/bin/bash
# Round-2 session M: config table (every BASELINE config, DIRECT + STAGED stream lanes), C5 budget sweep
# (rings vs NCCL), the default bench (e2e host-side check) and the multi-process bench contract tests.
OUT=gpurun_out/r2m
mkdir -p $OUT
timeout 1500 python tools/config_table.py > $OUT/config_table.jsonl 2> $OUT/config_table.err; cat $OUT/config_table.jsonl
timeout 1500 python tools/c5_budget_sweep.py > $OUT/c5_budget_sweep.jsonl 2> $OUT/c5_budget_sweep.err; cat $OUT/c5_budget_sweep.jsonl
timeout 1200 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_n1.json')); print(d['ms_per_step'], d['staged']['ms_per_step'], json.dumps(d['e2e']))"
timeout 1200 python -m pytest tests/test_bench_contract.py -m gpu -q -p no:cacheprovider > $OUT/pytest_contract.txt 2>&1; tail -2 $OUT/pytest_contract.txt
