#!/bin/bash
# Round-2 session r4f: strict STAGED (layer-scoped roles, tuned lane share) on
# every BASELINE config; parity subset; full C2 strict bench line.
OUT=gpurun_out/r4f
mkdir -p $OUT
for c in "c1 0" "c2 0" "c3 16" "c3zb 16" "c4 16" "c5 0" "c5b 16"; do
  timeout 900 python tools/strict_sweep.py $c 128:0 >> $OUT/strict_configs.jsonl 2>> $OUT/strict_configs.err
done
cat $OUT/strict_configs.jsonl; tail -3 $OUT/strict_configs.err
timeout 1500 python -m pytest tests/test_gpu_executor.py tests/test_relay.py -m gpu -x -q -p no:cacheprovider -k "strict or stream or relay" \
  > $OUT/pytest_strict.txt 2>&1; echo "rc=$?" >> $OUT/pytest_strict.txt; tail -3 $OUT/pytest_strict.txt
timeout 900 python bench.py --mode staged --strict 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
  > $OUT/bench_staged_strict.json 2> $OUT/bench_staged_strict.err
head -c 700 $OUT/bench_staged_strict.json
