#!/bin/bash
# Round-2 session r4r: strict STAGED with run-segmented local roles and the
# per-layer lane / local split (weight 1.5): sanitizer, parity subset, every
# config strict, full C2 strict bench line.
OUT=gpurun_out/r4r
mkdir -p $OUT
bash tools/sanitize_r2.sh r4r/san
timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_relay.py tests/test_multiprocess.py -m gpu -x -q -p no:cacheprovider \
  -k "strict or stream or relay or two_processes" > $OUT/pytest_strict.txt 2>&1; echo "rc=$?" >> $OUT/pytest_strict.txt; tail -3 $OUT/pytest_strict.txt
RS_TABLE_MODES=staged-strict timeout 1800 python tools/config_table.py > $OUT/config_table_strict.jsonl 2> $OUT/err.txt
cat $OUT/config_table_strict.jsonl | cut -c1-200
timeout 900 python bench.py --mode staged --strict 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
  > $OUT/bench_staged_strict.json 2> $OUT/bench_staged_strict.err
head -c 400 $OUT/bench_staged_strict.json
