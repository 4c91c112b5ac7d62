#!/bin/bash
# Round-2 session r4j: strict STAGED with pipelined in-launch local copies
# (loads kStages ahead): parity subset, then the lane-share sweep on full C2.
OUT=gpurun_out/r4j
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -p no:cacheprovider -k "strict or stream" \
  > $OUT/pytest_strict.txt 2>&1; echo "rc=$?" >> $OUT/pytest_strict.txt; tail -3 $OUT/pytest_strict.txt
timeout 1200 python tools/strict_sweep.py c2 0 128:0,128:0.85,128:0.88,128:0.91,128:0.94 > $OUT/strict_sweep3.jsonl 2> $OUT/strict_sweep3.err
cat $OUT/strict_sweep3.jsonl; tail -3 $OUT/strict_sweep3.err
