#!/bin/bash
# Round-2 session r4l: deterministic lane water-filling -- multi-process
# parity (auto lanes: rings sized by rs_comm_alloc_plan before prepare),
# strict/stream subset, and the strict A/B on full C2.
OUT=gpurun_out/r4l
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_multiprocess.py -m gpu -x -q -p no:cacheprovider -k "two_processes_one_gpu" \
  > $OUT/pytest_mp.txt 2>&1; echo "rc=$?" >> $OUT/pytest_mp.txt; tail -3 $OUT/pytest_mp.txt
timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_relay.py -m gpu -x -q -p no:cacheprovider -k "strict or stream or relay" \
  > $OUT/pytest_strict.txt 2>&1; echo "rc=$?" >> $OUT/pytest_strict.txt; tail -3 $OUT/pytest_strict.txt
for rep in 1 2; do
  for g in 0 1; do
    RS_RING_NO_GROW=$g timeout 600 python tools/strict_sweep.py c2 0 128:0 \
      | sed "s/^{/{\"no_grow\": $g, \"rep\": $rep, /" >> $OUT/grow_strict.jsonl 2>> $OUT/err.txt
  done
done
for g in 0 1; do
  RS_RING_NO_GROW=$g timeout 600 python tools/strict_sweep.py c5b 16 128:0 \
    | sed "s/^{/{\"no_grow\": $g, /" >> $OUT/grow_strict.jsonl 2>> $OUT/err.txt
done
cat $OUT/grow_strict.jsonl; tail -3 $OUT/err.txt
