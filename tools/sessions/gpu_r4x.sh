#!/bin/bash
# Round-2 session r4x: strict STAGED local-weight sweep on the configs the
# C2/C4/C5b tuning did not cover (C1, C3-8, C3z-16, C3zb-16).
OUT=gpurun_out/r4x
mkdir -p $OUT
for c in "c1 0" "c3 8" "c3z 16" "c3zb 16"; do
  for w in 1 1.5 2.5; do
    RS_STRICT_LOCAL_WEIGHT=$w timeout 600 python tools/strict_sweep.py $c 128:0 \
      | sed "s/^{/{\"local_weight\": $w, /" >> $OUT/local_sweep2.jsonl 2>> $OUT/err.txt
  done
done
cat $OUT/local_sweep2.jsonl | cut -c1-200; tail -3 $OUT/err.txt
