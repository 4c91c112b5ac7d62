#!/bin/bash
# Round-2 session r5a: why ~130 STAGED receivers start ~half-way through the
# fused lane launch -- with the local copies after the lanes (same stream)
# instead of beside them (aux stream): per-lane receiver start times (trace)
# and untraced full-C2 timings of both.
OUT=gpurun_out/r5a
mkdir -p $OUT
RS_STREAM_LOCAL_AFTER=1 timeout 600 python tools/strict_tail.py c2 0 fused > $OUT/fused_tail_local_after.jsonl 2>&1
grep lane_group $OUT/fused_tail_local_after.jsonl | cut -c1-200
for rep in 1 2; do
  for la in 0 1; do
    RS_STREAM_LOCAL_AFTER=$la RS_SWEEP_STEPS=7 timeout 600 python tools/stream_sweep.py c2 0 2:0:0:0 \
      | sed "s/^{/{\"local_after\": $la, \"rep\": $rep, /" >> $OUT/local_after.jsonl 2>> $OUT/err.txt
  done
done
cat $OUT/local_after.jsonl
