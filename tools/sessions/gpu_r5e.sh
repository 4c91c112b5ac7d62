#!/bin/bash
# Round-2 session r5e: one-slot fused STAGED with lanes dealt as
# (sender, receiver) pairs by ticket and oversubscribed beyond the co-resident
# capacity (RS_RING_OVERSUB), vs the default; full C2, alternated.
OUT=gpurun_out/r5e
mkdir -p $OUT
for rep in 1 2; do
  for o in none 1 1.5 2 3; do
    E=""; [ "$o" != none ] && E="RS_RING_OVERSUB=$o"
    env $E RS_SWEEP_STEPS=7 timeout 600 python tools/stream_sweep.py c2 0 2:0:0:0 \
      | sed "s/^{/{\"oversub\": \"$o\", \"rep\": $rep, /" >> $OUT/oversub.jsonl 2>> $OUT/err.txt
  done
done
cat $OUT/oversub.jsonl | cut -c1-220; tail -3 $OUT/err.txt
RS_RING_OVERSUB=2 timeout 600 python tools/strict_tail.py c2 0 fused > $OUT/fused_tail_oversub2.jsonl 2>&1
grep "quantile\|device_ms\|lane_MB" $OUT/fused_tail_oversub2.jsonl | cut -c1-200
