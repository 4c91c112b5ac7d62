#!/bin/bash
# Round-2 session r5c: STAGED fused -- the local copies issued before the lane
# kernel as a small persistent LDG grid (placed first, leaving every lane CTA
# room) vs the default (TMA-NP flood issued after the lanes).
OUT=gpurun_out/r5c
mkdir -p $OUT
for rep in 1 2; do
  for v in "0 0 0" "1 2 1" "1 2 2" "1 1 1" "1 1 2"; do
    set -- $v
    E=""; [ "$1" = 1 ] && E="RS_STREAM_LOCAL_FIRST=1"
    env $E RS_STREAM_LOCAL_VARIANT=$2 RS_STREAM_LOCAL_GRID_PER_SM=$3 RS_SWEEP_STEPS=7 timeout 600 python tools/stream_sweep.py c2 0 2:0:0:0 \
      | sed "s/^{/{\"local_first\": $1, \"local_variant\": $2, \"grid_per_sm\": $3, \"rep\": $rep, /" >> $OUT/local_first.jsonl 2>> $OUT/err.txt
  done
done
cat $OUT/local_first.jsonl | cut -c1-220; tail -3 $OUT/err.txt
RS_STREAM_LOCAL_FIRST=1 RS_STREAM_LOCAL_VARIANT=2 RS_STREAM_LOCAL_GRID_PER_SM=1 timeout 600 python tools/strict_tail.py c2 0 fused > $OUT/fused_tail_first.jsonl 2>&1
grep "lane_group\|device_ms" $OUT/fused_tail_first.jsonl | cut -c1-200
