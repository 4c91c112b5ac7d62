#!/bin/bash
# Round-2 session r5b: STAGED fused -- the aux-stream local copies as a small
# persistent LDG8 grid (registers only, no shared memory) so every lane CTA
# stays resident, vs the default TMA-NP flood.
OUT=gpurun_out/r5b
mkdir -p $OUT
for rep in 1 2; do
  for v in "0 0" "2 1" "2 2" "1 1"; do
    set -- $v
    RS_STREAM_LOCAL_VARIANT=$1 RS_STREAM_LOCAL_GRID_PER_SM=$2 RS_SWEEP_STEPS=7 timeout 600 python tools/stream_sweep.py c2 0 2:0:0:0 \
      | sed "s/^{/{\"local_variant\": $1, \"grid_per_sm\": $2, \"rep\": $rep, /" >> $OUT/local_variant.jsonl 2>> $OUT/err.txt
  done
done
cat $OUT/local_variant.jsonl | cut -c1-200; tail -3 $OUT/err.txt
RS_STREAM_LOCAL_VARIANT=2 RS_STREAM_LOCAL_GRID_PER_SM=1 timeout 600 python tools/strict_tail.py c2 0 fused > $OUT/fused_tail_ldg.jsonl 2>&1
grep "lane_group\|device_ms" $OUT/fused_tail_ldg.jsonl | cut -c1-200
