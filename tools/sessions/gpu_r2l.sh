#!/bin/bash
# Round-2 session L: STAGED lane share vs co-resident local copies (full C2).
OUT=gpurun_out/r2l
mkdir -p $OUT
export RS_SWEEP_STEPS=3
for fr in 0.98 0.9 0.83 0.75; do
  echo "frac $fr" >> $OUT/share.jsonl
  RS_RING_CAPACITY_FRAC=$fr timeout 600 python tools/stream_sweep.py c2 0 2:2:64:2,2:2:64:2:15 >> $OUT/share.jsonl 2>&1
done
cat $OUT/share.jsonl
