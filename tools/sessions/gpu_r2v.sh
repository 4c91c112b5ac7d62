#!/bin/bash
OUT=gpurun_out/r2v
mkdir -p $OUT
export RS_SWEEP_STEPS=5
for d in 0 4 5; do RS_SWEEP_RING_DISCARD=$d timeout 600 python tools/stream_sweep.py c2 0 2:2:64:2 | sed "s/^/discard=$d /" >> $OUT/relaxed_credit.jsonl 2>&1; done
for d in 0 4; do RS_SWEEP_RING_DISCARD=$d timeout 600 python tools/stream_sweep.py c2 0 2:2:64:2 | sed "s/^/discard=$d /" >> $OUT/relaxed_credit.jsonl 2>&1; done
cat $OUT/relaxed_credit.jsonl
