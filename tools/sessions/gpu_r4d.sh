#!/bin/bash
# Round-2 session r4d: strict STAGED with layer-scoped roles -- per-layer trace
# and the lane-count / capacity sweep on full C2.
OUT=gpurun_out/r4d
mkdir -p $OUT
timeout 600 python tools/strict_trace.py c2 0 > $OUT/strict_trace_scoped.jsonl 2> $OUT/strict_trace.err
head -4 $OUT/strict_trace_scoped.jsonl; sed -n 17,20p $OUT/strict_trace_scoped.jsonl; tail -1 $OUT/strict_trace_scoped.jsonl
timeout 1200 python tools/strict_sweep.py c2 0 64:0,128:0,128:0.95,32:0,24:0 > $OUT/strict_sweep.jsonl 2> $OUT/strict_sweep.err
cat $OUT/strict_sweep.jsonl; tail -3 $OUT/strict_sweep.err
