#!/bin/bash
# Round-2 session r4e: strict STAGED lane-count x lane-share sweep (full C2).
OUT=gpurun_out/r4e
mkdir -p $OUT
timeout 1500 python tools/strict_sweep.py c2 0 96:0,128:0,192:0,256:0,128:0.80,192:0.80,256:0.80,192:0.90,256:0.90,256:0.75 \
  > $OUT/strict_sweep2.jsonl 2> $OUT/strict_sweep2.err
cat $OUT/strict_sweep2.jsonl; tail -3 $OUT/strict_sweep2.err
