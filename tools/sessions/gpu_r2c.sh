#!/bin/bash
# Round-2 session C: stream-lane descriptor prefetch (per-role frame layout) -- correctness + sweep.
OUT=gpurun_out/r2c
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -p no:cacheprovider -k "staged or ring or stream or lanes or trace or tiny" > $OUT/pytest_staged.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest_staged.txt
tail -3 $OUT/pytest_staged.txt
export RS_SWEEP_STEPS=3
RS_STREAM_PROF=1 timeout 600 python tools/stream_sweep.py c2 4 2:2:64:2,2:2:64:2:15 > $OUT/prof_slice4.txt 2>&1
grep -v "^\s*$" $OUT/prof_slice4.txt | awk '/prof/{c++; if (c%3==1 || c%3==2) print; next} {print}' | head -20
timeout 900 python tools/stream_sweep.py c2 0 2:2:64:2,2:2:64:2:15,2:1:64:2,2:1:32:2,2:3:96:2 > $OUT/sweep_full.jsonl 2>&1
cat $OUT/sweep_full.jsonl
