#!/bin/bash
# Round-2 session D: lean release/acquire in stream lanes -- correctness + sweep.
OUT=gpurun_out/${1:-r2d}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_relay.py tests/test_multiprocess.py -m gpu -x -q -p no:cacheprovider -k "staged or ring or stream or lanes or trace or tiny or relay or ipc" > $OUT/pytest_staged.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest_staged.txt
tail -3 $OUT/pytest_staged.txt
export RS_SWEEP_STEPS=3
RS_STREAM_PROF=1 timeout 600 python tools/stream_sweep.py c2 4 2:2:64:2,3:2:64:2 > $OUT/prof_slice4.txt 2>&1

grep -v "^\s*$" $OUT/prof_slice4.txt | awk '/prof/{c++; if (c<=2 || (c>6 && c<=8)) print; next} {print}' | head -20
timeout 900 python tools/stream_sweep.py c2 0 2:2:64:2,3:2:64:2,3:3:64:2,3:2:96:2,3:2:48:2,3:4:64:2 > $OUT/sweep_full.jsonl 2>&1
cat $OUT/sweep_full.jsonl
