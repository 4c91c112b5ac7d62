#!/bin/bash
# One gpurun session: GPU test suite, then the default bench (N=1), outputs under gpurun_out/$1.
set -x
OUT=gpurun_out/${1:-run}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 900 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout 1200 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
tail -3 $OUT/pytest_gpu.txt
cat $OUT/bench_n1.json | head -c 3000
