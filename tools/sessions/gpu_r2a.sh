#!/bin/bash
# Round-2 session A: GPU suite, smoke, default bench (N=1, DIRECT + STAGED sub-object), launch list.
OUT=gpurun_out/${1:-r2a}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > $OUT/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 600 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 1200 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench rc=$?" >> $OUT/bench_n1.err
tail -3 $OUT/pytest_gpu.txt; tail -2 $OUT/smoke.txt
head -c 1500 $OUT/bench_n1.json
