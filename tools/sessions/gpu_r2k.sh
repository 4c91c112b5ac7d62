#!/bin/bash
# Round-2 session K: launch list + per-launch DRAM bytes of the default bench command
# (DIRECT headline + STAGED sub-object, full C2), ncu single pass per kernel.
OUT=gpurun_out/r2k
mkdir -p $OUT
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches_c2_full.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
echo "ncu rc=$?"
grep -c "rs_" $OUT/launches_c2_full.csv
