#!/bin/bash
# Round-2 session U: final captures -- launch list + per-launch DRAM bytes of the default bench,
# ncu --set full of the headline TMA copy kernel and of the stream-lane kernel (C2 4-layer slice).
OUT=gpurun_out/r2u
mkdir -p $OUT
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches_c2_full.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
export RS_SWEEP_STEPS=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_stream_lane_kernel -c 1 -f -o $OUT/stream_final_c2slice4 python tools/stream_sweep.py c2 4 2:2:64:2 > $OUT/ncu_stream.log 2>&1
echo "stream rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_copy_tma_np_kernel -c 1 -f -o $OUT/tma_np_final_c2slice4 python bench.py --steps 1 --warmup 3 --profile-layers 4 --no-e2e --no-cpu-baseline --no-staged > $OUT/ncu_tma.log 2>&1
echo "tma rc=$?"
ls -la $OUT
