#!/bin/bash
# Round-2 session E: ncu source-level capture of the current stream-lane kernel (C2 4-layer slice).
OUT=gpurun_out/${1:-r2e}
mkdir -p $OUT
export RS_SWEEP_STEPS=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_stream_lane_kernel -c 1 -f -o $OUT/stream_${2:-v2}_c2slice4 python tools/stream_sweep.py c2 4 2:2:64:2 > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
