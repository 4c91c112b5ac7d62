mkdir -p gpurun_out/s5
export RS_SWEEP_STEPS=3
RS_STREAM_PROF=1 timeout 600 python tools/stream_sweep.py c2 4 2:6:128:2,2:4:128:2 2>&1 | grep -v "^\s*$" | awk 'NR%1==0' | tail -8 > gpurun_out/s5/prof.txt
timeout 900 python tools/stream_sweep.py c2 0 1:6:128:2,2:4:128:2,2:6:128:2,2:8:128:2,2:4:256:2,2:4:128:3 > gpurun_out/s5/full.jsonl 2>&1
cat gpurun_out/s5/prof.txt gpurun_out/s5/full.jsonl
