export RS_SWEEP_STEPS=1
RS_STREAM_PROF=1 timeout 600 python tools/stream_sweep.py c2 4 2:4:128:2,2:6:128:2 2>&1 | grep -v "^\s*$" | tail -8
