export RS_SWEEP_STEPS=3
RS_STREAM_PROF=1 timeout 600 python tools/stream_sweep.py c2 4 2:2:128:2,2:3:128:2 2>&1 | grep -v "^\s*$" | awk '/prof/{c++; if (c%3==1) print; next} {print}'
timeout 900 python tools/stream_sweep.py c2 0 2:2:128:2,2:3:128:2,2:2:64:2,2:2:128:3,2:3:64:3
RS_RING_MAX_LANES=128 timeout 900 python tools/stream_sweep.py c2 0 2:2:128:2,2:2:64:2
