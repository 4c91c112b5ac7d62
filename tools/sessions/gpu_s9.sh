export RS_SWEEP_STEPS=3
timeout 1200 python tools/stream_sweep.py c2 0 2:2:32:2,2:2:48:2,2:3:32:2,2:3:48:2,2:3:64:2,2:2:32:3,2:4:64:2,2:4:32:2,2:2:16:4
