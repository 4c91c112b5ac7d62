export RS_SWEEP_STEPS=3
timeout 900 python tools/stream_sweep.py c2 0 2:1:32:2,2:1:48:2,2:1:64:2,2:1:16:2,2:2:64:2
RS_RING_MAX_LANES=128 timeout 900 python tools/stream_sweep.py c2 0 2:1:32:2,2:1:64:2
