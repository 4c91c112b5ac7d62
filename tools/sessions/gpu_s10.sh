export RS_SWEEP_STEPS=3
for fr in 0.7 0.85 0.98; do echo "frac $fr"; RS_RING_CAPACITY_FRAC=$fr timeout 900 python tools/stream_sweep.py c2 0 2:2:64:2,2:2:96:2,2:3:96:2; done
