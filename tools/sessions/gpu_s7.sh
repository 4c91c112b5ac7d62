export RS_SWEEP_STEPS=3
for f in 0 64 128 256; do
  echo "== flags $f"
  RS_STREAM_FLAGS=$f RS_STREAM_PROF=1 timeout 600 python tools/stream_sweep.py c2 4 2:4:128:2,2:6:128:2 2>&1 | grep -v "^\s*$" | awk '/prof/{c++; if (c%3==1) print; next} {print}'
done
for f in 128 256; do RS_STREAM_FLAGS=$f timeout 600 python tools/stream_sweep.py c2 0 2:4:128:2,2:6:128:2; done
