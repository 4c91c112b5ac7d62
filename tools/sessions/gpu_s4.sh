mkdir -p gpurun_out/s4
export RS_SWEEP_STEPS=2
for f in 0 64; do
  echo "== flags $f"
  RS_STREAM_FLAGS=$f RS_STREAM_PROF=1 timeout 600 python tools/stream_sweep.py c2 4 2:6:128:2,2:4:128:2 2>&1 | grep -v "^\s*$" | tail -12
done > gpurun_out/s4/prof.txt 2>&1
RS_STREAM_FLAGS=64 timeout 600 python tools/stream_sweep.py c2 0 2:6:128:2,2:4:128:2,2:8:128:2 > gpurun_out/s4/full_regstore.jsonl 2>&1
cat gpurun_out/s4/prof.txt gpurun_out/s4/full_regstore.jsonl
