mkdir -p gpurun_out/s3
export RS_SWEEP_STEPS=3
RS_SWEEP_TRACE=1 timeout 600 python tools/stream_sweep.py c2 4 1:6:128:2,2:6:128:2,2:4:128:2 > gpurun_out/s3/trace_slice.jsonl 2>&1
RS_STREAM_LOCAL_AFTER=1 RS_SWEEP_TRACE=1 timeout 600 python tools/stream_sweep.py c2 4 2:6:128:2,2:4:128:2 > gpurun_out/s3/trace_slice_after.jsonl 2>&1
RS_STREAM_LOCAL_AFTER=1 timeout 600 python tools/stream_sweep.py c2 0 2:6:128:2,2:4:128:2 > gpurun_out/s3/full_after.jsonl 2>&1
cat gpurun_out/s3/*.jsonl
