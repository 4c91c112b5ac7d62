mkdir -p gpurun_out/s2
timeout 900 python -m pytest tests/test_gpu_executor.py -x -q -p no:cacheprovider -k "staged or known_answer or tiny or budget or trace or c1" > gpurun_out/s2/pytest_staged.txt 2>&1
tail -3 gpurun_out/s2/pytest_staged.txt
timeout 900 python tools/stream_sweep.py c2 0 1:6:128:2,2:6:128:2,2:8:128:2,2:4:128:2,2:6:256:2,2:6:128:3,2:13:128:2,2:10:128:2 > gpurun_out/s2/sweep.jsonl 2> gpurun_out/s2/sweep.err
cat gpurun_out/s2/sweep.jsonl; tail -3 gpurun_out/s2/sweep.err
