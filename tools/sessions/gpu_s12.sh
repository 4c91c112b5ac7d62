mkdir -p gpurun_out/s12
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s12/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/s12/pytest_gpu.txt
tail -3 gpurun_out/s12/pytest_gpu.txt
export RS_SWEEP_STEPS=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_stream_lane_kernel -c 1 -f -o gpurun_out/s12/stream_c2slice4 python tools/stream_sweep.py c2 4 2:2:64:2 > gpurun_out/s12/ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:rs_exchange_kernel -c 1 -f -o gpurun_out/s12/classic_c2slice4 python tools/stream_sweep.py c2 4 1:6:128:2 >> gpurun_out/s12/ncu.log 2>&1
tail -5 gpurun_out/s12/ncu.log
