#!/bin/bash
# Round-2 session B: relay chains across processes on one GPU + multi-process suite.
OUT=gpurun_out/r2b
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_relay.py tests/test_multiprocess.py tests/test_bench_contract.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_relay.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest_relay.txt
tail -40 $OUT/pytest_relay.txt
