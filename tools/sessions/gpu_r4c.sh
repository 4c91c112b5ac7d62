#!/bin/bash
# Round-2 session r4c: STAGED strict layers with layer-scoped lane roles
# (lanes of links that never share a layer reuse the same CTA slots):
# parity tests for strict / stream lanes / relay / multi-process, then full C2
# strict STAGED timed.
OUT=gpurun_out/r4c
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -p no:cacheprovider -k "strict or stream" \
  > $OUT/pytest_strict.txt 2>&1; echo "rc=$?" >> $OUT/pytest_strict.txt
timeout 1200 python -m pytest tests/test_relay.py tests/test_multiprocess.py -m gpu -x -q -p no:cacheprovider \
  > $OUT/pytest_mp.txt 2>&1; echo "rc=$?" >> $OUT/pytest_mp.txt
tail -3 $OUT/pytest_strict.txt $OUT/pytest_mp.txt
timeout 900 python bench.py --mode staged --strict 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
  > $OUT/bench_staged_strict.json 2> $OUT/bench_staged_strict.err
head -c 1500 $OUT/bench_staged_strict.json; tail -5 $OUT/bench_staged_strict.err
