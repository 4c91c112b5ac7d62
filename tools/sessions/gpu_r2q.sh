#!/bin/bash
# Round-2 session Q: strict layers on the stream lanes -- parity + full C2 cost.
OUT=gpurun_out/r2q
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_executor.py tests/test_multiprocess.py -m gpu -x -q -p no:cacheprovider -k "strict or stream or ring_geometry or relay" > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt; tail -4 $OUT/pytest.txt
timeout 600 python bench.py --mode staged --strict 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_staged_strict.json 2> $OUT/err.txt
timeout 600 python bench.py --mode staged --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_staged.json 2>> $OUT/err.txt
tail -3 $OUT/err.txt
for f in $OUT/bench_staged*.json; do python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], d['ms_per_step'], d['roofline']['frac'], d['config']['strict_layers'], d['config']['copy_kernel'][:40], d['gpu_launches'], d['correct'])" $f; done
