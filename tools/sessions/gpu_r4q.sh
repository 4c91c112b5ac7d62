#!/bin/bash
# Round-2 session r4p: strict STAGED with per-layer lane / local-copy splits
# (layer-scoped local roles): parity subset, then weight sweep vs the uniform
# local count on full C2, C5b-16, C4-16.
OUT=gpurun_out/r4q
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_relay.py -m gpu -x -q -p no:cacheprovider -k "strict or stream or relay" \
  > $OUT/pytest_strict.txt 2>&1; echo "rc=$?" >> $OUT/pytest_strict.txt; tail -3 $OUT/pytest_strict.txt
timeout 900 python -m pytest tests/test_multiprocess.py -m gpu -x -q -p no:cacheprovider -k "strict" \
  > $OUT/pytest_mp.txt 2>&1; echo "rc=$?" >> $OUT/pytest_mp.txt; tail -3 $OUT/pytest_mp.txt
for c in "c2 0" "c5b 16" "c4 16"; do
  RS_STRICT_UNIFORM_LOCAL=1 RS_STRICT_LOCAL_WEIGHT=1.5 timeout 600 python tools/strict_sweep.py $c 128:0 \
    | sed 's/^{/{"local": "uniform", /' >> $OUT/local_sweep.jsonl 2>> $OUT/err.txt
  for w in 1 1.5 2; do
    RS_STRICT_LOCAL_WEIGHT=$w timeout 600 python tools/strict_sweep.py $c 128:0 \
      | sed "s/^{/{\"local_weight\": $w, /" >> $OUT/local_sweep.jsonl 2>> $OUT/err.txt
  done
done
cat $OUT/local_sweep.jsonl; tail -3 $OUT/err.txt
