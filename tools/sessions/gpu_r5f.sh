#!/bin/bash
# Round-2 session r5f: NCCL comparator with stream-ordered rounds (no host
# round trip per round): parity tests, then the C5 staging-budget sweep with
# both NCCL variants beside the ring path.
OUT=gpurun_out/r5f
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_nccl_xfer.py tests/test_capi.py -x -q -p no:cacheprovider > $OUT/pytest_xfer.txt 2>&1
echo "rc=$?" >> $OUT/pytest_xfer.txt; tail -3 $OUT/pytest_xfer.txt
timeout 1800 python tools/c5_budget_sweep.py > $OUT/c5_budget_sweep.jsonl 2> $OUT/err.txt
python - <<'PY'
import json
for l in open("gpurun_out/r5f/c5_budget_sweep.jsonl"):
    d = json.loads(l)
    print(d.get("path"), d.get("B_MiB"), d.get("device_ms") or d.get("host_ms"), d.get("rounds"), d.get("mismatches"), d.get("error"))
PY
tail -3 $OUT/err.txt
