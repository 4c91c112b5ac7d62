#!/bin/bash
# Round-2 session T: DP-broadcast pairing in the DIRECT copy kernels -- parity + C3 / C5b timing.
OUT=gpurun_out/r2t
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_executor.py tests/test_gpu_copy_variants.py tests/test_gpu_window.py tests/test_multiprocess.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt; tail -3 $OUT/pytest.txt
cat > $OUT/bcast.py <<'PY'
import json, sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import config_table as T
for case, layers in (("c3", 8), ("c5b", 16), ("c3zb", 8)):
    r = T.run(case, "direct", layers)
    r["bcast"] = os.environ.get("RS_DIRECT_BCAST", "1")
    print(json.dumps(r), flush=True)
PY
python $OUT/bcast.py > $OUT/bcast.jsonl 2>&1
RS_DIRECT_BCAST=0 python $OUT/bcast.py >> $OUT/bcast.jsonl 2>&1
cat $OUT/bcast.jsonl
