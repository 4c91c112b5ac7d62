for d in 16 32 64; do RS_FRAME_ITEMS=$d timeout 300 python - <<PY
import sys, json, statistics, os
sys.path.insert(0, ".")
from paper_2605_22014_b200 import reshard as R, specs
from paper_2605_22014_b200.native import RS_DST, RS_SRC
for case, L in (("c2", None), ("c5", 8)):
    sp, co, cn = specs.sliced_case(case, L) if L else specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    for cap in (128, 256):
        eng = R.Engine([0], staging_bytes=1 << 30, mode="staged", ring_slot_kib=cap)
        eng.layout(RS_SRC, sp, co); eng.layout(RS_DST, sp, cn); eng.alloc(RS_SRC); eng.alloc(RS_DST)
        eng.fill_pattern(RS_SRC, 42); eng.prepare(plan); eng.run()
        ms = statistics.median(eng.run()["device_ms"] for _ in range(3))
        print(json.dumps({"items_per_slot": int(os.environ["RS_FRAME_ITEMS"]), "case": case, "cap": cap, "ms": round(ms, 3), "bad": eng.verify_pattern(RS_DST, 42)[0]}), flush=True)
        eng.close()
PY
done
