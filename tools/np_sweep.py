#!/usr/bin/env python3
"""Persistent (grid-stride, LDG8) vs non-persistent (one item per warp,
RS_COPY_LDG8_NP) copy grids x work-item size, on full C2 fused, full C2 strict
per-layer and C1.  Diagnostic; every run pattern-checked."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def run(case, strict, ck, item_kib):
    sp, co, cn = specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    eng = R.Engine([0], staging_bytes=1 << 30, strict_layers=strict, copy_kernel=ck, item_bytes=item_kib << 10)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 42)
    eng.prepare(plan)
    eng.run()
    ms = statistics.median(eng.run()["device_ms"] for _ in range(7))
    bad = eng.verify_pattern(RS_DST, 42)[0]
    eng.close()
    hbm = 2 * (s["total_bytes"] + s["carryover_bytes"]) / ms / 1e6
    return {"case": case, "strict": strict, "copy_kernel": ck, "item_KiB": item_kib, "ms": round(ms, 4),
            "hbm_GBps": round(hbm, 1), "mismatches": bad}


def main():
    for case, strict in (("c2", False), ("c2", True), ("c1", False)):
        for ck, items in ((0, (0,)), (15, (0, 8, 16, 32, 64, 128, 256))):
            for item in items:
                print(json.dumps(run(case, strict, ck, item)), flush=True)


if __name__ == "__main__":
    main()
