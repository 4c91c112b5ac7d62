#!/usr/bin/env python3
"""Copy-engine work-item size x CTAs/SM on (a) the small C1 GPT-2 handoff and
(b) the full C2 handoff with strict per-layer launches (where the last items
of every layer form a tail).  Diagnostic; every run pattern-checked."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def run(case, strict, item_kib, bps):
    sp, co, cn = specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    eng = R.Engine([0], staging_bytes=1 << 30, strict_layers=strict, item_bytes=item_kib << 10,
                   blocks_per_sm=bps)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 42)
    eng.prepare(plan)
    eng.run()
    ms = statistics.mean(eng.run()["device_ms"] for _ in range(5))
    bad = eng.verify_pattern(RS_DST, 42)[0]
    eng.close()
    return {"case": case, "strict": strict, "item_KiB": item_kib, "blocks_per_sm": bps, "ms": round(ms, 4),
            "reshard_GBps": round(s["total_bytes"] / ms / 1e6, 1), "mismatches": bad}


def main():
    if os.environ.get("RS_SWEEP_FULL_C2"):
        for item in (16, 32, 64, 128, 256):
            for bps in (3, 4):
                print(json.dumps(run("c2", False, item, bps)), flush=True)
        return
    for item in (0, 16, 32, 64, 128, 256):
        for bps in (0, 2, 3, 4):
            print(json.dumps(run("c1", False, item, bps)), flush=True)
    for item in (0, 16, 32, 64, 256):
        print(json.dumps(run("c2", True, item, 0)), flush=True)


if __name__ == "__main__":
    main()
