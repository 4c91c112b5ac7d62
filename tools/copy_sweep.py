#!/usr/bin/env python3
"""Copy-engine variant sweep on the full C2 workload (one B200).

Each variant: fresh engine + stores, fill, 2 warm-up runs, 5 timed runs
(CUDA events inside rs_run), then the analytic-pattern check of the
destination.  Prints one JSON line per variant.  Not a bench number.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402

VARIANTS = [dict(name="ldg4_auto", copy_kernel=1)]
for ck, cname in ((1, "ldg4"), (2, "ldg8"), (4, "ldg4cs"), (5, "ldg8cs")):
    for bps in (2, 3, 4):
        for item in (0, 256 << 10):
            VARIANTS.append(dict(name=f"{cname}_bps{bps}_item{item >> 10}k", copy_kernel=ck,
                                 blocks_per_sm=bps, item_bytes=item))


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    if layers:
        sp, co, cn = specs.sliced_case("c2", layers)
    else:
        sp, co, cn = specs.baseline_case("c2")
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    algo = 2 * (s["total_bytes"] + s["carryover_bytes"])
    for v in VARIANTS:
        if only and v["name"] not in only:
            continue
        kw = {k: x for k, x in v.items() if k != "name"}
        eng = R.Engine([0], staging_bytes=1 << 30, **kw)
        eng.layout(RS_SRC, sp, co)
        eng.layout(RS_DST, sp, cn)
        eng.alloc(RS_SRC)
        eng.alloc(RS_DST)
        eng.fill_pattern(RS_SRC, 42)
        eng.fill_pattern(RS_DST, 7)
        eng.prepare(plan)
        for _ in range(2):
            eng.run()
        ms = [eng.run()["device_ms"] for _ in range(5)]
        bad = eng.verify_pattern(RS_DST, 42)[0]
        best, mean = min(ms), sum(ms) / len(ms)
        print(json.dumps({"variant": v["name"], "mean_ms": round(mean, 3), "best_ms": round(best, 3),
                          "reshard_GBps": round(s["total_bytes"] / mean / 1e6, 1),
                          "hbm_GBps": round(algo / mean / 1e6, 1), "mismatches": bad}), flush=True)
        eng.close()


if __name__ == "__main__":
    main()
