#!/usr/bin/env python3
"""STAGED (ring) transfer sweep on one B200: lanes per link x slots per link x
staging budget, on an L-layer slice of C2 (every logical rank on cuda:0, so
every cross-rank byte goes src -> ring slot -> dst).  Diagnostic only."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    sp, co, cn = specs.sliced_case("c2", layers)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    for lanes in (2, 4, 8, 16):
        for slots in (2, 4):
            for B in (256 << 20, 1 << 30):
                eng = R.Engine([0], staging_bytes=B, mode="staged", lanes_per_link=lanes, slots_per_link=slots)
                eng.layout(RS_SRC, sp, co)
                eng.layout(RS_DST, sp, cn)
                eng.alloc(RS_SRC)
                eng.alloc(RS_DST)
                eng.fill_pattern(RS_SRC, 42)
                eng.fill_pattern(RS_DST, 7)
                try:
                    eng.prepare(plan)
                    eng.run()
                    ms = [eng.run()["device_ms"] for _ in range(3)]
                    bad = eng.verify_pattern(RS_DST, 42)[0]
                    rep = eng.run()
                    mean = sum(ms) / len(ms)
                    print(json.dumps({"lanes": lanes, "slots": slots, "B_MiB": B >> 20, "mean_ms": round(mean, 3),
                                      "reshard_GBps": round(s["total_bytes"] / mean / 1e6, 1),
                                      "peak_staging": rep["peak_staging_bytes"], "mismatches": bad}), flush=True)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"lanes": lanes, "slots": slots, "B_MiB": B >> 20, "error": str(e)[:200]}),
                          flush=True)
                eng.close()


if __name__ == "__main__":
    main()
