#!/usr/bin/env python3
"""STAGED lane budget sweep (diagnostic): share of the device's co-resident
CTAs given to ring lanes (RS_RING_CAPACITY_FRAC) x the per-link lane cap
(RS_RING_MAX_LANES), on full C2 and a 16-layer C5b (heavy carryover)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    fracs = os.environ.get("RS_SWEEP_FRACS", "auto,0.5,0.6,0.7,0.8").split(",")
    caps = os.environ.get("RS_SWEEP_MAXLANES", "16,32").split(",")
    for case, layers in (("c2", None), ("c5b", 16)):
        sp, co, cn = specs.sliced_case(case, layers) if layers else specs.baseline_case(case)
        plan = R.compute_transfer_plan(co, cn, sp)
        eng = None
        for f in fracs:
            for ml in caps:
                if f == "auto":
                    os.environ.pop("RS_RING_CAPACITY_FRAC", None)
                else:
                    os.environ["RS_RING_CAPACITY_FRAC"] = f
                os.environ["RS_RING_MAX_LANES"] = ml
                eng = R.Engine([0], staging_bytes=1 << 30, mode="staged")
                eng.layout(RS_SRC, sp, co)
                eng.layout(RS_DST, sp, cn)
                eng.alloc(RS_SRC)
                eng.alloc(RS_DST)
                eng.fill_pattern(RS_SRC, 42)
                eng.prepare(plan)
                eng.run()
                ms = statistics.median(eng.run()["device_ms"] for _ in range(3))
                bad = eng.verify_pattern(RS_DST, 42)[0]
                print(json.dumps({"case": case, "slice": layers, "frac": f, "max_lanes": int(ml), "ms": round(ms, 3),
                                  "mismatches": bad}), flush=True)
                eng.close()


if __name__ == "__main__":
    main()
