#!/usr/bin/env python3
"""STAGED strict_layers (stream lanes, layer-scoped roles) on one B200:
lane-count and capacity variants of the same full-size (or sliced) resize,
bound to one DIRECT engine's stores; device-timed, pattern-verified.

    python tools/strict_sweep.py [case] [layers|0] [max_lanes:capacity_frac,...]
(capacity_frac 0 = the engine's default share; RS_RING_MAX_LANES /
RS_RING_CAPACITY_FRAC are read at prepare)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "c2"
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["64:0"]
    steps = int(os.environ.get("RS_SWEEP_STEPS", "5"))
    sp, co, cn = specs.sliced_case(case, layers) if layers else specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    summ = plan.summary()
    base = R.Engine([0], mode="direct")
    base.layout(RS_SRC, sp, co)
    base.layout(RS_DST, sp, cn)
    base.alloc(RS_SRC)
    base.alloc(RS_DST)
    base.fill_pattern(RS_SRC, 42)
    floor_ms = 2 * (summ["total_bytes"] + summ["carryover_bytes"]) / 6552.3e9 * 1e3
    for v in variants:
        ml, frac = v.split(":")
        os.environ["RS_RING_MAX_LANES"] = ml
        if float(frac) > 0:
            os.environ["RS_RING_CAPACITY_FRAC"] = frac
        else:
            os.environ.pop("RS_RING_CAPACITY_FRAC", None)
        eng = R.Engine([0], staging_bytes=1 << 30, mode="staged", strict_layers=True)
        eng.layout(RS_SRC, sp, co)
        eng.layout(RS_DST, sp, cn)
        for which in (RS_SRC, RS_DST):
            for ti, r, n in eng.entries(which):
                eng.bind(which, r, ti, base.ptr(which, r, ti)[0], n)
        eng.comm_alloc(plan)
        eng.prepare(plan)
        base.fill_pattern(RS_DST, 7)
        for _ in range(2):
            rep = eng.run()
            assert rep["ok"], rep
        ms = []
        for _ in range(steps):
            rep = eng.run()
            assert rep["ok"], rep
            ms.append(rep["device_ms"])
        bad = base.verify_pattern(RS_DST, 42)[0]
        print(json.dumps({"case": case, "layers": layers, "variant": v, "ms": round(statistics.median(ms), 3),
                          "ms_min": round(min(ms), 3), "frac_2x_floor": round(floor_ms / statistics.median(ms), 4),
                          "peak_staging_MiB": round(rep["peak_staging_bytes"] / 2**20, 2),
                          "kernel": rep.get("ring_kernel"), "mismatches": int(bad)}), flush=True)
        eng.close()
    base.close()


if __name__ == "__main__":
    main()
