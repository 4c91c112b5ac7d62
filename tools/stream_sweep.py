#!/usr/bin/env python3
"""STAGED lane-kernel sweep on one B200: full-size (or sliced) BASELINE
resize, one set of device stores (a DIRECT engine's) bound into STAGED
engines of every variant; device-timed handoffs, pattern-verified.

    python tools/stream_sweep.py [case] [layers|0] [variant,...]
variant = kernel:stages:slot_kib:K[:copy_kernel]  (kernel 1 classic, 2 stream;
copy_kernel = RS_COPY_* of the local copies, e.g. 15 LDG8-NP, default 0 = auto)
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
    variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1:6:128:2", "2:6:128:2"]
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
        fields = [int(x) for x in v.split(":")]
        kern, stages, slot, K = fields[:4]
        copy = fields[4] if len(fields) > 4 else 0
        eng = R.Engine([0], staging_bytes=1 << 30, mode="staged", ring_kernel=kern, ring_stages=stages,
                       ring_slot_kib=slot, slots_per_link=K, copy_kernel=copy,
                       ring_discard=int(os.environ.get("RS_SWEEP_RING_DISCARD", "0")),
                       trace=bool(os.environ.get("RS_SWEEP_TRACE")))
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
        row = {"case": case, "layers": layers, "variant": v, "ms": round(statistics.median(ms), 3),
               "ms_min": round(min(ms), 3), "frac_2x_floor": round(floor_ms / statistics.median(ms), 4),
               "peak_staging_MiB": round(rep["peak_staging_bytes"] / 2**20, 2), "launches": rep["kernel_launches"],
               "mismatches": int(bad)}
        if os.environ.get("RS_SWEEP_TRACE"):
            tr = eng.trace(0)
            for role in (0, 1):
                rs = [r for r in tr if r["role"] == role]
                if rs:
                    lanes = {r["lane"] for r in rs}
                    durs = sorted(r["t_end"] - r["t_begin"] for r in rs)
                    span = max(r["t_end"] for r in tr) - min(r["t_begin"] for r in tr)
                    row[f"role{role}"] = {"lanes": len(lanes), "batch_us_median": durs[len(durs) // 2] / 1e3,
                                          "GBps_per_lane": sum(r["bytes"] for r in rs) / len(lanes) / span}
        print(json.dumps(row), flush=True)
        eng.close()
    base.close()


if __name__ == "__main__":
    main()
