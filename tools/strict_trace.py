#!/usr/bin/env python3
"""Per-layer timeline of a STAGED strict_layers handoff from the transport
trace (rs_trace_read): for each plan layer the span from its first batch
begin to its last batch end, its ring bytes and rate, and the gap to the
next layer's first batch (barrier + pipeline refill).

    python tools/strict_trace.py [case] [layers|0] [ring_kernel]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "c2"
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    kern = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    sp, co, cn = specs.sliced_case(case, layers) if layers else specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    eng = R.Engine([0], staging_bytes=1 << 30, mode="staged", strict_layers=True, trace=True, ring_kernel=kern)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 42)
    eng.prepare(plan)
    for _ in range(2):
        rep = eng.run()
        assert rep["ok"], rep
    rep = eng.run()
    tr = [r for r in eng.trace(0) if r["t_end"]]
    by = {}
    for r in tr:
        b = by.setdefault(r["layer"], {"t0": r["t_begin"], "t1": r["t_end"], "bytes": 0, "batches": 0})
        b["t0"] = min(b["t0"], r["t_begin"])
        b["t1"] = max(b["t1"], r["t_end"])
        if r["role"] == 0:
            b["bytes"] += r["bytes"]
            b["batches"] += 1
    ls = sorted(by)
    t_start = by[ls[0]]["t0"]
    for i, l in enumerate(ls):
        b = by[l]
        gap = (by[ls[i + 1]]["t0"] - b["t1"]) / 1e3 if i + 1 < len(ls) else None
        print(json.dumps({"layer": l, "start_us": round((b["t0"] - t_start) / 1e3, 1),
                          "span_us": round((b["t1"] - b["t0"]) / 1e3, 1), "ring_MB": round(b["bytes"] / 1e6, 1),
                          "GBps": round(b["bytes"] / max(1, b["t1"] - b["t0"]), 1), "batches": b["batches"],
                          "gap_to_next_us": None if gap is None else round(gap, 1)}))
    print(json.dumps({"device_ms": rep["device_ms"], "ring_kernel": rep["ring_kernel"],
                      "trace_span_ms": round((by[ls[-1]]["t1"] - t_start) / 1e6, 3)}))
    eng.close()


if __name__ == "__main__":
    main()
