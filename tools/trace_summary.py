#!/usr/bin/env python3
"""Where does a STAGED handoff spend its time?  Runs an L-layer slice of C2
with the transport trace on and summarises it: per-role batch service time
(flag acquired -> flag published), per-lane busy fraction of the kernel span,
and the gap a receiver waits after its sender published.  Diagnostic."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    layers = int(os.environ.get("RS_TRACE_LAYERS", "4"))
    sp, co, cn = specs.sliced_case("c2", layers)
    plan = R.compute_transfer_plan(co, cn, sp)
    fracs = os.environ.get("RS_TRACE_FRACS")
    for cap in (64, 128, 256) if not fracs else (128,):
      for frac in ([float(f) for f in fracs.split(",")] if fracs else [None]):
        if frac is not None:
            os.environ["RS_RING_CAPACITY_FRAC"] = str(frac)
        if os.environ.get("RS_TRACE_MAX_LANES"):
            os.environ["RS_RING_MAX_LANES"] = os.environ["RS_TRACE_MAX_LANES"]
        eng = R.Engine([0], staging_bytes=1 << 30, mode="staged", ring_slot_kib=cap, trace=True)
        eng_frac = frac
        eng.layout(RS_SRC, sp, co)
        eng.layout(RS_DST, sp, cn)
        eng.alloc(RS_SRC)
        eng.alloc(RS_DST)
        eng.fill_pattern(RS_SRC, 42)
        eng.prepare(plan)
        eng.run()
        rep = eng.run()
        tr = eng.trace(0)
        t0 = min(r["t_begin"] for r in tr)
        t1 = max(r["t_end"] for r in tr)
        span = t1 - t0
        out = {"slot_KiB": cap, "lane_capacity_frac": eng_frac, "max_lanes": os.environ.get("RS_RING_MAX_LANES"), "device_ms": round(rep["device_ms"], 3), "trace_span_ms": round(span / 1e6, 3),
               "batches": len(tr) // 2}
        for role, name in ((0, "sender"), (1, "receiver")):
            rr = [r for r in tr if r["role"] == role]
            svc = [r["t_end"] - r["t_begin"] for r in rr]
            lanes = {}
            for r in rr:
                lanes.setdefault(r["lane"], []).append(r)
            busy = [sum(x["t_end"] - x["t_begin"] for x in v) / span for v in lanes.values()]
            out[name] = {"lanes": len(lanes), "batch_us_median": round(statistics.median(svc) / 1e3, 2),
                         "batch_us_p90": round(sorted(svc)[int(0.9 * len(svc))] / 1e3, 2),
                         "busy_frac_median": round(statistics.median(busy), 3),
                         "GBps_per_lane": round(statistics.median(
                             [sum(x["bytes"] for x in v) / (span / 1e9) / 1e9 for v in lanes.values()]), 2)}
        tx = {(r["lane"], r["batch"]): r for r in tr if r["role"] == 0}
        waits = [r["t_begin"] - tx[(r["lane"], r["batch"])]["t_end"] for r in tr if r["role"] == 1]
        out["rx_start_after_tx_publish_us_median"] = round(statistics.median(waits) / 1e3, 2)
        print(json.dumps(out), flush=True)
        eng.close()


if __name__ == "__main__":
    main()
