#!/usr/bin/env python3
"""Per-layer lane finish spread of a STAGED strict_layers handoff (transport
trace): for each plan layer, when each lane's receiver finished its last
batch of the layer, relative to the layer's first batch begin -- the median
and slowest lane, i.e. how much of the layer is the slowest lane's tail.

    python tools/strict_tail.py [case] [layers|0] [fused]
(fused: the default fused launch; the whole run is one "layer")
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
    fused = len(sys.argv) > 3 and sys.argv[3] == "fused"
    sp, co, cn = specs.sliced_case(case, layers) if layers else specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    eng = R.Engine([0], staging_bytes=1 << 30, mode="staged", strict_layers=not fused, trace=True)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 42)
    eng.prepare(plan)
    for _ in range(2):
        assert eng.run()["ok"]
    rep = eng.run()
    tr = [r for r in eng.trace(0) if r["t_end"]]
    by = {}
    for r in tr:
        by.setdefault(-9 if fused else r["layer"], []).append(r)
    for l in sorted(by):
        rs = by[l]
        t0 = min(r["t_begin"] for r in rs)
        rx_end = {}
        tx_first = {}
        rx_first = {}
        for r in rs:
            if r["role"] == 1:
                rx_end[r["lane"]] = max(rx_end.get(r["lane"], 0), r["t_end"])
                rx_first[r["lane"]] = min(rx_first.get(r["lane"], 1 << 62), r["t_begin"])
            else:
                tx_first[r["lane"]] = min(tx_first.get(r["lane"], 1 << 62), r["t_begin"])
        lane_bytes = {}
        for r in rs:
            if r["role"] == 0:
                lane_bytes[r["lane"]] = lane_bytes.get(r["lane"], 0) + r["bytes"]
        if fused:  # bytes per lane vs finish time: is the tail the allocation or the lanes' speed?
            pairs = sorted((rx_end[k] - t0, lane_bytes.get(k, 0)) for k in rx_end)
            for q in (0.0, 0.1, 0.5, 0.9, 1.0):
                e, b = pairs[min(len(pairs) - 1, int(q * (len(pairs) - 1)))]
                print(json.dumps({"quantile_end": q, "end_us": round(e / 1e3, 1), "lane_MB": round(b / 1e6, 1)}))
            # lanes in compile order (link by link): where do the slow ones sit?
            order = sorted(rx_end)
            nb = 16
            for i in range(nb):
                grp = order[i * len(order) // nb:(i + 1) * len(order) // nb]
                if grp:
                    es = sorted((rx_end[k] - t0) / 1e3 for k in grp)
                    rf = sorted((rx_first[k] - t0) / 1e3 for k in grp)
                    print(json.dumps({"lane_group": i, "lanes": len(grp), "first_lane_id": grp[0],
                                      "rx_first_begin_us_median": round(rf[len(rf) // 2], 1),
                                      "rx_first_begin_us_max": round(rf[-1], 1),
                                      "end_us_min": round(es[0], 1), "end_us_median": round(es[len(es) // 2], 1),
                                      "end_us_max": round(es[-1], 1)}))
            bs = sorted(lane_bytes.values())
            print(json.dumps({"lane_MB_min": round(bs[0] / 1e6, 1), "lane_MB_median": round(bs[len(bs) // 2] / 1e6, 1),
                              "lane_MB_max": round(bs[-1] / 1e6, 1)}))
        ends = sorted((e - t0) / 1e3 for e in rx_end.values())
        starts = sorted((s - t0) / 1e3 for s in tx_first.values())
        print(json.dumps({"layer": l, "lanes": len(ends), "first_start_us": round(starts[0], 1),
                          "median_start_us": round(statistics.median(starts), 1),
                          "last_start_us": round(starts[-1], 1),
                          "first_end_us": round(ends[0], 1), "median_end_us": round(statistics.median(ends), 1),
                          "p90_end_us": round(ends[int(0.9 * (len(ends) - 1))], 1), "last_end_us": round(ends[-1], 1)}))
    print(json.dumps({"device_ms": rep["device_ms"]}))
    eng.close()


if __name__ == "__main__":
    main()
