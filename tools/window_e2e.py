#!/usr/bin/env python3
"""Full-size reshard of host-resident state larger than HBM through one B200
(windowed rs_execute_host).  Default: BASELINE config 3 with the distributed
optimizer (Llama-3-8B TP8 -> TP4DP2-ZeRO: 112 GB source + 128 GB destination,
240 GB > 180 GB HBM).  Host: the pinned source store (112 GB) plus a 4 GiB
pinned destination window that successive shards overwrite.  Timing only --
the source bytes are whatever the pinned pages hold; correctness of the
windowed path is covered by tests/test_gpu_window.py.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "c3z"
    window = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    sp, co, cn = specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    eng = R.Engine([0], staging_bytes=1 << 30)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    src, dst = eng.entries(RS_SRC), eng.entries(RS_DST)
    h2d, d2h = sum(n for *_, n in src), sum(n for *_, n in dst)
    host_src = R.PinnedBuffer(h2d)
    win = R.PinnedBuffer(4 << 30)
    sp_, off = [], 0
    for *_, n in src:
        sp_.append(host_src.ptr + off)
        off += n
    dp_, w = [], 0
    for *_, n in dst:
        if w + n > win.nbytes:
            w = 0
        dp_.append(win.ptr + w)
        w += n
    times = []
    for i in range(steps + 1):
        t0 = time.perf_counter()
        rep = eng.execute_host(plan, sp_, dp_, window_layers=window)
        dt = time.perf_counter() - t0
        if i:  # first call also compiles the window program
            times.append(dt)
        assert rep["ok"], rep
    mean = sum(times) / len(times)
    print(json.dumps({"workload": case, "window_layers": window, "state_src_GB": round(h2d / 1e9, 1),
                      "state_dst_GB": round(d2h / 1e9, 1), "plan_GB": round(s["total_bytes"] / 1e9, 1),
                      "s_per_step": round(mean, 3), "e2e_GBps": round(s["total_bytes"] / mean / 1e9, 2),
                      "pcie_GBps": round((h2d + d2h) / mean / 1e9, 1)}), flush=True)
    host_src.free()
    win.free()


if __name__ == "__main__":
    main()
