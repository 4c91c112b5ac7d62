#!/usr/bin/env python3
"""BASELINE config 4 at full size on one B200: Llama-2-13B TP2PP4 -> TP4PP2
with the uneven 21/19 stage split (pipeline stage migration).

The full state (bf16 params + fp32 master / m / v: 182 GB of source, the same
again of destination) does not fit one GPU, so two legs:

* ``groups``: the full plan, all 40 layers, run on the device one state group
  at a time (bf16 params 26 GB, then fp32 master, m1, m2 at 52 GB each: source
  + destination of a group fit HBM), DIRECT and STAGED, every destination
  byte checked against the analytic pattern.  Same tasks, same boxes as the
  full plan (the plan of a group is the full plan restricted to its tensors).
* ``window``: the whole state through ``rs_execute_host`` with the layer
  window (state > HBM): host source shards H2D, layer by layer, destination
  D2H into a pinned window; source shards alias a bounded pinned buffer (the
  box has ~196 GB of RAM), so this leg is timing only -- correctness of the
  windowed path is tests/test_gpu_window.py.

    python tools/c4_full.py [groups|window|all] [steps] [case]   (case default c4; c3zb works too)
One JSON line per measurement.
"""
import dataclasses
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402

SEED = 42


def group(sp, suffix):
    ts = [dataclasses.replace(t) for t in sp.tensors if t.tensor_id.endswith("." + suffix)]
    return specs.ModelSpec(f"{sp.name}[{suffix}]", sp.num_layers, ts, ts[0].bpe)


def run_groups(steps, case="c4"):
    sp, co, cn = specs.baseline_case(case)
    for suffix in ("param", "master", "m1", "m2"):
        g = group(sp, suffix)
        plan = R.compute_transfer_plan(co, cn, g)
        s = plan.summary()
        base = R.Engine([0], mode="direct")
        base.layout(RS_SRC, g, co)
        base.layout(RS_DST, g, cn)
        base.alloc(RS_SRC)
        base.alloc(RS_DST)
        base.fill_pattern(RS_SRC, SEED)
        floor_ms = 2 * (s["total_bytes"] + s["carryover_bytes"]) / 6552.3e9 * 1e3
        for mode in ("direct", "staged"):
            eng = base if mode == "direct" else R.Engine([0], staging_bytes=1 << 30, mode="staged")
            if mode == "staged":
                eng.layout(RS_SRC, g, co)
                eng.layout(RS_DST, g, cn)
                for which in (RS_SRC, RS_DST):
                    for ti, r, n in eng.entries(which):
                        eng.bind(which, r, ti, base.ptr(which, r, ti)[0], n)
                eng.comm_alloc(plan)
            eng.prepare(plan)
            base.fill_pattern(RS_DST, SEED ^ 0xDEAD)
            ms = []
            for i in range(steps + 2):
                rep = eng.run()
                assert rep["ok"], rep
                if i >= 2:
                    ms.append(rep["device_ms"])
            bad = base.verify_pattern(RS_DST, SEED)[0]
            med = statistics.median(ms)
            print(json.dumps({"leg": "groups", "case": case, "group": suffix, "mode": mode,
                              "layers": g.num_layers, "new": f"TP{cn.tp}PP{cn.pp}DP{cn.dp}"
                              + (" stages 21/19" if case == "c4" else "") + (" flat buckets" if cn.dist_opt == 2 else ""),
                              "plan_GB": round(s["total_bytes"] / 1e9, 3),
                              "carryover_GB": round(s["carryover_bytes"] / 1e9, 3),
                              "remote_GB": round(s["remote_bytes"] / 1e9, 3), "ms": round(med, 3),
                              "GBps": round(s["total_bytes"] / med / 1e6, 1),
                              "frac_2x_floor": round(floor_ms / med, 4), "kernel_launches": rep["kernel_launches"],
                              "peak_staging_MiB": round(rep["peak_staging_bytes"] / 2**20, 2),
                              "dst_pattern_mismatches": int(bad)}), flush=True)
            if mode == "staged":
                eng.close()
        base.close()


def run_window(steps, window=2, src_cap=96 << 30, case="c4"):
    sp, co, cn = specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    eng = R.Engine([0], staging_bytes=1 << 30)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    src, dst = eng.entries(RS_SRC), eng.entries(RS_DST)
    h2d, d2h = sum(n for *_, n in src), sum(n for *_, n in dst)
    host_src = R.PinnedBuffer(min(h2d, src_cap))
    win = R.PinnedBuffer(4 << 30)
    sp_, off = [], 0
    for *_, n in src:
        if off + n > host_src.nbytes:
            off = 0
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
        assert rep["ok"], rep
        if i:  # the first call also compiles the window program
            times.append(dt)
    mean = statistics.mean(times)
    print(json.dumps({"leg": "window", "case": case, "window_layers": window,
                      "state_src_GB": round(h2d / 1e9, 1), "state_dst_GB": round(d2h / 1e9, 1),
                      "plan_GB": round(s["total_bytes"] / 1e9, 1), "s_per_step": round(mean, 3),
                      "e2e_GBps": round(s["total_bytes"] / mean / 1e9, 2),
                      "pcie_GBps": round((h2d + d2h) / mean / 1e9, 1),
                      "host_src_pinned_GB": round(host_src.nbytes / 1e9, 1)}), flush=True)
    host_src.free()
    win.free()
    eng.close()


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    case = sys.argv[3] if len(sys.argv) > 3 else "c4"
    if what in ("groups", "all"):
        run_groups(steps, case)
    if what in ("window", "all"):
        run_window(max(1, steps - 1), case=case)


if __name__ == "__main__":
    main()
