#!/usr/bin/env python3
"""STAGED ring geometry sweep on one B200: ring-slot cap x ring depth K x
L2 discard, on an L-layer slice of a BASELINE resize (every logical rank on
cuda:0: every cross-rank byte goes src -> ring slot -> dst).  The question is
whether the rings stay L2-resident: if they do, the staging costs no HBM
traffic and the ring path approaches the DIRECT roofline (2 bytes of HBM per
moved byte) instead of 4.  Diagnostic only; every run is pattern-checked."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    case = os.environ.get("RS_SWEEP_CASE", "c5")
    layers = int(os.environ.get("RS_SWEEP_LAYERS", "8"))
    B = int(os.environ.get("RS_SWEEP_B_MIB", "1024")) << 20
    caps = [int(c) for c in os.environ.get("RS_SWEEP_CAPS", "32,64,128,256,512,1024,-1").split(",")]
    depths = [int(k) for k in os.environ.get("RS_SWEEP_K", "2,4").split(",")]
    lanes_list = [int(x) for x in os.environ.get("RS_SWEEP_LANES", "0").split(",")]
    threads_list = [int(x) for x in os.environ.get("RS_SWEEP_THREADS", "256").split(",")]
    sp, co, cn = specs.sliced_case(case, layers)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    modes = [int(x) for x in os.environ.get("RS_SWEEP_L2MODES", "0,1,4,5").split(",")]
    for l2mode, threads in [(m, t) for m in modes for t in threads_list]:
        for lanes in lanes_list:
            for K in depths:
                for cap in caps:
                    eng = R.Engine([0], staging_bytes=B, mode="staged", slots_per_link=K, lanes_per_link=lanes,
                                   ring_slot_kib=cap, ring_discard=l2mode, ring_cta_threads=threads,
                                   spin_limit=50_000_000)
                    eng.layout(RS_SRC, sp, co)
                    eng.layout(RS_DST, sp, cn)
                    eng.alloc(RS_SRC)
                    eng.alloc(RS_DST)
                    eng.comm_alloc(plan)
                    eng.fill_pattern(RS_SRC, 42)
                    eng.fill_pattern(RS_DST, 7)
                    row = {"case": case, "layers": layers, "B_MiB": B >> 20, "l2_discard": bool(l2mode & 1), "l2_hints": bool(l2mode & 4), "warp_spec": bool(l2mode & 8),
                           "lanes": lanes, "K": K, "cta_threads": threads, "slot_cap_KiB": cap}
                    try:
                        eng.prepare(plan)
                        eng.run()
                        eng.run()
                        reps = [eng.run() for _ in range(4)]
                        bad = eng.verify_pattern(RS_DST, 42)[0]
                        ms = statistics.mean(r["device_ms"] for r in reps)
                        algo4 = 2 * (s["total_bytes"] + s["carryover_bytes"]) + 2 * s["remote_bytes"]
                        algo2 = 2 * (s["total_bytes"] + s["carryover_bytes"])
                        row.update({"ms": round(ms, 3), "reshard_GBps": round(s["total_bytes"] / ms / 1e6, 1),
                                    "hbm_GBps_4x": round(algo4 / ms / 1e6, 1),
                                    "hbm_GBps_2x": round(algo2 / ms / 1e6, 1),
                                    "peak_staging_MiB": round(reps[-1]["peak_staging_bytes"] / 2**20, 1),
                                    "mismatches": bad})
                    except Exception as e:  # noqa: BLE001
                        row["error"] = str(e)[:200]
                    print(json.dumps(row), flush=True)
                    eng.close()


if __name__ == "__main__":
    main()
