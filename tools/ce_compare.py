#!/usr/bin/env python3
"""Copy-engine comparator: the same DIRECT handoff with the
bytes moved by the DMA copy engines (RS_COPY_CE: one cudaMemcpy2DAsync per
descriptor plane, runs uncut) instead of our copy kernel, on every BASELINE
resize that fits one B200 (16-layer slices otherwise).  CUDA-event device
time; every run pattern-checked.  One JSON line per (config, engine)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402

RS_COPY_CE = 16


def main():
    for case, layers in (("c1", None), ("c2", None), ("c3z", 16), ("c4", 16), ("c5b", 16)):
        sp, co, cn = specs.sliced_case(case, layers) if layers else specs.baseline_case(case)
        plan = R.compute_transfer_plan(co, cn, sp)
        s = plan.summary()
        for name, ck in (("kernel", 0), ("copy_engine", RS_COPY_CE)):
            eng = R.Engine([0], staging_bytes=1 << 30, copy_kernel=ck)
            eng.layout(RS_SRC, sp, co)
            eng.layout(RS_DST, sp, cn)
            eng.alloc(RS_SRC)
            eng.alloc(RS_DST)
            eng.fill_pattern(RS_SRC, 42)
            eng.fill_pattern(RS_DST, 7)
            eng.prepare(plan)
            eng.run()
            reps = [eng.run() for _ in range(3)]
            bad = eng.verify_pattern(RS_DST, 42)[0]
            ms = statistics.mean(r["device_ms"] for r in reps)
            print(json.dumps({"config": case, "slice_layers": layers, "engine": name,
                              "plan_GB": round(s["total_bytes"] / 1e9, 2), "ms": round(ms, 3),
                              "host_ms": round(statistics.mean(r["host_ms"] for r in reps), 3),
                              "reshard_GBps": round(s["total_bytes"] / ms / 1e6, 1),
                              "calls": reps[-1]["kernel_launches"], "mismatches": bad}), flush=True)
            eng.close()


if __name__ == "__main__":
    main()
