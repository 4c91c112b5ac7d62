#!/usr/bin/env python3
"""Non-persistent copy kernels on every BASELINE config (one B200, full size
or 16-layer slices): LDG8-NP vs TMA-NP (16 / 32 KB items).  Diagnostic."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    for case, layers, strict in (("c1", None, 0), ("c2", None, 0), ("c2", None, 1), ("c3", 8, 0), ("c3z", 16, 0),
                                 ("c4", 16, 0), ("c5b", 16, 0)):
        sp, co, cn = specs.sliced_case(case, layers) if layers else specs.baseline_case(case)
        plan = R.compute_transfer_plan(co, cn, sp)
        s = plan.summary()
        for ck in (15, 17, 18):
            eng = R.Engine([0], staging_bytes=1 << 30, copy_kernel=ck, strict_layers=strict)
            eng.layout(RS_SRC, sp, co)
            eng.layout(RS_DST, sp, cn)
            eng.alloc(RS_SRC)
            eng.alloc(RS_DST)
            eng.fill_pattern(RS_SRC, 42)
            eng.prepare(plan)
            eng.run()
            ms = statistics.median(eng.run()["device_ms"] for _ in range(5))
            bad = eng.verify_pattern(RS_DST, 42)[0]
            eng.close()
            print(json.dumps({"case": case, "slice": layers, "strict": strict, "copy_kernel": ck, "ms": round(ms, 4),
                              "hbm_GBps": round(2 * (s["total_bytes"] + s["carryover_bytes"]) / ms / 1e6, 1),
                              "mismatches": bad}), flush=True)


if __name__ == "__main__":
    main()
