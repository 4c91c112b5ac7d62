#!/usr/bin/env python3
"""STAGED rings x persisting-L2 set-aside (RS_L2_PERSIST_MB) on the C5
8-layer slice, one B200: does reserving L2 for the evict-last ring slots keep
more of the staging traffic out of DRAM?  Diagnostic only."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402


def main():
    layers = int(os.environ.get("RS_SWEEP_LAYERS", "8"))
    sp, co, cn = specs.sliced_case("c5", layers)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    prop = torch.cuda.get_device_properties(0)
    print(json.dumps({"l2_bytes": prop.L2_cache_size,
                      "persisting_max": getattr(prop, "persisting_l2_cache_max_size", None)}), flush=True)
    for cap in (128, 256):
        for mb in ("auto", "0", "8", "16", "32", "64", "96"):
            if mb == "auto":
                os.environ.pop("RS_L2_PERSIST_MB", None)
            else:
                os.environ["RS_L2_PERSIST_MB"] = mb
            eng = R.Engine([0], staging_bytes=1 << 30, mode="staged", ring_slot_kib=cap)
            eng.layout(RS_SRC, sp, co)
            eng.layout(RS_DST, sp, cn)
            eng.alloc(RS_SRC)
            eng.alloc(RS_DST)
            eng.fill_pattern(RS_SRC, 42)
            eng.prepare(plan)
            eng.run()
            eng.run()
            ms = statistics.mean(eng.run()["device_ms"] for _ in range(5))
            bad = eng.verify_pattern(RS_DST, 42)[0]
            print(json.dumps({"slot_cap_KiB": cap, "persist_MB": mb, "ms": round(ms, 3),
                              "reshard_GBps": round(s["total_bytes"] / ms / 1e6, 1), "mismatches": bad}),
                  flush=True)
            eng.close()


if __name__ == "__main__":
    main()
