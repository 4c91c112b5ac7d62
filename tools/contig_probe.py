#!/usr/bin/env python3
"""Headroom probe: how fast is our copy kernel on a perfectly contiguous copy,
vs torch's copy_ (the MEASURED_PEAKS.json denominator) on the same bytes?
A one-tensor model [n] moves whole from rank 0 to rank 1 (one contiguous
task).  If the kernel matches copy_ here, the gap on the real plans comes from
their access pattern, not the kernel's issue rate.  Diagnostic only."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402
from paper_2605_22014_b200.specs import ModelSpec, ParallelConfig, TensorSpec  # noqa: E402


def main():
    for gib in (2, 8, 32):
        n = (gib << 30) // 2
        sp = ModelSpec("contig", 1, [TensorSpec("blob", 0, [n], None, "param", 2)], 2)
        co, cn = ParallelConfig(1, 1, 1, 1, [0]), ParallelConfig(2, 1, 1, 1, [1])
        plan = R.compute_transfer_plan(co, cn, sp)
        row = {"GiB": gib}
        for bps, ck in ((3, 0), (3, 17), (3, 18)):
            for item in (0,):
                eng = R.Engine([0], staging_bytes=1 << 30, blocks_per_sm=bps, copy_kernel=ck, item_bytes=item)
                eng.layout(RS_SRC, sp, co)
                eng.layout(RS_DST, sp, cn)
                eng.alloc(RS_SRC)
                eng.alloc(RS_DST)
                eng.prepare(plan)
                eng.run()
                ms = statistics.median(eng.run()["device_ms"] for _ in range(7))
                row[f"kernel{ck}_item{item >> 10}k_GBps"] = round(2 * (gib << 30) / ms / 1e6, 1)
                eng.close()
        a = torch.empty(gib << 30, dtype=torch.uint8, device="cuda")
        b = torch.empty_like(a)
        b.copy_(a)
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row["torch_copy_GBps"] = round(2 * (gib << 30) / statistics.median(ts) / 1e6, 1)
        del a, b
        torch.cuda.empty_cache()
        print(json.dumps(row), flush=True)


def c2_variants():
    from paper_2605_22014_b200 import specs
    sp, co, cn = specs.baseline_case("c2")
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    for ck in (0, 17, 18, 17, 18):
        eng = R.Engine([0], staging_bytes=1 << 30, copy_kernel=ck)
        eng.layout(RS_SRC, sp, co)
        eng.layout(RS_DST, sp, cn)
        eng.alloc(RS_SRC)
        eng.alloc(RS_DST)
        eng.fill_pattern(RS_SRC, 42)
        eng.prepare(plan)
        eng.run()
        ms = statistics.median(eng.run()["device_ms"] for _ in range(7))
        bad = eng.verify_pattern(RS_DST, 42)[0]
        print(json.dumps({"c2_copy_kernel": ck, "ms": round(ms, 3), "hbm_GBps": round(
            2 * (s["total_bytes"] + s["carryover_bytes"]) / ms / 1e6, 1), "mismatches": bad}), flush=True)
        eng.close()


if __name__ == "__main__":
    main()
    c2_variants()
