#!/usr/bin/env python3
"""Prepare-phase planning cost (host, no GPU): our compute_transfer_plan and
exact verify_plan vs the reference's compute_transfer_plan (oracle/_ref; its
time includes write_plan serialisation) on every BASELINE resize and the
SPEC's 175B-like 96-layer / 1024-rank case (< 1 s).  The
reference's verify_plan is brute force over elements (2.4 s for GPT-2 alone,
SURVEY §6) and is not run at full size.  One JSON line per case."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402


def big175():
    ts = []
    for l in range(96):
        for name, shape, axis in (("qkv", (96, 3, 128, 12288), 0), ("o", (12288, 12288), 1),
                                  ("fc1", (49152, 12288), 0), ("fc2", (12288, 49152), 1), ("ln", (12288,), None)):
            ts.append(specs.TensorSpec(f"L{l}.{name}", l, list(shape), axis, "param", 2))
    return specs.ModelSpec("175b", 96, ts, 2), specs.iota_config(1, 8, 16, 8), specs.iota_config(2, 4, 32, 8)


def best(fn, n=3):
    ts = []
    out = None
    for _ in range(n):
        t = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t)
    return min(ts), out


def main():
    from oracle.pyoracle import Oracle, available
    ref = Oracle("ref") if available("ref") else None
    cases = [(c,) + specs.baseline_case(c) for c in ("c1", "c2", "c3", "c3z", "c4", "c5", "c5b")]
    cases.append(("175b-1024r",) + big175())
    for name, sp, co, cn in cases:
        t_plan, plan = best(lambda: R.compute_transfer_plan(co, cn, sp))
        t_ver, v = best(lambda: R.verify_plan(plan, co, cn))
        row = {"case": name, "tasks": plan.summary()["task_count"], "ours_plan_ms": round(t_plan * 1e3, 2),
               "ours_verify_ms": round(t_ver * 1e3, 2), "violations": len(v)}
        uni = sp.uniform_bpe()
        if ref is not None and not getattr(cn, "dist_opt", False):
            groups = [sp] if uni else [specs.group_spec(sp, b) for b in sorted({t.bpe for t in sp.tensors})]
            t_ref = sum(best(lambda g=g: ref.plan_text(g, co, cn))[0] for g in groups)
            row["reference_plan_ms_incl_write_plan"] = round(t_ref * 1e3, 2)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
