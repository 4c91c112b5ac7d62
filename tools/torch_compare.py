#!/usr/bin/env python3
"""PyTorch-eager comparator: the same handoff written the way a PyTorch
runtime would (the paper's system is Python on PyTorch): for
every task / keep of the plan, `dst_view[region].copy_(src_view[region])` on
strided torch views of the same device shard buffers (zero-copy DLPack
aliases of the engine's stores), one copy_ per box on one stream.  CUDA-event
timed; the destination is checked with the analytic pattern.  One JSON line
per config, next to our default engine on the same stores."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402
from paper_2605_22014_b200.xfer import device_bytes  # noqa: E402

SEED = 42
DT = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}


def box(text):
    return [tuple(int(x) for x in d.split(":")) for d in text.split(",")]


def main():
    for case, layers in (("c1", None), ("c2", None), ("c4", 16)):
        sp, co, cn = specs.sliced_case(case, layers) if layers else specs.baseline_case(case)
        plan = R.compute_transfer_plan(co, cn, sp)
        s = plan.summary()
        eng = R.Engine([0], staging_bytes=1 << 30)
        eng.layout(RS_SRC, sp, co)
        eng.layout(RS_DST, sp, cn)
        eng.alloc(RS_SRC)
        eng.alloc(RS_DST)
        eng.fill_pattern(RS_SRC, SEED)
        index = {t.tensor_id: i for i, t in enumerate(sp.tensors)}
        views = {}

        def view(which, cfg, rank, ti):
            key = (which, rank, ti)
            if key not in views:
                ptr, nbytes = eng.ptr(which, rank, ti)
                t = sp.tensors[ti]
                v = R.view(sp, ti, cfg, rank)
                flat = device_bytes(ptr, nbytes, 0).view(DT[t.bpe])
                views[key] = (flat.view([h - l for l, h in v]), [l for l, _ in v])
            return views[key]

        ops = []
        for line in plan.text().splitlines():
            tok = line.split()
            if tok[0] == "task":
                ti, src, dst, b = index[tok[1]], int(tok[3]), int(tok[4]), box(tok[5])
            elif tok[0] == "keep":
                ti, src, dst, b = index[tok[1]], int(tok[3]), int(tok[3]), box(tok[4])
            else:
                continue
            sv, so = view(RS_SRC, co, src, ti)
            dv, do = view(RS_DST, cn, dst, ti)
            ss = tuple(slice(lo - o, hi - o) for (lo, hi), o in zip(b, so))
            ds = tuple(slice(lo - o, hi - o) for (lo, hi), o in zip(b, do))
            ops.append((dv[ds], sv[ss]))

        def torch_step():
            for d, src in ops:
                d.copy_(src)

        def timed(fn, n=5):
            fn()
            ts = []
            for _ in range(n):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return statistics.median(ts)

        eng.fill_pattern(RS_DST, 7)
        t_torch = timed(torch_step)
        bad_torch = eng.verify_pattern(RS_DST, SEED)[0]
        eng.fill_pattern(RS_DST, 7)
        eng.prepare(plan)
        eng.run()
        t_ours = statistics.median(eng.run()["device_ms"] for _ in range(5))
        bad_ours = eng.verify_pattern(RS_DST, SEED)[0]
        print(json.dumps({"config": case, "slice_layers": layers, "copy_ops": len(ops),
                          "plan_GB": round(s["total_bytes"] / 1e9, 2),
                          "torch_eager_ms": round(t_torch, 3), "ours_ms": round(t_ours, 3),
                          "speedup": round(t_torch / t_ours, 2),
                          "torch_reshard_GBps": round(s["total_bytes"] / t_torch / 1e6, 1),
                          "ours_reshard_GBps": round(s["total_bytes"] / t_ours / 1e6, 1),
                          "mismatches": {"torch": bad_torch, "ours": bad_ours}}), flush=True)
        del ops, views
        eng.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
