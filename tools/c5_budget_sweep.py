#!/usr/bin/env python3
"""BASELINE config 5 on one B200: Llama-2-7B scale-out TP2PP2 (4) -> TP4PP2 (8),
staging-budget sweep B = 256 MiB .. 4 GiB per destination rank, our ring path
(STAGED) vs the NCCL send/recv path (RS_MODE_XFER: our pack/unpack kernels
around ncclSend/ncclRecv), plus DIRECT (zero staging) for reference.

One GPU: STAGED keeps every logical rank on cuda:0 (every cross-rank byte goes
src -> ring slot -> dst); the NCCL path gives every rank its own virtual slot
on cuda:0 (every cross-rank byte goes src -> send buffer -> NCCL -> receive
buffer -> dst).  Both move the same plan under the same budget B; every run's
destination is checked against the analytic pattern.  An L-layer slice of the
model (default 8) keeps source + destination + 2 x 8 x B of link buffers in
HBM.  One JSON line per (B, path)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs, xfer  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402

SEED = 42


def staged(sp, co, cn, plan, B, mode, steps, warmup):
    eng = R.Engine([0], staging_bytes=B, mode=mode)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    if mode == "staged":
        eng.comm_alloc(plan)
    eng.fill_pattern(RS_SRC, SEED)
    eng.fill_pattern(RS_DST, 7)
    eng.prepare(plan)
    for _ in range(warmup):
        eng.run()
    reps = [eng.run() for _ in range(steps)]
    bad = eng.verify_pattern(RS_DST, SEED)[0]
    eng.close()
    torch.cuda.empty_cache()
    return {"device_ms": statistics.mean(r["device_ms"] for r in reps),
            "host_ms": statistics.mean(r["host_ms"] for r in reps),
            "peak_staging": reps[-1]["peak_staging_bytes"], "launches": reps[-1]["kernel_launches"],
            "mismatches": bad}


def nccl_path(sp, co, cn, plan, B, nccl, steps, warmup, stream_ordered=False):
    nslots = max(max(co.ranks), max(cn.ranks)) + 1
    engs = []
    for s in range(nslots):
        e = R.Engine([0], staging_bytes=B, mode="xfer", world_slots=nslots, first_local_slot=s)
        e.layout(RS_SRC, sp, co, list(co.ranks))
        e.layout(RS_DST, sp, cn, list(cn.ranks))
        e.alloc(RS_SRC)
        e.alloc(RS_DST)
        e.fill_pattern(RS_SRC, SEED)
        e.fill_pattern(RS_DST, 7)
        engs.append(e)
    for e in engs:
        e.prepare(plan)
    for _ in range(warmup):
        xfer.run_local_slots(engs, nccl, 0, stream_ordered=stream_ordered)
    infos = [xfer.run_local_slots(engs, nccl, 0, stream_ordered=stream_ordered) for _ in range(steps)]
    bad = sum(e.verify_pattern(RS_DST, SEED)[0] for e in engs)
    for e in engs:
        e.close()
    torch.cuda.empty_cache()
    return {"host_ms": statistics.mean(i["seconds"] for i in infos) * 1e3, "rounds": infos[0]["rounds"],
            "links": infos[0]["links"], "bytes_sent": infos[0]["bytes_sent"], "mismatches": bad}


def main():
    layers = int(os.environ.get("RS_SWEEP_LAYERS", "8"))
    steps = int(os.environ.get("RS_SWEEP_STEPS", "3"))
    budgets = [int(b) << 20 for b in os.environ.get("RS_SWEEP_MIB", "256,512,1024,2048,4096").split(",")]
    sp, co, cn = specs.sliced_case("c5", layers)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    nccl = xfer.Nccl(0)
    base = {"config": f"c5 Llama-2-7B TP2PP2(4)->TP4PP2(8), {layers}-layer slice, one B200",
            "plan_GB": round(s["total_bytes"] / 1e9, 3), "remote_GB": round(s["remote_bytes"] / 1e9, 3),
            "carry_GB": round(s["carryover_bytes"] / 1e9, 3), "nccl_version": nccl.version}
    r = staged(sp, co, cn, plan, 1 << 30, "direct", steps, 2)
    print(json.dumps({**base, "path": "direct", "B_MiB": 0, **r,
                      "reshard_GBps": round(s["total_bytes"] / r["device_ms"] / 1e6, 1)}), flush=True)
    for B in budgets:
        for path in ("staged", "nccl", "nccl-stream"):
            t0 = time.time()
            try:
                if path == "staged":
                    r = staged(sp, co, cn, plan, B, "staged", steps, 2)
                    ms = r["device_ms"]
                else:  # nccl: the paper's host-driven rounds; nccl-stream: rounds ordered by events
                    r = nccl_path(sp, co, cn, plan, B, nccl, steps, 1, stream_ordered=path == "nccl-stream")
                    ms = r["host_ms"]
                print(json.dumps({**base, "path": path, "B_MiB": B >> 20, **r,
                                  "reshard_GBps": round(s["total_bytes"] / ms / 1e6, 1),
                                  "wall_s": round(time.time() - t0, 1)}), flush=True)
            except Exception as e:  # noqa: BLE001 (report and continue the sweep)
                print(json.dumps({**base, "path": path, "B_MiB": B >> 20, "error": str(e)[:300]}), flush=True)
                torch.cuda.empty_cache()
    nccl.close()


if __name__ == "__main__":
    main()
