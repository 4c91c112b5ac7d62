#!/usr/bin/env python3
"""Per-configuration roofline from the plan (SURVEY.md §8d definition).

Per GPU g (one rank per GPU, iota placement):
  out_g = remote task bytes with src g      (NVLink egress)
  in_g  = remote task bytes with dst g      (NVLink ingress)
  HBM_g = out_g + in_g + 2*local_g + 2*carry_g   (every moved byte read + written once)
  t_roof = max_g max(out_g / NVL, in_g / NVL, HBM_g / HBM)
1-GPU relayout: every logical rank on one GPU, HBM = 2*(plan bytes + carryover).
"placed_*": the same resize with the destination rank list chosen by
rs_plan_placement (placement-aware ordering over GPUs 0..7).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402

NVL = 900e9      # per direction per GPU, nominal (770 measured peer copy)
HBM = 6552.3e9   # MEASURED_PEAKS.json copy (read+write bytes)


def per_gpu(case: str, placed: bool = False):
    sp, co, cn = specs.baseline_case(case)
    if placed:
        cn, _ = R.choose_placement(co, cn, sp, candidates=list(range(8)), nvlink_gbs=NVL / 1e9,
                                   hbm_gbs=HBM / 1e9)
    plan = R.compute_transfer_plan(co, cn, sp)
    out, inn, loc, car = {}, {}, {}, {}
    for line in plan.text().splitlines():
        t = line.split()
        if t[0] == "task":
            src, dst, b = int(t[3]), int(t[4]), int(t[6])
            if src == dst:
                loc[src] = loc.get(src, 0) + b
            else:
                out[src] = out.get(src, 0) + b
                inn[dst] = inn.get(dst, 0) + b
        elif t[0] == "keep":
            car[int(t[3])] = car.get(int(t[3]), 0) + int(t[5])
    gpus = sorted(set(co.ranks) | set(cn.ranks))
    s = plan.summary()
    rows = []
    for g in gpus:
        hbm = out.get(g, 0) + inn.get(g, 0) + 2 * loc.get(g, 0) + 2 * car.get(g, 0)
        rows.append((g, out.get(g, 0), inn.get(g, 0), hbm))
    t_nvl = max(max(o, i) for _, o, i, _ in rows) / NVL
    t_hbm = max(h for *_, h in rows) / HBM
    one_gpu = 2 * (s["total_bytes"] + s["carryover_bytes"]) / HBM
    return {"case": case, "dst_ranks": cn.ranks, "gpus": len(gpus), "remote_GB": s["remote_bytes"] / 1e9,
            "local_GB": s["local_bytes"] / 1e9, "carry_GB": s["carryover_bytes"] / 1e9,
            "max_out_GB": max(r[1] for r in rows) / 1e9, "max_in_GB": max(r[2] for r in rows) / 1e9,
            "t_nvlink_ms": t_nvl * 1e3, "t_hbm_ms": t_hbm * 1e3, "roofline_ms": max(t_nvl, t_hbm) * 1e3,
            "one_gpu_hbm_roofline_ms": one_gpu * 1e3,
            "one_gpu_fits_180GB": 2 * sp.total_bytes() < 190e9}


if __name__ == "__main__":
    for c in ("c1", "c2", "c3", "c3z", "c4", "c5", "c5b"):
        for placed in (False, True):
            row = per_gpu(c, placed)
            row["placement"] = "searched" if placed else "iota"
            print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()}))
