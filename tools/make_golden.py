#!/usr/bin/env python3
"""Generate tests/golden/ from the REFERENCE itself (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile).  Run in the build container:

    make -C oracle && python tools/make_golden.py

Fixtures written (all produced by the reference's own compute_transfer_plan /
verify_plan / execute_plan / ShardStore pattern):

* ``kat.json``            -- SPEC.md known-answer cases
* ``random_pairs.json``   -- 200 random toy pairs: plan digests,
                             verify results, mutation verdicts, execution
                             reports at two staging budgets, destination digests
* ``baseline_plans.json`` -- BASELINE configs c1..c5b: plan digests and byte
                             aggregates; ``plans/<case>.txt.gz`` full plan text
* ``c1_exec.json``        -- the reference executing BASELINE config 1 in full
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle, OracleError  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.specs import (ModelSpec, ParallelConfig, TensorSpec,  # noqa: E402
                                         iota_config)

GOLD = os.path.join(ROOT, "tests", "golden")
SEED = 42


def sha(s) -> str:
    if isinstance(s, str):
        s = s.encode()
    return hashlib.sha256(s).hexdigest()


def store_digest(store) -> str:
    h = hashlib.sha256()
    for key in sorted(store.entries):
        h.update(f"{key[0]}:{key[1]}:".encode())
        h.update(store.entries[key].tobytes())
    return h.hexdigest()


def cfg_json(c: ParallelConfig) -> dict:
    return {"gen": c.gen, "tp": c.tp, "pp": c.pp, "dp": c.dp, "ranks": c.ranks,
            "layer_stage": c.layer_stage}


def plan_aggregates(text: str) -> dict:
    remote = local = carry = 0
    tasks = keeps = 0
    out, inn = {}, {}
    for line in text.splitlines():
        tok = line.split()
        if tok[0] == "task":
            tasks += 1
            b = int(tok[6])
            src, dst = int(tok[3]), int(tok[4])
            if src == dst:
                local += b
            else:
                remote += b
                out[src] = out.get(src, 0) + b
                inn[dst] = inn.get(dst, 0) + b
        elif tok[0] == "keep":
            keeps += 1
            carry += int(tok[5])
    return {"tasks": tasks, "keeps": keeps, "remote_bytes": remote, "local_bytes": local,
            "carryover_bytes": carry, "total_bytes": remote + local,
            "max_out": max(out.values(), default=0), "max_in": max(inn.values(), default=0)}


def kat_cases(ref: Oracle) -> list:
    cases = []
    W = lambda axis, bpe=2: ModelSpec("w", 1, [TensorSpec("W", 0, [1024, 1024], axis, "param", bpe)], bpe)
    # TP4 -> TP8 column-sharded W, fp16
    for name, axis in (("tp4_tp8_col", 1), ("tp4_tp8_row", 0)):
        sp = W(axis)
        co, cn = iota_config(1, 4, 1, 1), iota_config(2, 8, 1, 1)
        text, _ = ref.plan_text(sp, co, cn)
        cases.append({"name": name, "spec": sp.to_text(), "old": cfg_json(co), "new": cfg_json(cn),
                      "plan": text})
    # DP2 -> DP4, replicated
    sp = ModelSpec("rep", 1, [TensorSpec("R", 0, [64, 64], None, "param", 4)], 4)
    co, cn = iota_config(1, 1, 1, 2), iota_config(2, 1, 1, 4)
    cases.append({"name": "dp2_dp4_replicated", "spec": sp.to_text(), "old": cfg_json(co),
                  "new": cfg_json(cn), "plan": ref.plan_text(sp, co, cn)[0]})
    # identity layout
    sp = W(1)
    co, cn = iota_config(1, 4, 1, 1), iota_config(2, 4, 1, 1)
    cases.append({"name": "identity", "spec": sp.to_text(), "old": cfg_json(co),
                  "new": cfg_json(cn), "plan": ref.plan_text(sp, co, cn)[0]})
    # SPEC.md:63 + PP move: layer migrates between stages
    sp = ModelSpec("pp", 4, [TensorSpec(f"T{l}", l, [16, 8], 0, "param", 4) for l in range(4)], 4)
    co, cn = iota_config(1, 1, 2, 1), iota_config(2, 1, 2, 1, layer_stage=[0, 0, 0, 1])
    cases.append({"name": "pp_move", "spec": sp.to_text(), "old": cfg_json(co),
                  "new": cfg_json(cn), "plan": ref.plan_text(sp, co, cn)[0]})
    # error cases (messages are part of the contract)
    sp = W(1)
    for name, co, cn in (
            ("err_same_gen", iota_config(1, 4, 1, 1), iota_config(1, 8, 1, 1)),
            ("err_bad_product", ParallelConfig(1, 3, 1, 1, [0, 1]), iota_config(2, 2, 1, 1)),
            ("err_dup_rank", ParallelConfig(1, 2, 1, 1, [0, 0]), iota_config(2, 2, 1, 1)),
            ("err_axis_short", iota_config(1, 2, 1, 1), iota_config(2, 2048, 1, 1))):
        try:
            ref.plan_text(sp, co, cn)
            msg = None
        except OracleError as e:
            msg = str(e)
        cases.append({"name": name, "spec": sp.to_text(), "old": cfg_json(co), "new": cfg_json(cn),
                      "error": msg})
    return cases


def main() -> None:
    ref = Oracle("ref")
    os.makedirs(os.path.join(GOLD, "plans"), exist_ok=True)

    with open(os.path.join(GOLD, "kat.json"), "w") as f:
        json.dump(kat_cases(ref), f, indent=1)

    rows = []
    for seed, sp, co, cn in specs.iter_random_cases(200):
        row = {"seed": seed}
        text, pairs = ref.plan_text(sp, co, cn)
        row["plan_sha"] = sha(text)
        row["plan_balanced_sha"] = sha(ref.plan_text(sp, co, cn, True)[0])
        row["pairs_checked"] = pairs
        row["verify"] = ref.verify_plan(sp, co, cn, text)
        lines = text.splitlines()
        tl = [i for i, l in enumerate(lines) if l.startswith("task")]
        if tl:
            drop = "\n".join(lines[:tl[0]] + lines[tl[0] + 1:]) + "\n"
            dup = "\n".join(lines + [lines[tl[-1]]]) + "\n"
            row["verify_drop"] = ref.verify_plan(sp, co, cn, drop)
            row["verify_dup"] = ref.verify_plan(sp, co, cn, dup)
        row["exec"] = {}
        for B in (4096, 64):
            rep, store = ref.execute(sp, co, cn, text, SEED, B)
            rep.pop("seconds")
            rep["dst_sha"] = store_digest(store)
            row["exec"][str(B)] = rep
        rows.append(row)
    with open(os.path.join(GOLD, "random_pairs.json"), "w") as f:
        json.dump({"base_seed": 20260517, "fill_seed": SEED, "cases": rows}, f, indent=0)

    base = {}
    for case in ("c1", "c2", "c3", "c4", "c5", "c5b"):
        sp, co, cn = specs.baseline_case(case)
        for bpe in sorted({t.bpe for t in sp.tensors}):
            g = specs.group_spec(sp, bpe)
            text, pairs = ref.plan_text(g, co, cn)
            key = f"{case}_{bpe}B"
            base[key] = {"plan_sha": sha(text), "pairs_checked": pairs, **plan_aggregates(text)}
            with gzip.open(os.path.join(GOLD, "plans", f"{key}.txt.gz"), "wt") as f:
                f.write(text)
    with open(os.path.join(GOLD, "baseline_plans.json"), "w") as f:
        json.dump(base, f, indent=1)

    sp, co, cn = specs.baseline_case("c1")
    text, _ = ref.plan_text(sp, co, cn)
    c1 = {}
    for B in (4096, 1 << 30):
        rep, store = ref.execute(sp, co, cn, text, SEED, B)
        rep.pop("seconds")
        rep["dst_sha"] = store_digest(store)
        c1[str(B)] = rep
        del store
    with open(os.path.join(GOLD, "c1_exec.json"), "w") as f:
        json.dump(c1, f, indent=1)
    print("golden fixtures written to", GOLD)


if __name__ == "__main__":
    main()
