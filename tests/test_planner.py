"""Product host planner (libreshard_b200.so, C++) vs the reference.

CPU only: planning is host code; no CUDA call is made here.
"""

import gzip
import os
import time

import pytest

from helpers import cfg_from_json, sha, spec_from_text
from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_kat(golden):
    for case in golden["kat"]:
        sp = spec_from_text(case["spec"])
        co, cn = cfg_from_json(case["old"]), cfg_from_json(case["new"])
        if case.get("error") is not None:
            with pytest.raises(ValueError) as e:
                R.compute_transfer_plan(co, cn, sp)
            assert str(e.value) == case["error"], case["name"]
        else:
            assert R.compute_transfer_plan(co, cn, sp).text() == case["plan"], case["name"]


def test_identity_is_all_carryover():
    sp = specs.ModelSpec("w", 1, [specs.TensorSpec("W", 0, [64, 64], 1, "param", 2)], 2)
    p = R.compute_transfer_plan(specs.iota_config(1, 4, 1, 1), specs.iota_config(2, 4, 1, 1), sp)
    s = p.summary()
    assert s["task_count"] == 0 and s["carryover_count"] == 4 and s["total_bytes"] == 0


def test_random_pairs(golden):
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    for seed, sp, co, cn in specs.iter_random_cases(200, golden["random_pairs"]["base_seed"]):
        row = rows[seed]
        stats = R.PlannerStats()
        plan = R.compute_transfer_plan(co, cn, sp, stats=stats)
        text = plan.text()
        assert sha(text) == row["plan_sha"], seed
        assert stats.pairs_checked == row["pairs_checked"]
        assert sha(R.compute_transfer_plan(co, cn, sp, R.PlanOptions(True)).text()) == row["plan_balanced_sha"]
        assert R.verify_plan(plan, co, cn) == row["verify"]
        lines = text.splitlines()
        tl = [i for i, l in enumerate(lines) if l.startswith("task")]
        if tl:
            drop = "\n".join(lines[:tl[0]] + lines[tl[0] + 1:]) + "\n"
            dup = "\n".join(lines + [lines[tl[-1]]]) + "\n"
            assert R.verify_plan(R.read_plan(drop, sp), co, cn) == row["verify_drop"]
            assert R.verify_plan(R.read_plan(dup, sp), co, cn) == row["verify_dup"]
        # write/read round trip (SPEC.md cli invariant)
        assert R.read_plan(text, sp).text() == text


def test_baseline_plans(golden):
    for case in ("c1", "c2", "c3", "c4", "c5", "c5b"):
        sp, co, cn = specs.baseline_case(case)
        for bpe in sorted({t.bpe for t in sp.tensors}):
            key = f"{case}_{bpe}B"
            plan = R.compute_transfer_plan(co, cn, specs.group_spec(sp, bpe))
            assert sha(plan.text()) == golden["baseline_plans"][key]["plan_sha"], key
        # the mixed-dtype plan is the union of the group plans (per-tensor bytes)
        mixed = R.compute_transfer_plan(co, cn, sp)
        groups = sum(golden["baseline_plans"][f"{case}_{b}B"]["total_bytes"]
                     for b in sorted({t.bpe for t in sp.tensors}))
        assert mixed.total_bytes() == groups
        assert R.verify_plan(mixed, co, cn) == []


def test_mixed_plan_matches_oracle(oracle_c):
    for case in ("c1", "c2", "c4"):
        sp, co, cn = specs.baseline_case(case)
        assert R.compute_transfer_plan(co, cn, sp).text() == oracle_c.plan_text(sp, co, cn)[0]


def test_verify_detects_escape_and_unknown():
    sp = specs.ModelSpec("w", 1, [specs.TensorSpec("W", 0, [8, 8], 0, "param", 4)], 4)
    co, cn = specs.iota_config(1, 2, 1, 1), specs.iota_config(2, 1, 1, 1)
    bad = "plan src_gen=1 dst_gen=2\ntask W 0 1 0 0:8,0:8 256\n"
    v = R.verify_plan(R.read_plan(bad, sp), co, cn)
    assert any("escape source view" in x for x in v)
    with pytest.raises(ValueError, match="unknown tensor"):
        R.read_plan("plan src_gen=1 dst_gen=2\ntask X 0 1 0 0:8,0:8 256\n", sp)


def test_chunk_bounds_matches_oracle(oracle_c):
    cases = [([0, 0, 0], [10, 7, 3], 50, 2), ([3, 0], [17, 9], 40, 4), ([0, 0, 0], [2, 5, 64], 100, 1),
             ([0], [1000], 64, 8), ([1, 1, 1], [2, 2, 9], 4, 1)]
    for lo, hi, mx, bpe in cases:
        assert R.chunk_bounds(lo, hi, mx, bpe) == oracle_c.chunk_bounds(lo, hi, mx, bpe)
    with pytest.raises(ValueError, match="one element exceeds the staging budget"):
        R.chunk_bounds([0], [4], 1, 2)


def test_validate_config_messages():
    sp = specs.gpt2_124m(4)
    bad = specs.ParallelConfig(1, 3, 2, 1, [0, 1, 2, 3])
    assert R.validate_config(bad, sp)[0] == "tp*pp*dp = 6 != world size 4"
    dup = specs.ParallelConfig(1, 2, 1, 1, [5, 5])
    assert "duplicate rank id 5" in R.validate_config(dup, sp)
    gap = specs.ParallelConfig(1, 1, 2, 1, [0, 1], [0, 0, 0, 0])
    assert "pipeline stage 1 receives no layers" in R.validate_config(gap, sp)


def test_view_known_answers():
    sp = specs.ModelSpec("w", 6, [specs.TensorSpec("W", 0, [1024, 1024], 1, "param", 2),
                                  specs.TensorSpec("X", 5, [16], None, "param", 2)], 2)
    assert R.view(sp, 0, specs.iota_config(1, 4, 1, 1), 0) == [(0, 1024), (0, 256)]
    assert R.view(sp, 0, specs.iota_config(1, 1, 1, 1), 0) == [(0, 1024), (0, 1024)]
    pp = specs.iota_config(1, 1, 2, 1, layer_stage=[0, 0, 0, 0, 1, 1])
    assert R.view(sp, 1, pp, 0) is None


def test_planner_scalability():
    """96 layers, 1024 ranks, metadata only, < 1 s; pairs linear in ranks."""
    L = 96
    ts = []
    for l in range(L):
        for name, shape, axis in (("qkv", (96, 3, 128, 12288), 0), ("o", (12288, 12288), 1),
                                  ("fc1", (49152, 12288), 0), ("fc2", (12288, 49152), 1),
                                  ("ln", (12288,), None)):
            ts.append(specs.TensorSpec(f"L{l}.{name}", l, list(shape), axis, "param", 2))
    sp = specs.ModelSpec("175b", L, ts, 2)
    co = specs.iota_config(1, 8, 16, 8)    # 1024 ranks
    cn = specs.iota_config(2, 4, 32, 8)    # 1024 ranks
    t0 = time.perf_counter()
    stats = R.PlannerStats()
    plan = R.compute_transfer_plan(co, cn, sp, stats=stats)
    dt = time.perf_counter() - t0
    assert dt < 1.0, dt
    half = R.PlannerStats()
    R.compute_transfer_plan(specs.iota_config(1, 8, 16, 4), specs.iota_config(2, 4, 32, 4), sp, stats=half)
    assert stats.pairs_checked <= 2.2 * half.pairs_checked
    assert plan.summary()["task_count"] > 0


def test_distributed_optimizer_extension_matches_oracle(oracle_c):
    """ZeRO-1 re-partition (BASELINE config 3; no reference counterpart, so the
    C restatement carries the same extension): plans identical, exact cover."""
    for seed, sp, co, cn in specs.iter_random_zero_cases(300):
        for bal in (False, True):
            plan = R.compute_transfer_plan(co, cn, sp, R.PlanOptions(bal))
            assert plan.text() == oracle_c.plan_text(sp, co, cn, bal)[0], (seed, bal)
        assert R.verify_plan(plan, co, cn) == [], seed


def test_c3_distributed_optimizer_plan(oracle_c):
    sp, co, cn = specs.baseline_case("c3z")
    plan = R.compute_transfer_plan(co, cn, sp)
    assert plan.text() == oracle_c.plan_text(sp, co, cn)[0]
    assert R.verify_plan(plan, co, cn) == []
    # the dp-sharded fp32 state halves what the replicated-DP plan moves
    rep = R.compute_transfer_plan(*specs.baseline_case("c3")[1:], specs.baseline_case("c3")[0])
    assert plan.total_bytes() < 0.55 * rep.total_bytes()
    # each DP rank of the new config holds half of every sharded fp32 tensor
    ti = next(i for i, t in enumerate(sp.tensors) if t.tensor_id == "L0.embed.master")
    v0, v1 = R.view(sp, ti, cn, 0), R.view(sp, ti, cn, 4)
    assert v0 and v1 and v0 != v1


def test_plan_text_rejects_malformed_records():
    """read_plan parses every field strictly (records.hpp) and names the line;
    write_plan -> read_plan -> write_plan is the identity on golden plans
    (test above), and the optional ' local' flag / unknown header keys are
    accepted like the reference's reader (transfer_plan.cpp:73-141)."""
    from paper_2605_22014_b200.native import IntegrityError
    sp = specs.ModelSpec("w", 1, [specs.TensorSpec("W", 0, [8, 8], 0, "param", 4)], 4)
    ok = "plan src_gen=1 dst_gen=2 note=x\ntask W 0 0 1 0:4,0:8 128\ntask W 0 1 1 4:8,0:8 128 local\nkeep W 0 1 4:8,0:8 128\n"
    plan = R.read_plan(ok, sp)
    assert plan.text() == ok.replace(" note=x", "")
    for bad, where in (("task W 0 0 x 0:4,0:8 128\n", "line 2"), ("task W 0 0 1 0-4,0:8 128\n", "bounds"),
                       ("task W 0 0 1 0:4,0:8\n", "byte size"), ("keep W 0 1 4:8,0:8 12z\n", "byte size"),
                       ("frob W\n", "unknown record")):
        with pytest.raises(IntegrityError, match=where):
            R.read_plan("plan src_gen=1 dst_gen=2\n" + bad, sp)
