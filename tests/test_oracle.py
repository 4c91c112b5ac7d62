"""Pin the C restatement oracle (oracle/oracle.c) to the reference.

Golden fixtures in tests/golden/ were produced by the reference itself
(oracle/_ref, tools/make_golden.py).  These tests run on CPU only.
"""

import gzip
import hashlib
import os

import pytest

from helpers import cfg_from_json, sha, spec_from_text
from paper_2605_22014_b200 import specs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def store_digest(store) -> str:
    h = hashlib.sha256()
    for key in sorted(store.entries):
        h.update(f"{key[0]}:{key[1]}:".encode())
        h.update(store.entries[key].tobytes())
    return h.hexdigest()


def test_kat_plans(oracle_c, golden):
    from oracle.pyoracle import OracleError
    for case in golden["kat"]:
        sp = spec_from_text(case["spec"])
        co, cn = cfg_from_json(case["old"]), cfg_from_json(case["new"])
        if "error" in case and case["error"] is not None:
            with pytest.raises(OracleError) as e:
                oracle_c.plan_text(sp, co, cn)
            assert str(e.value) == case["error"], case["name"]
        else:
            assert oracle_c.plan_text(sp, co, cn)[0] == case["plan"], case["name"]


def test_spec_known_answers(oracle_c):
    # TP4 -> TP8 column-sharded W, fp16: each source emits 2
    # tasks (one local), 2 MiB total
    sp = specs.ModelSpec("w", 1, [specs.TensorSpec("W", 0, [1024, 1024], 1, "param", 2)], 2)
    text, _ = oracle_c.plan_text(sp, specs.iota_config(1, 4, 1, 1), specs.iota_config(2, 8, 1, 1))
    tasks = [l.split() for l in text.splitlines() if l.startswith("task")]
    per_src = {}
    for t in tasks:
        per_src.setdefault(int(t[3]), []).append(t)
    assert all(len(v) == 2 for v in per_src.values()) and len(per_src) == 4
    assert sum(int(t[6]) for t in tasks) == 2 * 1024 * 1024
    # DP2 -> DP4 replicated: 0->2, 0->3 full views + 2 keeps
    sp = specs.ModelSpec("r", 1, [specs.TensorSpec("R", 0, [8, 8], None, "param", 4)], 4)
    text, _ = oracle_c.plan_text(sp, specs.iota_config(1, 1, 1, 2), specs.iota_config(2, 1, 1, 4))
    assert [l.split()[3:5] for l in text.splitlines() if l.startswith("task")] == [["0", "2"], ["0", "3"]]
    assert sum(l.startswith("keep") for l in text.splitlines()) == 2


def test_slice_local_kat(oracle_c):
    import numpy as np
    buf = np.arange(16, dtype=np.uint8)  # owner 4x4, 1-byte elements
    out = oracle_c.slice_local(buf, [0, 0], [4, 4], [1, 2], [3, 4], 1)
    assert list(out) == [6, 7, 10, 11]


def test_chunk_bounds_kat(oracle_c):
    pieces = oracle_c.chunk_bounds([0, 0, 0], [10, 7, 3], 50, 2)
    assert pieces == [([i, 0, 0], [i + 1, 7, 3]) for i in range(10)]
    from oracle.pyoracle import OracleError
    with pytest.raises(OracleError, match="one element exceeds the staging budget"):
        oracle_c.chunk_bounds([0], [4], 1, 2)


def test_random_pairs_against_golden(oracle_c, golden):
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    seed_fill = golden["random_pairs"]["fill_seed"]
    for seed, sp, co, cn in specs.iter_random_cases(200, golden["random_pairs"]["base_seed"]):
        row = rows[seed]
        text, pairs = oracle_c.plan_text(sp, co, cn)
        assert sha(text) == row["plan_sha"], seed
        assert sha(oracle_c.plan_text(sp, co, cn, True)[0]) == row["plan_balanced_sha"], seed
        assert pairs == row["pairs_checked"]
        assert oracle_c.verify_plan(sp, co, cn, text) == row["verify"]
        lines = text.splitlines()
        tl = [i for i, l in enumerate(lines) if l.startswith("task")]
        if tl:
            drop = "\n".join(lines[:tl[0]] + lines[tl[0] + 1:]) + "\n"
            dup = "\n".join(lines + [lines[tl[-1]]]) + "\n"
            assert oracle_c.verify_plan(sp, co, cn, drop) == row["verify_drop"]
            assert oracle_c.verify_plan(sp, co, cn, dup) == row["verify_dup"]
            assert row["verify_drop"] and row["verify_dup"]  # 100 % mutation detection
        for B, want in row["exec"].items():
            rep, store = oracle_c.execute(sp, co, cn, text, seed_fill, int(B))
            rep.pop("seconds")
            assert dict(rep, dst_sha=store_digest(store)) == want, (seed, B)


def test_baseline_plans_against_golden(oracle_c, golden):
    for case in ("c1", "c2", "c3", "c4", "c5", "c5b"):
        sp, co, cn = specs.baseline_case(case)
        for bpe in sorted({t.bpe for t in sp.tensors}):
            key = f"{case}_{bpe}B"
            text, pairs = oracle_c.plan_text(specs.group_spec(sp, bpe), co, cn)
            assert sha(text) == golden["baseline_plans"][key]["plan_sha"], key
            with gzip.open(os.path.join(GOLD, "plans", key + ".txt.gz"), "rt") as f:
                assert f.read() == text


def test_c1_execution_against_reference_digest(oracle_c, golden):
    sp, co, cn = specs.baseline_case("c1")
    text, _ = oracle_c.plan_text(sp, co, cn)
    for B, want in golden["c1_exec"].items():
        rep, store = oracle_c.execute(sp, co, cn, text, 42, int(B))
        rep.pop("seconds")
        assert dict(rep, dst_sha=store_digest(store)) == want, B
        del store


def test_oracle_matches_reference_library(oracle_c, oracle_ref):
    """Where the reference compiled here, compare live on fresh random pairs."""
    for seed, sp, co, cn in specs.iter_random_cases(40, base_seed=777):
        a = oracle_c.plan_text(sp, co, cn)
        b = oracle_ref.plan_text(sp, co, cn)
        assert a == b
        ra, sa = oracle_c.execute(sp, co, cn, a[0], 9, 512)
        rb, sb = oracle_ref.execute(sp, co, cn, b[0], 9, 512)
        ra.pop("seconds"); rb.pop("seconds")
        assert ra == rb
        assert store_digest(sa) == store_digest(sb)


def test_distributed_optimizer_execution_is_analytic(oracle_c):
    """The restatement's executor on ZeRO plans lands every byte where the
    extended view function says (the analytic pattern of C_new)."""
    for seed, sp, co, cn in specs.iter_random_zero_cases(60):
        text, _ = oracle_c.plan_text(sp, co, cn)
        rep, store = oracle_c.execute(sp, co, cn, text, 42, 4096)
        assert rep["ok"], seed
        want = oracle_c.store_pattern(sp, cn, 42)
        for k, arr in want.entries.items():
            assert (store.entries[k] == arr).all(), (seed, k)


def _layered(L):
    ts = [specs.TensorSpec(f"w{l}", l, [32, 16], 0, "param", 4) for l in range(L)]
    return specs.ModelSpec(f"layers{L}", L, ts, 4)


def test_bounded_memory_invariant_in_layers(oracle_c, oracle_ref):
    """peak staging <= B and invariant in L (L in {2, 8, 64}),
    on the reference itself and on the restatement, B = 4096."""
    peaks = []
    for L in (2, 8, 64):
        sp = _layered(L)
        co, cn = specs.iota_config(1, 2, 1, 1), specs.iota_config(2, 4, 1, 1)
        text = oracle_ref.plan_text(sp, co, cn)[0]
        rr, _ = oracle_ref.execute(sp, co, cn, text, 7, 4096)
        rc, _ = oracle_c.execute(sp, co, cn, text, 7, 4096)
        assert rr["ok"] and rc["ok"] and rr["layers_processed"] == rc["layers_processed"] == L
        assert rr["peak_staging_bytes"] == rc["peak_staging_bytes"] <= 4096
        peaks.append(rr["peak_staging_bytes"])
    assert len(set(peaks)) == 1 and peaks[0] > 0
