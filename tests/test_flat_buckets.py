"""Megatron flat-bucket distributed optimizer (extension).

Under a config with dist_opt=2 the fp32 optimizer state (every tensor with a
dp axis) is laid out like Megatron-LM's distributed optimizer: per pipeline
stage, role and TP index, the tensors' TP-local elements form one flat buffer
in reverse spec order (param starts padded to 64 elements), cut into buckets
(closed at >= bucket_elems, ends padded to lcm(dp, 128)), and DP rank d holds
the d-th of dp equal parts of every bucket -- a contiguous element range of
each tensor's TP block, i.e. <= 3 boxes of a matrix.  (megatron/core/
distributed/param_and_grad_buffer.py, megatron/core/optimizer/
distrib_optimizer.py; parity unpinned: no reference implementation, the C
oracle is an independent restatement.)

CPU: layout properties checked from first principles, the planner against
the C oracle (plan text, pairs) and against verify_plan (exact cover of every
held element), and the oracle's own execution against the analytic pattern.
GPU parity lives in test_gpu_executor.py::test_flat_bucket_*.
"""
import dataclasses
import math

import numpy as np
import pytest

from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs


def _tp_local(t, tp, i):
    n = 1
    for k, d in enumerate(t.shape):
        if t.tp_shard_axis == k:
            blk = -(-d // tp)
            lo, hi = blk * i, min(blk * (i + 1), d)
            if lo >= hi:
                return 0
            n *= hi - lo
        else:
            n *= d
    return n


def _ranges(sp, cfg, ti):
    """{(tp, dp): (lo, hi)} from rs_view_range for every position on the tensor's stage."""
    st = cfg.stages(sp.num_layers)[sp.tensors[ti].layer]
    out = {}
    for tp in range(cfg.tp):
        for dp in range(cfg.dp):
            r = cfg.ranks[tp + cfg.tp * (dp + cfg.dp * st)]
            lo, hi, flat = R.view_range(sp, ti, cfg, r)
            assert flat
            out[(tp, dp)] = (lo, hi)
    return out


@pytest.mark.parametrize("dp,bucket", [(2, 0), (2, 3_000_000), (4, 1_000_000), (3, 777_777), (8, 5_000_000)])
def test_ranges_partition_each_tp_block(dp, bucket):
    """Every TP block of every DP-sharded tensor is partitioned by the dp ranks'
    ranges, in rank order; ranges of consecutive tensors in the flat buffer
    respect the 64-element start padding and the bucket-end padding."""
    sp = specs.llama("llama-mini-a16", 3, zero=True)
    cfg = dataclasses.replace(specs.iota_config(1, 2, 1, dp), dist_opt=2, bucket_elems=bucket)
    sharded = [i for i, t in enumerate(sp.tensors) if t.dp_axis is not None]
    for ti in sharded:
        t = sp.tensors[ti]
        rg = _ranges(sp, cfg, ti)
        for tp in range(cfg.tp):
            n = _tp_local(t, cfg.tp, tp)
            cur = 0
            for d in range(dp):
                lo, hi = rg[(tp, d)]
                if lo == hi:
                    continue
                assert lo == cur, (t.tensor_id, tp, d, lo, cur)
                cur = hi
            assert cur == n, (t.tensor_id, tp)


def test_bucket_geometry_from_first_principles():
    """Rebuild the flat buffer of one (stage, role, TP index) in Python and
    compare every tensor's range with the library's."""
    sp = specs.llama("llama-mini-a16", 2, zero=True)
    dp, cap = 4, 400_000
    cfg = dataclasses.replace(specs.iota_config(1, 2, 1, dp), dist_opt=2, bucket_elems=cap)
    align = math.lcm(dp, 128)
    for role in ("param", "m1", "m2"):
        for tp in range(cfg.tp):
            members = [i for i, t in enumerate(sp.tensors) if t.dp_axis is not None and t.role == role]
            pos, bstart, slots, buckets = 0, 0, {}, []
            for i in reversed(members):
                n = _tp_local(sp.tensors[i], cfg.tp, tp)
                if not n:
                    continue
                pos = -(-pos // 64) * 64
                slots[i] = (len(buckets), pos, n)
                pos += n
                if pos - bstart >= cap:
                    end = -(-pos // align) * align
                    buckets.append((bstart, end))
                    bstart = pos = end
            if pos > bstart:
                buckets.append((bstart, -(-pos // align) * align))
            assert all((e - s) % align == 0 for s, e in buckets)
            for i, (b, start, n) in slots.items():
                s, e = buckets[b]
                part = (e - s) // dp
                for d in range(dp):
                    lo, hi = max(start, s + d * part), min(start + n, s + (d + 1) * part)
                    want = (lo - start, hi - start) if lo < hi else (0, 0)
                    r = cfg.ranks[tp + cfg.tp * d]
                    got = R.view_range(sp, i, cfg, r)
                    assert (got[0], got[1]) == want, (sp.tensors[i].tensor_id, tp, d)


def _row_major_boxes(cols, lo, hi):
    """Boxes of the element range [lo, hi) of a [rows, cols] block."""
    out, cur = [], lo
    while cur < hi:
        if cur % cols or hi - cur < cols:  # a partial row
            end = min(hi, (cur // cols + 1) * cols)
        else:  # whole rows
            end = cur + (hi - cur) // cols * cols
        out.append((cur, end))
        cur = end
    return out


def test_matrix_ranges_are_at_most_three_boxes():
    """A matrix's range is a partial first row, whole rows, a partial last
    row: <= 3 boxes -- and the bucket cuts do land mid-row, so the layout is
    not the per-tensor dim chunking."""
    sp = specs.llama("llama-mini-a16", 2, zero=True)
    cn = dataclasses.replace(specs.iota_config(2, 2, 1, 2), dist_opt=2, bucket_elems=150_000)
    mid_row = 0
    for ti, t in enumerate(sp.tensors):
        if t.dp_axis is None or len(t.shape) != 2:
            continue
        for r in cn.ranks:
            v = R.view(sp, ti, cn, r)
            lo, hi, _ = R.view_range(sp, ti, cn, r)
            if v is None or lo == hi:
                continue
            cols = v[1][1] - v[1][0]
            assert len(_row_major_boxes(cols, lo, hi)) <= 3
            mid_row += lo % cols != 0 or hi % cols != 0
    assert mid_row > 0


def test_planner_matches_oracle_and_verifies(oracle_c):
    n = 0
    for seed, sp, co, cn in specs.iter_random_flat_cases(200):
        if co.dist_opt != 2 and cn.dist_opt != 2:
            continue
        plan = R.compute_transfer_plan(co, cn, sp)
        text, pairs = oracle_c.plan_text(sp, co, cn)
        assert plan.text() == text, seed
        assert plan.summary()["pairs_checked"] == pairs, seed
        assert R.verify_plan(plan, co, cn) == [], seed
        assert oracle_c.verify_plan(sp, co, cn, text) == [], seed
        n += 1
    assert n >= 100


def test_verify_catches_dropped_and_duplicated_flat_tasks(oracle_c):
    sp = specs.llama("llama-mini-a16", 2, zero=True)
    co = dataclasses.replace(specs.iota_config(1, 2, 1, 2), dist_opt=2, bucket_elems=100_000)
    cn = dataclasses.replace(specs.iota_config(2, 1, 1, 4), dist_opt=2, bucket_elems=300_000)
    text = R.compute_transfer_plan(co, cn, sp).text()
    lines = text.splitlines()
    idx = [i for i, ln in enumerate(lines) if ln.startswith("task") and ".master" in ln]
    dropped = "\n".join(ln for i, ln in enumerate(lines) if i != idx[len(idx) // 2]) + "\n"
    dup = "\n".join(lines + [lines[idx[0]]]) + "\n"
    for bad, word in ((dropped, "gap"), (dup, "overlap")):
        plan = R.read_plan(bad, sp)
        got = R.verify_plan(plan, co, cn)
        assert any(word in g for g in got), got
        assert any(word in g for g in oracle_c.verify_plan(sp, co, cn, bad))


def test_oracle_execution_matches_pattern(oracle_c):
    """The oracle's executor over flat-bucket stores: every destination byte
    equals the analytic pattern (shard_store.cpp:51-85) of its element."""
    n = 0
    for seed, sp, co, cn in specs.iter_random_flat_cases(60):
        if co.dist_opt != 2 and cn.dist_opt != 2:
            continue
        text, _ = oracle_c.plan_text(sp, co, cn)
        rep, got = oracle_c.execute(sp, co, cn, text, 42, 1 << 12)
        assert rep["ok"], (seed, rep)
        want = oracle_c.store_pattern(sp, cn, 42)
        assert sorted(got.entries) == sorted(want.entries)
        for k, arr in want.entries.items():
            assert np.array_equal(got.entries[k], arr), (seed, k)
        n += 1
    assert n >= 30


def test_c3z_flat_full_size_plan(oracle_c):
    """BASELINE config 3 with Megatron's layout (c3zb): Llama-3-8B TP8 ->
    TP4DP2, default 40M-element buckets: the plan covers every held element
    exactly once and equals the oracle's."""
    sp, co, cn = specs.baseline_case("c3zb")
    plan = R.compute_transfer_plan(co, cn, sp)
    assert R.verify_plan(plan, co, cn) == []
    assert plan.text() == oracle_c.plan_text(sp, co, cn)[0]
    s = plan.summary()
    zs = R.compute_transfer_plan(*specs.baseline_case("c3z")[1:], specs.baseline_case("c3z")[0]).summary()
    # the same new state, cut differently: the bytes it holds are equal
    assert s["total_bytes"] + s["carryover_bytes"] == zs["total_bytes"] + zs["carryover_bytes"]
