"""Placement-aware rank ordering (rs_plan_placement).

The search is pinned against brute force over the real planner: for small
random resizes every injective rank list is planned (rs_plan_compute) and
scored from rs_plan_traffic, and the chosen list must reach the minimum.
Host only (no device)."""

import dataclasses
import itertools

import pytest

from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs
from paper_2605_22014_b200.native import DomainError

NVL, HBM = 900.0, 6552.0


def roofline_ms(sp, co, cn, nslots):
    plan = R.compute_transfer_plan(co, cn, sp)
    tr = R.plan_traffic(plan, co, list(co.ranks), cn, list(cn.ranks), nslots)
    t = 0.0
    for eg, ing, intra, carry in tr:
        t = max(t, max(eg, ing) / (NVL * 1e9), (eg + ing + 2 * intra + 2 * carry) / (HBM * 1e9))
    return t * 1e3, plan.summary()


def test_exhaustive_matches_brute_force():
    n = 0
    for seed, sp, co, cn in specs.iter_random_cases(200):
        if cn.world > 4 or co.world > 6:
            continue
        cand = sorted(set(co.ranks) | set(cn.ranks) | {max(co.ranks + cn.ranks) + 1})
        nslots = max(cand) + 1
        best = min(roofline_ms(sp, co, dataclasses.replace(cn, ranks=list(p)), nslots)[0]
                   for p in itertools.permutations(cand, cn.world))
        got, st = R.choose_placement(co, cn, sp, candidates=cand, nvlink_gbs=NVL, hbm_gbs=HBM)
        assert st["exhaustive"]
        t, s = roofline_ms(sp, co, got, nslots)
        assert t == pytest.approx(best, rel=1e-9, abs=1e-12), seed
        assert st["roofline_ms"] == pytest.approx(t, rel=1e-9, abs=1e-12)
        assert st["remote_bytes"] == s["remote_bytes"] and st["carryover_bytes"] == s["carryover_bytes"]
        given, _ = roofline_ms(sp, co, cn, nslots)
        assert st["given_roofline_ms"] == pytest.approx(given, rel=1e-9, abs=1e-12)
        assert t <= given * (1 + 1e-9)
        assert sorted(got.ranks) == sorted(set(got.ranks)) and set(got.ranks) <= set(cand)
        n += 1
    assert n >= 20


def test_local_search_never_worse_than_given():
    for seed, sp, co, cn in specs.iter_random_cases(60, 777):
        cand = sorted(set(co.ranks) | set(cn.ranks))
        got, st = R.choose_placement(co, cn, sp, candidates=cand, exhaustive_limit=1)
        assert not st["exhaustive"] or len(cand) == 1
        assert st["roofline_ms"] <= st["given_roofline_ms"] * (1 + 1e-9), seed
        assert R.verify_plan(R.compute_transfer_plan(co, got, sp), co, got) == []


def test_baseline_configs_halve_the_8gpu_roofline():
    """Every BASELINE resize on 8 GPUs (one rank per GPU): the searched list
    at least halves the iota list's NVLink-bound roofline (C1: no remote bytes)."""
    for case in ("c1", "c2", "c3", "c3z", "c4", "c5", "c5b"):
        sp, co, cn = specs.baseline_case(case)
        got, st = R.choose_placement(co, cn, sp, candidates=list(range(8)))
        assert st["exhaustive"]
        assert st["roofline_ms"] <= 0.55 * st["given_roofline_ms"], (case, st)
        assert st["remote_bytes"] < st["given_remote_bytes"], case
        assert R.verify_plan(R.compute_transfer_plan(co, got, sp), co, got) == []
    sp, co, cn = specs.baseline_case("c2")
    got, _ = R.choose_placement(co, cn, sp, candidates=list(range(8)))
    assert got.ranks == [0, 2, 4, 6]  # each new TP rank keeps the old quarter it already holds


def test_placement_errors():
    sp, co, cn = specs.baseline_case("c1")
    with pytest.raises(DomainError):
        R.choose_placement(co, cn, sp, candidates=[0, 1, 2])  # fewer candidates than positions
    with pytest.raises(DomainError):
        R.choose_placement(co, cn, sp, candidates=[0, 1, 2, 3, 4, 5, 6, 6])
    with pytest.raises(DomainError):
        R.choose_placement(co, cn, sp, candidates=list(range(8)), nvlink_gbs=-1.0)
