"""Relay chains for DP broadcasts (forwarding).

The reference sources every region a new DP replica needs from the dp-0
owner (proj/src/planner.cpp:154-171), so a DP scale-out (BASELINE config 5b)
sends each box once per replica from one GPU.  With relay chains the
destination receivers forward drained ring batches to the next replica.

* CPU: rs_plan_traffic_ex(RS_TRAFFIC_RELAY) on the BASELINE resizes (C5b's hot
  source drops from 47.2 to 23.6 GB of egress), conservation of bytes, and
  that relaying never raises a slot's peak egress.
* GPU: STAGED with relay across 3-4 processes sharing one B200 (CUDA-IPC
  mapped rings, forwarded hops): every destination shard equals the
  reference executor's bytes (oracle/_ref) and the analytic pattern.
"""
import hashlib
import json
import os

import pytest

from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs

GB = 1e9


def _slots(cfg, n, nranks):
    return [r * n // nranks for r in cfg.ranks]


def _traffic(case, n=8, relay=True):
    sp, co, cn = specs.baseline_case(case)
    plan = R.compute_transfer_plan(co, cn, sp)
    nr = max(max(co.ranks), max(cn.ranks)) + 1
    so, sn = _slots(co, n, nr), _slots(cn, n, nr)
    return plan, R.plan_traffic(plan, co, so, cn, sn, n, relay=relay), R.plan_traffic(plan, co, so, cn, sn, n)


def test_c5b_hot_source_egress_halves():
    plan, relay, p2p = _traffic("c5b")
    assert max(t[0] for t in p2p) == pytest.approx(47.2 * GB, rel=2e-3)
    assert max(t[0] for t in relay) == pytest.approx(23.6 * GB, rel=2e-3)
    # ingress, intra-GPU and carryover bytes are what the plan says either way
    assert [t[1:] for t in relay] == [t[1:] for t in p2p]
    s = plan.summary()
    assert sum(t[0] for t in relay) == sum(t[1] for t in relay)
    assert sum(t[0] + t[2] for t in relay) == s["total_bytes"]
    # the BASELINE roofline: 52.4 ms (dp0 hot spot) -> 26.2 ms (the ingress bound)
    roof = lambda tr: max(max(o, i) / 900e9 for o, i, _, _ in tr) * 1e3  # noqa: E731
    assert roof(p2p) == pytest.approx(52.4, rel=3e-3)
    assert roof(relay) == pytest.approx(26.2, rel=3e-3)


@pytest.mark.parametrize("case", ["c1", "c2", "c3", "c5", "c5b"])
def test_relay_never_raises_peak_egress(case):
    _, relay, p2p = _traffic(case)
    assert max(t[0] for t in relay) <= max(t[0] for t in p2p)
    assert sum(t[1] for t in relay) == sum(t[1] for t in p2p)


def _dp_scaleout_cases():
    """Small DP scale-out resizes of the 16 B-aligned mini Llama with a
    placement that puts two replicas of one source on two other slots."""
    out = []
    # C5b's shape: TP2PP2 -> TP2PP2DP2 over 4 slots (new replicas shifted one slot)
    out.append({"name": "c5b-mini", "layers": 4, "bpe": 4, "old": [2, 2, 1], "new": [2, 2, 2],
                "slot_old": [0, 1, 2, 3], "slot_new": [(r // 2 + 1) % 4 for r in range(8)], "world": 4})
    # TP1PP2 -> TP1PP2DP2 over 3 slots, bf16 group, two lanes per link
    out.append({"name": "pp2-dp2", "layers": 3, "bpe": 2, "old": [1, 2, 1], "new": [1, 2, 2],
                "slot_old": [0, 1], "slot_new": [2, 2, 0, 2], "world": 3, "lanes": 2})
    # the same with the reference's layer barriers (strict layers on the stream lanes)
    out.append(dict(out[0], name="c5b-mini-strict", strict=True))
    # the engine's own lane allocation (water-filled lanes; strict: per-layer
    # caps and run-segmented local roles), fused and strict
    out.append(dict(out[0], name="c5b-mini-auto", lanes=0))
    out.append(dict(out[0], name="c5b-mini-strict-auto", strict=True, lanes=0))
    # TP2 -> TP1PP1DP4 (a box fans out to 3 new replicas: chains of length 3)
    out.append({"name": "tp2-dp4", "layers": 2, "bpe": 4, "old": [2, 1, 1], "new": [1, 1, 4],
                "slot_old": [0, 1], "slot_new": [2, 3, 0, 1], "world": 4, "staging": 256 << 10})
    return out


def _random_relay_cases(n=6, seed=7):
    """Random DP scale-outs of the aligned mini Llama (either dtype group)
    over 3-4 slots with random rank placements, kept when relay chains
    change the traffic (so every case forwards)."""
    import random
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        tp0, pp0 = rng.choice([1, 2, 4]), rng.choice([1, 2])
        dpn, tpn, ppn = rng.choice([2, 3, 4]), rng.choice([1, 2]), rng.choice([1, 2])
        wo, wn = tp0 * pp0, tpn * ppn * dpn
        if wn > 8:
            continue
        w, layers, bpe = rng.choice([3, 4]), rng.choice([2, 3, 4]), rng.choice([2, 4])
        so = [rng.randrange(w) for _ in range(wo)]
        sn = [rng.randrange(w) for _ in range(wn)]
        if len(set(so) | set(sn)) < w:
            continue
        sp = specs.group_spec(specs.llama("llama-mini-a16", layers), bpe)
        co, cn = specs.iota_config(1, tp0, pp0, 1), specs.iota_config(2, tpn, ppn, dpn)
        plan = R.compute_transfer_plan(co, cn, sp)
        if R.plan_traffic(plan, co, so, cn, sn, w, relay=True) == R.plan_traffic(plan, co, so, cn, sn, w):
            continue
        out.append({"name": f"rand{len(out)}", "layers": layers, "bpe": bpe, "old": [tp0, pp0, 1],
                    "new": [tpn, ppn, dpn], "slot_old": so, "slot_new": sn, "world": w,
                    "lanes": rng.choice([1, 2])})
    return out


@pytest.mark.parametrize("case", _dp_scaleout_cases(), ids=lambda c: c["name"])
def test_mini_cases_have_relay_chains(case):
    """CPU: the test placements do exercise relays (chains exist and the hot
    slot's egress drops)."""
    sp = specs.group_spec(specs.llama("llama-mini-a16", case["layers"]), case["bpe"])
    co, cn = specs.iota_config(1, *case["old"]), specs.iota_config(2, *case["new"])
    plan = R.compute_transfer_plan(co, cn, sp)
    w = case["world"]
    relay = R.plan_traffic(plan, co, case["slot_old"], cn, case["slot_new"], w, relay=True)
    p2p = R.plan_traffic(plan, co, case["slot_old"], cn, case["slot_new"], w)
    assert max(t[0] for t in relay) < max(t[0] for t in p2p)


@pytest.mark.gpu
@pytest.mark.parametrize("case", _dp_scaleout_cases() + _random_relay_cases(), ids=lambda c: c["name"])
def test_relay_staged_bitexact_vs_reference(case, oracle_ref):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from test_multiprocess import launch
    os.environ["RS_RELAY_CASE"] = json.dumps(case)
    try:
        outs = launch("relay", world=case["world"], timeout=900)
    finally:
        del os.environ["RS_RELAY_CASE"]
    sp = specs.group_spec(specs.llama("llama-mini-a16", case["layers"]), case["bpe"])
    co, cn = specs.iota_config(1, *case["old"]), specs.iota_config(2, *case["new"])
    text = oracle_ref.plan_text(sp, co, cn)[0]
    _, want = oracle_ref.execute(sp, co, cn, text, 42, 1 << 20)
    got = {}
    for o in outs:
        r = o["result"]
        assert r["ok"], r
        assert r["mismatches"] == 0, r
        got.update(r["digests"])
    assert r["traffic"] != r["traffic_p2p"]  # relays ran
    assert sorted(got) == sorted(f"{ti}:{rk}" for ti, rk in want.entries)
    for (ti, rk), arr in want.entries.items():
        assert got[f"{ti}:{rk}"] == hashlib.sha256(arr.tobytes()).hexdigest(), (ti, rk)
    assert all(o["result"]["relay_routes"] > 0 for o in outs)
