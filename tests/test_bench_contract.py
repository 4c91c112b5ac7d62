"""bench.py's reference arm runs on the host alone (the reference's CPU
executor from oracle/_ref): its JSON line carries the contract's keys.
CPU only, a 2-layer sample."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle.pyoracle import available
    if not available("ref"):
        pytest.skip("oracle/_ref not built")
    env = {**os.environ, "RS_BENCH_CPU_LAYERS": "2"}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["correct"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["higher_is_better"] is True and d["unit"] == "GB/s"


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_roofline_one_gpu_is_the_2x_hbm_floor():
    b = _bench_module()
    # one slot: everything intra-GPU -> 2 x (plan + carryover) bytes over HBM
    r = b.roofline([[0, 0, 91_060_551_680, 3_280_994_304]], 27.44, 6552.3, 900.0)
    assert r["bound"] == "hbm" and r["algorithmic_bytes_per_launch"] == 2 * (91_060_551_680 + 3_280_994_304)
    assert abs(r["frac"] - r["roofline_ms"] / 27.44) < 1e-3
    assert abs(r["achieved"] - 188_683_091_968 / 27.44e-3 / 1e9) < 0.1


@pytest.mark.parametrize("n", [2, 4, 8])
def test_roofline_multi_gpu_baseline_formula(n):
    """bench.py --gpus N computes BASELINE.md §3's per-GPU roofline from the
    plan's own per-slot traffic (rs_plan_traffic, the placement bench.py uses:
    rank r on GPU r*N//8) -- checked here against an independent evaluation of
    the formula on full-size C2 (CPU: planning only)."""
    b = _bench_module()
    from paper_2605_22014_b200 import reshard as R
    from paper_2605_22014_b200 import specs
    sp, co, cn = specs.baseline_case("c2")
    plan = R.compute_transfer_plan(co, cn, sp)
    so = [r * n // 8 for r in co.ranks]
    sn = [r * n // 8 for r in cn.ranks]
    traffic = R.plan_traffic(plan, co, so, cn, sn, n)
    s = plan.summary()
    assert sum(t[0] for t in traffic) == sum(t[1] for t in traffic)
    assert sum(t[0] + t[2] for t in traffic) == s["total_bytes"]
    assert sum(t[3] for t in traffic) == s["carryover_bytes"]
    step_ms = 40.0
    r = b.roofline(traffic, step_ms, 6552.3, 900.0)
    want = max(max(max(o, i) / 900e9, (o + i + 2 * l + 2 * c) / 6552.3e9) for o, i, l, c in traffic)
    assert abs(r["roofline_ms"] - want * 1e3) < 1e-3
    assert abs(r["frac"] - want * 1e3 / step_ms) < 1e-3
    assert len(r["per_gpu"]) == n and r["peak"] == (900.0 if r["bound"] == "nvlink" else 6552.3)
    if n == 8:  # C2 8 -> 4 is ingress-bound at 23.6 GB into each new GPU, 26.2 ms
        assert r["bound"] == "nvlink" and abs(r["roofline_ms"] - 26.2) < 0.1


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 4, 8])
def test_bench_multi_process_line(n):
    """The N>1 bench line end to end: torchrun with N processes (all on this
    one GPU, RS_BENCH_SAME_DEVICE=1, CUDA-IPC mapped arenas) on a 4-layer C2
    slice; the line carries the BASELINE roofline with per-GPU bytes, the
    STAGED sub-object (N=2: run; larger N: skipped, time-sliced contexts) and
    0 mismatching destination bytes."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {**os.environ, "RS_BENCH_SAME_DEVICE": "1", "RS_BENCH_STAGED": "1" if n == 2 else ""}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n), os.path.join(ROOT, "bench.py"),
           "--gpus", str(n), "--steps", "3", "--warmup", "3", "--profile-layers", "4", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-4000:])
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["correct"]["dst_pattern_mismatches"] == 0
    roof = d["roofline"]
    assert roof["formula"].startswith("max_g") and len(roof["per_gpu"]) == n
    assert roof["nvlink_peak_gbs"] in (900.0,) or "measured" in roof["peak_source"]
    assert d["e2e"]["ok"] and d["e2e"]["h2d_bytes_per_step"] > 0
    st = d["staged"]
    if n == 2:
        assert st["dst_pattern_mismatches"] == 0 and st["within_budget"] and st["kernel"] in ("rs_exchange_kernel", "rs_stream_lane_kernel")
    else:
        assert "skipped" in st


@pytest.mark.gpu
def test_bench_relay_line_c5b_slice():
    """--case c5b --mode staged at N=4 (four processes on this GPU, a 4-layer
    slice): the DP scale-out runs relay chains (relay_routes > 0), the
    roofline is computed from the relay traffic, and every destination byte
    checks out."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {**os.environ, "RS_BENCH_SAME_DEVICE": "1"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr", "127.0.0.1", "--master-port", "29644", os.path.join(ROOT, "bench.py"),
           "--gpus", "4", "--steps", "2", "--warmup", "3", "--profile-layers", "4", "--case", "c5b",
           "--mode", "staged", "--no-e2e", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-4000:])
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert d["correct"]["dst_pattern_mismatches"] == 0
    assert d["config"]["relay"] is True and d["config"]["relay_routes"] > 0
    from paper_2605_22014_b200 import reshard as R
    from paper_2605_22014_b200 import specs
    sp, co, cn = specs.sliced_case("c5b", 4)
    plan = R.compute_transfer_plan(co, cn, sp)
    so = [r * 4 // 8 for r in co.ranks]
    sn = [r * 4 // 8 for r in cn.ranks]
    relay = R.plan_traffic(plan, co, so, cn, sn, 4, relay=True)
    assert [g["out_GB"] for g in d["roofline"]["per_gpu"]] == [round(t[0] / 1e9, 3) for t in relay]
    assert max(t[0] for t in relay) < max(t[0] for t in R.plan_traffic(plan, co, so, cn, sn, 4))
