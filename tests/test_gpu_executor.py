"""Device executor parity: libreshard_b200.so on a B200 vs the reference.

Every case fills the source store with the reference pattern on the device,
poisons the destination with a different pattern, executes the plan through
the C ABI, and checks the destination bytes against (a) the reference's own
execute_plan digest (golden, produced by oracle/_ref) or the C oracle's bytes,
and (b) the analytic gather-reslice pattern via the verify kernel.  Bit-exact:
the tolerance is zero mismatched bytes.
"""

import dataclasses

import numpy as np
import pytest

from helpers import engine_store_digest
from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs
from paper_2605_22014_b200.native import RS_DST, RS_SRC, DomainError

pytestmark = pytest.mark.gpu

SEED = 42


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def make_engine(sp, co, cn, mode="direct", B=1 << 30, **kw):
    eng = R.Engine([0], staging_bytes=B, mode=mode, **kw)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, SEED)
    eng.fill_pattern(RS_DST, SEED ^ 0xDEAD)  # poison: unwritten bytes would show
    return eng


def dst_owners(oracle, sp, cn):
    return sorted(oracle.store_pattern(sp, cn, 0, fill=False).entries.keys())


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_random_pairs_bitexact(mode, golden, oracle_c):
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    for seed, sp, co, cn in specs.iter_random_cases(200, golden["random_pairs"]["base_seed"]):
        want = rows[seed]["exec"]["4096"]
        B = 4096 if mode == "direct" else 1 << 16
        eng = make_engine(sp, co, cn, mode, B, lanes_per_link=1)
        plan = R.compute_transfer_plan(co, cn, sp)
        rep = R.execute_plan(plan, eng)
        assert rep["ok"], (seed, rep)
        assert rep["bytes_moved"] == want["bytes_moved"] and rep["local_copy_bytes"] == want["local_copy_bytes"]
        assert rep["layers_processed"] == want["layers_processed"]
        assert rep["peak_staging_bytes"] <= B
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == want["dst_sha"], seed
        assert eng.verify_pattern(RS_DST, SEED)[0] == 0
        eng.close()


RS_COPY_TMA_NP, RS_COPY_LDG8_NP = 17, 15


@pytest.mark.parametrize("mode,copy_kernel", [("direct", 0), ("direct", RS_COPY_TMA_NP), ("direct", RS_COPY_LDG8_NP),
                                              ("direct", 1), ("direct", 2), ("direct", 3), ("staged", 0)])
def test_c1_gpt2_bitexact(mode, copy_kernel, golden, oracle_c):
    """Full GPT-2 C1 against the reference executor's own destination digest
    (oracle/_ref, tests/golden/c1_exec.json), for the default kernel (0 =
    auto, which must resolve to the TMA bulk copy that carries the headline
    bench) and every explicit variant."""
    sp, co, cn = specs.baseline_case("c1")
    eng = make_engine(sp, co, cn, mode, 1 << 30 if mode == "direct" else 256 << 20, lanes_per_link=2,
                      copy_kernel=copy_kernel)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    want = golden["c1_exec"]["1073741824"]
    if mode == "direct" and copy_kernel in (0, RS_COPY_TMA_NP):
        assert rep["copy_kernel"] == RS_COPY_TMA_NP, rep  # the headline kernel ran
    elif mode == "direct":
        assert rep["copy_kernel"] == copy_kernel, rep
    else:
        assert rep["copy_kernel"] == -1 and rep["ring_same_slot"] == 1, rep
    assert rep["ok"] and rep["bytes_moved"] == want["bytes_moved"]
    assert rep["local_copy_bytes"] == want["local_copy_bytes"]
    assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == want["dst_sha"]
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    # idempotent destination: a second run over the same stores changes nothing
    rep2 = eng.run()
    assert rep2["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


def mini_llama(layers=2):
    return specs.llama("llama-mini", layers)


@pytest.mark.parametrize("mode", ["direct", "staged", "bulk"])
@pytest.mark.parametrize("pair", [((4, 2, 1), (2, 2, 1)), ((2, 2, 1), (4, 2, 1)), ((8, 1, 1), (4, 1, 2)),
                                  ((2, 4, 1), (4, 1, 2)), ((1, 1, 2), (2, 2, 2))])
def test_mixed_dtype_gqa_glu_against_oracle(mode, pair, oracle_c):
    """bf16 params + fp32 master/m/v in one plan, fused GQA QKV + GLU fc1."""
    sp = mini_llama(4)
    (t0, p0, d0), (t1, p1, d1) = pair
    co, cn = specs.iota_config(1, t0, p0, d0), specs.iota_config(2, t1, p1, d1)
    if mode == "bulk":
        eng = make_engine(sp, co, cn, "direct", 1 << 20, copy_kernel=3)
    else:
        eng = make_engine(sp, co, cn, mode, 1 << 20, lanes_per_link=2)
    plan = R.compute_transfer_plan(co, cn, sp)
    text = plan.text()
    assert text == oracle_c.plan_text(sp, co, cn)[0]
    rep = R.execute_plan(plan, eng)
    orep, ostore = oracle_c.execute(sp, co, cn, text, SEED, 1 << 20)
    assert rep["ok"] and orep["ok"]
    assert (rep["bytes_moved"], rep["local_copy_bytes"]) == (orep["bytes_moved"], orep["local_copy_bytes"])
    for (ti, rank), want in ostore.entries.items():
        got = eng.read(RS_DST, rank, ti)
        assert np.array_equal(got, want), (ti, rank)
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


def test_failure_paths_match_oracle(oracle_c):
    sp = mini_llama(2)
    co, cn = specs.iota_config(1, 2, 1, 1), specs.iota_config(2, 4, 1, 1)
    text = oracle_c.plan_text(sp, co, cn)[0]
    # staging budget below one element (SURVEY §4 KAT: failed_layer 0)
    eng = make_engine(sp, co, cn, "direct", 1)
    rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    orep, _ = oracle_c.execute(sp, co, cn, text, SEED, 1)
    assert not rep["ok"] and not orep["ok"]
    assert (rep["failed_layer"], rep["error"], rep["layers_processed"]) == \
        (orep["failed_layer"], orep["error"], orep["layers_processed"])
    eng.close()
    # a task whose bounds escape its source view (mutated plan), in layer 1
    lines = text.splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith("task") and l.split()[2] == "1"
             and l.split()[3] != l.split()[4] and "attn.qkv" in l.split()[1])
    tok = lines[i].split()
    tok[3] = str((int(tok[3]) + 1) % 2)
    lines[i] = " ".join(tok)
    bad = "\n".join(lines) + "\n"
    eng = make_engine(sp, co, cn, "direct")
    rep = R.execute_plan(R.read_plan(bad, sp), eng)
    orep, _ = oracle_c.execute(sp, co, cn, bad, SEED, 1 << 30)
    assert not rep["ok"] and rep["error"] == orep["error"] == "integrity: task bounds escape source view"
    assert rep["failed_layer"] == orep["failed_layer"] == 1
    assert rep["layers_processed"] == orep["layers_processed"] == 1
    eng.close()


def test_verify_kernel_detects_corruption():
    sp = mini_llama(2)
    co, cn = specs.iota_config(1, 2, 1, 1), specs.iota_config(2, 1, 1, 1)
    eng = make_engine(sp, co, cn)
    R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    b = eng.read(RS_DST, 0, 3, 100, 1)
    eng.write(RS_DST, 0, 3, 100, b ^ 0x01)
    bad, first = eng.verify_pattern(RS_DST, SEED)
    assert bad == 1 and first >= 0
    eng.close()


def test_bound_caller_memory():
    """rs_store_bind: caller-owned device buffers (torch allocations)."""
    import torch
    sp = mini_llama(2)
    co, cn = specs.iota_config(1, 4, 1, 1), specs.iota_config(2, 2, 1, 1)
    eng = R.Engine([0], staging_bytes=1 << 20)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    keep = []
    for which, cfg in ((RS_SRC, co), (RS_DST, cn)):
        for ti, t in enumerate(sp.tensors):
            for r in cfg.ranks:
                v = R.view(sp, ti, cfg, r)
                if v is None:
                    continue
                n = int(np.prod([h - l for l, h in v])) * t.bpe
                buf = torch.empty(n, dtype=torch.uint8, device="cuda")
                keep.append(buf)
                eng.bind(which, r, ti, buf.data_ptr(), n)
    eng.fill_pattern(RS_SRC, SEED)
    rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


def test_host_buffers_roundtrip(oracle_c):
    """rs_execute_host: reference-style host stores in, host stores out."""
    sp = mini_llama(2)
    co, cn = specs.iota_config(1, 2, 1, 2), specs.iota_config(2, 4, 1, 1)
    src_store = oracle_c.store_pattern(sp, co, SEED)
    eng = R.Engine([0], staging_bytes=1 << 20)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    keys_src = sorted(src_store.entries)
    want = oracle_c.store_pattern(sp, cn, SEED)
    keys_dst = sorted(want.entries)
    outs = {k: np.zeros_like(want.entries[k]) for k in keys_dst}
    rep = eng.execute_host(R.compute_transfer_plan(co, cn, sp),
                           [src_store.entries[k].ctypes.data for k in keys_src],
                           [outs[k].ctypes.data for k in keys_dst])
    assert rep["ok"]
    for k in keys_dst:
        assert np.array_equal(outs[k], want.entries[k]), k
    eng.close()


@pytest.mark.slow
def test_full_size_c2_on_one_gpu():
    """BASELINE config 2 (Llama-2-7B bf16 + fp32 master/m/v, TP4PP2 -> TP2PP2)
    at full size on one B200 (all logical ranks on device 0): size-independent
    property check -- every destination byte equals the analytic reference
    pattern, and a second run is idempotent."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    sp, co, cn = specs.baseline_case("c2")
    need = 2 * sp.total_bytes()
    if free < need + (1 << 30):
        pytest.skip(f"needs {need / 1e9:.1f} GB free, have {free / 1e9:.1f}")
    eng = make_engine(sp, co, cn, "direct")
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and rep["bytes_moved"] + rep["local_copy_bytes"] == plan.total_bytes()
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    assert eng.verify_pattern(RS_SRC, SEED)[0] == 0  # sources untouched
    eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_distributed_optimizer_repartition(mode, oracle_c):
    """ZeRO-1 re-partition on the device (extension): random pairs vs the C
    oracle's bytes, plus a 4-layer slice of BASELINE config 3 (Llama-3-8B
    TP8 -> TP4DP2 with the distributed optimizer) vs the analytic pattern."""
    for seed, sp, co, cn in specs.iter_random_zero_cases(40):
        eng = make_engine(sp, co, cn, mode, 1 << 16, lanes_per_link=1)
        plan = R.compute_transfer_plan(co, cn, sp)
        rep = R.execute_plan(plan, eng)
        orep, ostore = oracle_c.execute(sp, co, cn, plan.text(), SEED, 1 << 16)
        assert rep["ok"] and orep["ok"], seed
        for (ti, rank), want in ostore.entries.items():
            assert np.array_equal(eng.read(RS_DST, rank, ti), want), (seed, ti, rank)
        eng.close()
    sp, co, cn = specs.sliced_case("c3z", 4)
    eng = make_engine(sp, co, cn, mode, 256 << 20)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


def test_staged_peer_failure_times_out_not_hangs():
    """Robustness of the ring transport: when the receiving side of every
    ring drops out (fault_inject=1), senders exhaust their credits and must
    give up after spin_limit polls with ok=False and a 'ring wait timed out'
    report (the reference's failed-layer contract, executor.cpp:210-215)
    instead of hanging the GPU.  A healthy engine then runs the same plan
    bit-exact, so a failed handoff leaves the device usable."""
    sp, co, cn = specs.sliced_case("c1", 2)
    plan = R.compute_transfer_plan(co, cn, sp)
    eng = make_engine(sp, co, cn, "staged", 1 << 16, lanes_per_link=1,
                      spin_limit=200_000, fault_inject=1)
    rep = R.execute_plan(plan, eng)
    assert not rep["ok"]
    assert "ring wait timed out" in rep["error"]
    eng.close()
    eng = make_engine(sp, co, cn, "staged", 1 << 16, lanes_per_link=1)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged"])
@pytest.mark.parametrize("pair", [((4, 2, 1), (2, 2, 1)), ((2, 2, 1), (4, 2, 1)), ((8, 1, 1), (4, 1, 2)),
                                  ((2, 2, 2), (4, 2, 1))])
def test_searched_placement_bitexact(mode, pair, oracle_c):
    """A destination rank list chosen by rs_plan_placement is an ordinary
    config: its plan (more carryovers / self-sourced tasks, fewer remote
    bytes) executes bit-exact against the C oracle."""
    sp = mini_llama(4)
    (t0, p0, d0), (t1, p1, d1) = pair
    co, cn = specs.iota_config(1, t0, p0, d0), specs.iota_config(2, t1, p1, d1)
    cn, st = R.choose_placement(co, cn, sp, candidates=list(range(max(co.world, cn.world))))
    assert st["remote_bytes"] <= st["given_remote_bytes"]
    eng = make_engine(sp, co, cn, mode, 1 << 20, lanes_per_link=2)
    plan = R.compute_transfer_plan(co, cn, sp)
    text = plan.text()
    assert text == oracle_c.plan_text(sp, co, cn)[0]
    rep = R.execute_plan(plan, eng)
    orep, ostore = oracle_c.execute(sp, co, cn, text, SEED, 1 << 20)
    assert rep["ok"] and orep["ok"] and rep["bytes_moved"] == orep["bytes_moved"] == st["remote_bytes"]
    for (ti, rank), want in ostore.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), want), (ti, rank)
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


@pytest.mark.parametrize("K,cap_kib,discard", [(2, 0, 1), (2, -1, 2), (8, 64, 5), (3, 4, 4), (2, 0, 0)])
def test_ring_geometry_variants_bitexact(K, cap_kib, discard, golden, oracle_c):
    """Ring depth K, the slot cap and the L2 discard of drained slots change
    how frames are batched and when slot lines may be dropped -- never the
    destination bytes (reference digests, 40 random pairs + full GPT-2 C1)."""
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    for seed, sp, co, cn in specs.iter_random_cases(40, golden["random_pairs"]["base_seed"]):
        eng = make_engine(sp, co, cn, "staged", 1 << 16, lanes_per_link=1, slots_per_link=K,
                          ring_slot_kib=cap_kib, ring_discard=discard)
        rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
        assert rep["ok"], (seed, rep)
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            rows[seed]["exec"]["4096"]["dst_sha"], seed
        eng.close()
    sp, co, cn = specs.baseline_case("c1")
    eng = make_engine(sp, co, cn, "staged", 256 << 20, slots_per_link=K, ring_slot_kib=cap_kib,
                      ring_discard=discard)
    plan = R.compute_transfer_plan(co, cn, sp)
    for _ in range(2):
        rep = R.execute_plan(plan, eng)
        assert rep["ok"] and rep["peak_staging_bytes"] <= 256 << 20
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            golden["c1_exec"]["1073741824"]["dst_sha"]
    eng.close()


def test_plan_sized_staging_arena():
    """rs_comm_alloc_plan sizes each destination rank's ring region to the
    plan's rings (<= B); rs_prepare re-sizes a single-process arena that is
    too small for a new plan; results stay bit-exact."""
    sp = mini_llama(4)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 1)
    B = 64 << 20
    eng = make_engine(sp, co, cn, "staged", B, ring_slot_kib=64)
    plan = R.compute_transfer_plan(co, cn, sp)
    eng.comm_alloc(plan)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    assert 0 < rep["peak_staging_bytes"] < B
    eng.close()
    # an arena sized for a lighter plan is grown by prepare (single process)
    eng = make_engine(sp, co, cn, "staged", B)
    light = R.compute_transfer_plan(co, specs.iota_config(2, 4, 2, 1), sp)  # identity layout: no rings
    eng.comm_alloc(light)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


@pytest.mark.parametrize("threads", [512, 1024])
def test_wide_ring_lanes_bitexact(threads, golden, oracle_c):
    """512 / 1024-thread ring-lane CTAs (fewer, wider lanes): same bytes as the
    reference's execute_plan on 30 random pairs."""
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    done = 0
    for seed, sp, co, cn in specs.iter_random_cases(30, golden["random_pairs"]["base_seed"]):
        eng = make_engine(sp, co, cn, "staged", 1 << 16, ring_cta_threads=threads)
        try:
            rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
        except DomainError as e:  # more links than wide lane CTAs fit the device: refused, not wrong
            assert "exceed the co-resident CTA capacity" in str(e)
            eng.close()
            continue
        assert rep["ok"], (seed, rep)
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            rows[seed]["exec"]["4096"]["dst_sha"], seed
        eng.close()
        done += 1
    assert done >= 15, done


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_identity_resize_is_all_carryover(mode, oracle_c):
    """Same layout, new generation: the plan is carryovers only (no tasks,
    no rings); the destination store still receives every byte."""
    sp = mini_llama(2)
    co, cn = specs.iota_config(1, 2, 2, 1), specs.iota_config(2, 2, 2, 1)
    plan = R.compute_transfer_plan(co, cn, sp)
    s = plan.summary()
    assert s["task_count"] == 0 and s["carryover_bytes"] > 0
    eng = make_engine(sp, co, cn, mode, 1 << 20)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and rep["bytes_moved"] == 0 and rep["carryover_bytes"] == s["carryover_bytes"]
    assert rep["peak_staging_bytes"] == 0
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_bounded_memory_invariant_in_layers(mode, oracle_c):
    """SPEC.md:562 on the device: resident staging <= B and independent of the
    number of layers (L in {2, 8, 64}, B = 4096), bytes equal to the C oracle's."""
    peaks = []
    for L in (2, 8, 64):
        ts = [specs.TensorSpec(f"w{l}", l, [32, 16], 0, "param", 4) for l in range(L)]
        sp = specs.ModelSpec(f"layers{L}", L, ts, 4)
        co, cn = specs.iota_config(1, 2, 1, 1), specs.iota_config(2, 4, 1, 1)
        eng = make_engine(sp, co, cn, mode, 4096, lanes_per_link=1)
        plan = R.compute_transfer_plan(co, cn, sp)
        rep = R.execute_plan(plan, eng)
        orep, ostore = oracle_c.execute(sp, co, cn, plan.text(), SEED, 4096)
        assert rep["ok"] and rep["layers_processed"] == orep["layers_processed"] == L
        assert rep["peak_staging_bytes"] <= 4096
        for (ti, rank), want in ostore.entries.items():
            assert np.array_equal(eng.read(RS_DST, rank, ti), want), (L, ti, rank)
        peaks.append(rep["peak_staging_bytes"])
        eng.close()
    assert len(set(peaks)) == 1
    assert (peaks[0] == 0) == (mode == "direct")


@pytest.mark.parametrize("K,cap_kib,mode", [(2, 0, 13), (2, 32, 13), (3, 64, 13), (4, 4, 13), (2, 0, 29),
                                            (3, 64, 29), (2, 1024, 29)])
def test_warp_specialised_lanes_bitexact(K, cap_kib, mode, golden, oracle_c):
    """ring_discard bit 8: warp-specialised ring lanes (a control warp runs the
    flag handshakes as an event loop while the copy warps stream batches);
    bit 16 with it: the copy warps move items with TMA bulk copies:
    same bytes as the reference's execute_plan on 40 random pairs + GPT-2 C1,
    including K = 2 where a blocking control loop would deadlock."""
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    done = 0
    for seed, sp, co, cn in specs.iter_random_cases(40, golden["random_pairs"]["base_seed"]):
        eng = make_engine(sp, co, cn, "staged", 1 << 16, slots_per_link=K,
                          ring_slot_kib=cap_kib, ring_discard=mode, spin_limit=20_000_000)
        try:
            rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
        except DomainError as e:  # TMA lanes hold 112 KB of smem: fewer co-resident lanes
            assert "exceed the co-resident CTA capacity" in str(e)
            eng.close()
            continue
        done += 1
        assert rep["ok"], (seed, rep)
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            rows[seed]["exec"]["4096"]["dst_sha"], seed
        eng.close()
    assert done >= 25, done
    sp, co, cn = specs.baseline_case("c1")
    eng = make_engine(sp, co, cn, "staged", 256 << 20, slots_per_link=K, ring_slot_kib=cap_kib, ring_discard=mode,
                      spin_limit=20_000_000)
    plan = R.compute_transfer_plan(co, cn, sp)
    for _ in range(2):
        rep = R.execute_plan(plan, eng)
        assert rep["ok"]
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            golden["c1_exec"]["1073741824"]["dst_sha"]
    eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_balanced_sources_same_bytes(mode, golden, oracle_c):
    """balance_sources (planner.hpp:18, round-robin over DP replicas) changes
    which replica sends, never the destination bytes: balanced plans execute
    to the reference's default-plan digests (replicas hold identical state)."""
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    n = 0
    for seed, sp, co, cn in specs.iter_random_cases(200, golden["random_pairs"]["base_seed"]):
        if co.dp < 2:
            continue
        plan = R.compute_transfer_plan(co, cn, sp, R.PlanOptions(True))
        eng = make_engine(sp, co, cn, mode, 1 << 16, lanes_per_link=1)
        rep = R.execute_plan(plan, eng)
        assert rep["ok"], (seed, rep)
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            rows[seed]["exec"]["4096"]["dst_sha"], seed
        eng.close()
        n += 1
        if n == 30:
            break
    assert n >= 10


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_shuffled_plan_text_same_bytes(mode, golden, oracle_c):
    """SURVEY §4 property: any order of a layer's tasks gives the same bytes.
    write_plan -> shuffle every task / keep line -> read_plan (re-indexed by
    tensor name, unlike the reference's first-appearance interning,
    transfer_plan.cpp:94-101) -> execute: the reference's digest."""
    import random
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    for seed, sp, co, cn in specs.iter_random_cases(25, golden["random_pairs"]["base_seed"]):
        lines = R.compute_transfer_plan(co, cn, sp).text().splitlines()
        head, body = lines[:1], lines[1:]
        random.Random(seed).shuffle(body)
        plan = R.read_plan("\n".join(head + body) + "\n", sp)
        eng = make_engine(sp, co, cn, mode, 1 << 16, lanes_per_link=1)
        rep = R.execute_plan(plan, eng)
        assert rep["ok"], (seed, rep)
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            rows[seed]["exec"]["4096"]["dst_sha"], seed
        eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_tensor_beyond_2_32_elements(mode):
    """Maximum-size edge: one bf16 tensor of 70001 x 70003 = 4.9 G elements
    (> 2^32, 9.8 GB) split on axis 1, TP3 -> TP4 (ragged ceil blocks on both
    sides, every row strided): 64-bit element / byte offsets in the
    descriptors and the pattern check; every destination byte verified."""
    ts = [specs.TensorSpec("huge", 0, [70001, 70003], 1, "param", 2)]
    sp = specs.ModelSpec("huge", 1, ts, 2)
    co, cn = specs.iota_config(1, 3, 1, 1), specs.iota_config(2, 4, 1, 1)
    eng = make_engine(sp, co, cn, mode, 1 << 30)
    plan = R.compute_transfer_plan(co, cn, sp)
    assert R.verify_plan(plan, co, cn) == []
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and rep["bytes_moved"] + rep["local_copy_bytes"] == plan.total_bytes()
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


def test_strict_layers_staged_global_layer_order(golden, oracle_c):
    """STAGED strict_layers: every CTA of the launch meets a barrier after each
    plan layer, so the transport trace shows the reference's global order
    (executor.cpp:208): every layer-l batch (both roles) ends
    before any layer-(l+1) batch begins.  Bytes stay bit-exact."""
    sp = mini_llama(4)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 1)
    eng = make_engine(sp, co, cn, "staged", 1 << 20, lanes_per_link=2, ring_slot_kib=4, trace=True,
                      strict_layers=True)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0, rep
    text = plan.text()
    orep, ostore = oracle_c.execute(sp, co, cn, text, SEED, 1 << 20)
    for (ti, rank), want in ostore.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), want), (ti, rank)
    tr = eng.trace(0)
    layers = sorted({r["layer"] for r in tr})
    assert len(layers) == 4
    for a, b in zip(layers, layers[1:]):
        end_a = max(r["t_end"] for r in tr if r["layer"] == a)
        begin_b = min(r["t_begin"] for r in tr if r["layer"] == b)
        assert begin_b >= end_a - 1000, (a, b, end_a, begin_b)  # globaltimer granularity
    # repeated strict runs (epoch-valued barrier flags, fresh arrival counter)
    for _ in range(3):
        assert eng.run()["ok"]
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()
    # every golden random pair, strict STAGED, against the reference's digests
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    for seed, sp, co, cn in specs.iter_random_cases(60, golden["random_pairs"]["base_seed"]):
        want = rows[seed]["exec"]["4096"]
        eng = make_engine(sp, co, cn, "staged", 1 << 16, lanes_per_link=1, strict_layers=True)
        rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
        assert rep["ok"] and rep["layers_processed"] == want["layers_processed"], (seed, rep)
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == want["dst_sha"], seed
        eng.close()


@pytest.mark.parametrize("ring_kernel", [2, 1])
def test_strict_layers_stream_lanes(ring_kernel, golden, oracle_c):
    """strict_layers on the TMA stream lanes (16 B-aligned plans): the lane
    launch also runs the local copies and every CTA meets a barrier after
    each layer, so the trace shows the global layer order; bytes equal the C
    oracle's (mixed-dtype Llama) and the reference's digest (full GPT-2 C1).
    ring_kernel 1 forces the classic lanes on the same plans."""
    sp = specs.llama("llama-mini-a16", 4)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 1)
    eng = make_engine(sp, co, cn, "staged", 1 << 20, lanes_per_link=2, ring_slot_kib=16, trace=True,
                      strict_layers=True, ring_kernel=ring_kernel)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and rep["ring_kernel"] == ring_kernel, rep
    _, want = oracle_c.execute(sp, co, cn, plan.text(), SEED, 1 << 20)
    for (ti, rank), arr in want.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), arr), (ti, rank)
    tr = [r for r in eng.trace(0) if r["t_end"]]
    layers = sorted({r["layer"] for r in tr})
    assert len(layers) == 4
    for a, b in zip(layers, layers[1:]):
        end_a = max(r["t_end"] for r in tr if r["layer"] == a)
        begin_b = min(r["t_begin"] for r in tr if r["layer"] == b)
        assert begin_b >= end_a - 1000, (a, b, end_a, begin_b)
    for _ in range(3):  # epoch-valued barrier flags, fresh arrival counter per launch
        assert eng.run()["ok"]
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()
    sp, co, cn = specs.baseline_case("c1")
    eng = make_engine(sp, co, cn, "staged", 256 << 20, strict_layers=True, ring_kernel=ring_kernel)
    rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    assert rep["ok"] and rep["ring_kernel"] == ring_kernel, rep
    assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == golden["c1_exec"]["1073741824"]["dst_sha"]
    eng.close()


def test_strict_scoped_roles_beyond_co_resident_capacity(oracle_c):
    """strict_layers on the stream lanes deals CTA roles by ticket in
    first-layer order and counts each barrier over the CTAs live in its
    layer, so a launch may hold more lane ends than can be co-resident as
    long as one layer's fit: here 96 lanes per link (PP2: the two stages'
    links never share a layer) give more lane CTAs than the device holds.
    The run must neither deadlock nor reorder layers, and lands the C
    oracle's bytes; repeated runs reuse the epoch-valued flags."""
    import torch
    sp = specs.llama("llama-mini-a16", 4)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 1)
    eng = make_engine(sp, co, cn, "staged", 64 << 20, lanes_per_link=96, ring_slot_kib=16, trace=True,
                      strict_layers=True)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and rep["ring_kernel"] == 2, rep
    _, want = oracle_c.execute(sp, co, cn, plan.text(), SEED, 64 << 20)
    for (ti, rank), arr in want.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), arr), (ti, rank)
    tr = [r for r in eng.trace(0) if r["t_end"]]
    lane_ends = 2 * len({r["lane"] for r in tr if r["role"] == 0})
    assert lane_ends > 6 * torch.cuda.get_device_properties(0).multi_processor_count, lane_ends
    layers = sorted({r["layer"] for r in tr})
    for a, b in zip(layers, layers[1:]):
        end_a = max(r["t_end"] for r in tr if r["layer"] == a)
        begin_b = min(r["t_begin"] for r in tr if r["layer"] == b)
        assert begin_b >= end_a - 1000, (a, b, end_a, begin_b)
    for _ in range(3):
        eng.fill_pattern(RS_DST, SEED ^ 0xBEEF)
        assert eng.run()["ok"]
        assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


def test_transport_trace_layer_order_and_causality():
    """STAGED transport trace (rs_trace_read, the reference's RecordingTransport
    on the device): every remote byte appears once per role; each lane
    streams its batches in layer order (SPEC.md:256 layer-ordering property);
    a receiver starts a batch only after its sender published it."""
    sp = mini_llama(4)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 1)
    eng = make_engine(sp, co, cn, "staged", 1 << 20, lanes_per_link=2, ring_slot_kib=4, trace=True)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    tr = eng.trace(0)
    tx = {(r["lane"], r["batch"]): r for r in tr if r["role"] == 0}
    rx = {(r["lane"], r["batch"]): r for r in tr if r["role"] == 1}
    assert tx.keys() == rx.keys() and len(tx) > 8
    assert sum(r["bytes"] for r in tx.values()) == rep["bytes_moved"]
    lanes = {}
    for (lane, b), r in sorted(tx.items()):
        lanes.setdefault(lane, []).append(r)
    for recs in lanes.values():
        layers = [r["layer"] for r in recs]
        assert layers == sorted(layers)
        assert all(a["t_end"] <= b["t_end"] for a, b in zip(recs, recs[1:]))
    for k, s in tx.items():
        assert rx[k]["t_begin"] >= s["t_end"] - 1000, (k, s, rx[k])  # globaltimer granularity
        assert rx[k]["t_end"] >= rx[k]["t_begin"] and s["t_end"] >= s["t_begin"]
    eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_tiny_staging_budget_like_reference(mode, golden, oracle_c):
    """B = 64 bytes per destination rank (the reference's golden B=64 runs all
    succeed): the ring path falls back to one lane per link and K = 1 where
    K slots per lane do not fit, and still lands the reference's bytes with
    resident staging <= B."""
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    for seed, sp, co, cn in specs.iter_random_cases(60, golden["random_pairs"]["base_seed"]):
        want = rows[seed]["exec"]["64"]
        eng = make_engine(sp, co, cn, mode, 64)
        rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
        assert rep["ok"] == bool(want["ok"]), (seed, rep["error"])
        assert rep["bytes_moved"] == want["bytes_moved"] and rep["layers_processed"] == want["layers_processed"]
        assert rep["peak_staging_bytes"] <= 64
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == want["dst_sha"], seed
        eng.close()


def test_budget_below_one_element_per_inbound_link(oracle_c):
    """B = 32 bytes, 16 inbound links into one destination (TP16 -> TP1, fp32):
    no ring fits (32 / 16 < 4 bytes), the reference executor still succeeds
    (B >= one element), so that destination gets direct stores -- same bytes,
    ok, zero staging."""
    sp = specs.ModelSpec("fan-in", 1, [specs.TensorSpec("W", 0, [64, 48], 0, "param", 4),
                                       specs.TensorSpec("b", 0, [64], 0, "param", 4)], 4)
    co, cn = specs.iota_config(1, 16, 1, 1), specs.iota_config(2, 1, 1, 1)
    text = oracle_c.plan_text(sp, co, cn)[0]
    orep, ostore = oracle_c.execute(sp, co, cn, text, SEED, 32)
    eng = make_engine(sp, co, cn, "staged", 32)
    rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    assert rep["ok"] and orep["ok"], rep["error"]
    assert rep["bytes_moved"] == orep["bytes_moved"] and rep["peak_staging_bytes"] == 0
    for (ti, rank), want in ostore.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), want), (ti, rank)
    eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged", "direct-ldg8"])
def test_spec_known_answer_cases_on_device(mode, golden, oracle_ref):
    """The SPEC's known-answer resizes (TP4->TP8 column / row split, DP2->DP4
    replicated, identity, PP layer move; tests/golden/kat.json from the
    reference) executed on the device: the plan is the reference's, and every
    destination byte equals the reference executor's own output (oracle/_ref)."""
    from helpers import cfg_from_json, spec_from_text
    n = 0
    for case in golden["kat"]:
        if case.get("error"):
            continue
        sp = spec_from_text(case["spec"])
        co, cn = cfg_from_json(case["old"]), cfg_from_json(case["new"])
        plan = R.compute_transfer_plan(co, cn, sp)
        assert plan.text() == case["plan"], case["name"]
        if mode == "direct-ldg8":
            eng = make_engine(sp, co, cn, "direct", 1 << 20, copy_kernel=RS_COPY_LDG8_NP)
        else:
            eng = make_engine(sp, co, cn, mode, 1 << 20)
        rep = R.execute_plan(plan, eng)
        orep, ostore = oracle_ref.execute(sp, co, cn, case["plan"], SEED, 1 << 20)
        assert rep["ok"] and orep["ok"], case["name"]
        if mode == "direct":  # every KAT spec is 16 B aligned: the default is the TMA bulk copy
            assert rep["copy_kernel"] == RS_COPY_TMA_NP, (case["name"], rep)
        assert (rep["bytes_moved"], rep["local_copy_bytes"]) == (orep["bytes_moved"], orep["local_copy_bytes"])
        for (ti, rank), want in ostore.entries.items():
            assert np.array_equal(eng.read(RS_DST, rank, ti), want), (case["name"], ti, rank)
        eng.close()
        n += 1
    assert n == 5


@pytest.mark.parametrize("same_slot", [1, 2])
def test_ring_same_slot_policy(same_slot, golden, oracle_c):
    """ring_same_slot: cross-rank tasks whose ranks share a GPU go through the
    rings (1; the one-slot default) or become direct copies (2; the
    multi-slot default) -- same bytes either way, no staging when direct."""
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    for seed, sp, co, cn in specs.iter_random_cases(30, golden["random_pairs"]["base_seed"]):
        eng = make_engine(sp, co, cn, "staged", 1 << 16, ring_same_slot=same_slot)
        rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
        want = rows[seed]["exec"]["4096"]
        assert rep["ok"] and rep["bytes_moved"] == want["bytes_moved"], (seed, rep)
        if same_slot == 2:
            assert rep["peak_staging_bytes"] == 0
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == want["dst_sha"], seed
        eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged", "staged-strict"])
def test_c4_uneven_stage_migration_on_device(mode):
    """BASELINE config 4's point on the device: Llama-2-13B shapes, TP2PP4 ->
    TP4PP2 with an uneven new stage split (4-layer slice: 3/1, the full-size
    21/19 proportion), bf16 + fp32 master/m/v; every destination byte checked
    against the analytic pattern (pinned to the reference's fill_pattern)."""
    sp, co, cn = specs.sliced_case("c4", 4)
    assert cn.layer_stage == [0, 0, 0, 1]
    strict = mode == "staged-strict"
    eng = make_engine(sp, co, cn, "staged" if strict else mode, 1 << 30, strict_layers=strict)
    plan = R.compute_transfer_plan(co, cn, sp)
    assert R.verify_plan(plan, co, cn) == []
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and rep["bytes_moved"] + rep["local_copy_bytes"] == plan.total_bytes(), rep
    assert rep["layers_processed"] == 4
    assert eng.verify_pattern(RS_DST, SEED)[0] == 0
    eng.close()


@pytest.mark.parametrize("ring_kernel,stages,slot_kib", [(2, 2, 64), (2, 1, 32), (2, 3, 128), (2, 4, 0), (2, 2, 16)])
def test_stream_lane_kernels_bitexact(ring_kernel, stages, slot_kib, golden, oracle_c):
    """The TMA stream lanes over stage counts and slot caps: full GPT-2 C1 equals the
    reference's digest (twice: epochs advance), and a 16 B-aligned mixed-dtype
    Llama resize equals the C oracle's bytes.  Descriptor chunks are staged in
    shared memory, so long lanes cross many chunk boundaries."""
    sp, co, cn = specs.baseline_case("c1")
    eng = make_engine(sp, co, cn, "staged", 256 << 20, ring_kernel=ring_kernel, ring_stages=stages,
                      ring_slot_kib=slot_kib)
    plan = R.compute_transfer_plan(co, cn, sp)
    for _ in range(2):
        rep = R.execute_plan(plan, eng)
        assert rep["ok"] and rep["ring_kernel"] == ring_kernel, rep
        assert engine_store_digest(eng, RS_DST, sp, dst_owners(oracle_c, sp, cn)) == \
            golden["c1_exec"]["1073741824"]["dst_sha"]
    eng.close()
    sp = specs.llama("llama-mini-a16", 4)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 2)
    eng = make_engine(sp, co, cn, "staged", 1 << 20, ring_kernel=ring_kernel, ring_stages=stages,
                      ring_slot_kib=slot_kib, lanes_per_link=2)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and rep["ring_kernel"] == ring_kernel, rep
    _, want = oracle_c.execute(sp, co, cn, plan.text(), SEED, 1 << 20)
    for (ti, rank), arr in want.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), arr), (ti, rank)
    eng.close()


@pytest.mark.parametrize("mode", ["direct", "staged", "xfer-free"])
def test_flat_bucket_distributed_optimizer_bitexact(mode, oracle_c):
    """Megatron flat-bucket distributed optimizer on the device (extension,
    SURVEY §8(f)1): flat-bucket shards hold element ranges of their TP block,
    addressed through the block's strides from an offset origin.  Random
    pairs (small buckets: ranges cut mid-row) vs the C oracle's bytes; a
    4-layer slice of BASELINE config 3 with Megatron's layout (c3zb, TP8 ->
    TP4DP2, the default 40M-element buckets) vs the analytic pattern, and its
    16 B-aligned mini version through the STAGED stream lanes."""
    kw = {"lanes_per_link": 1}
    m = "direct" if mode == "xfer-free" else mode
    if mode == "xfer-free":
        kw["copy_kernel"] = 15  # the LDG8 warp copy over flat shards
    n = 0
    for seed, sp, co, cn in specs.iter_random_flat_cases(60):
        if co.dist_opt != 2 and cn.dist_opt != 2:
            continue
        eng = make_engine(sp, co, cn, m, 1 << 16, **kw)
        plan = R.compute_transfer_plan(co, cn, sp)
        rep = R.execute_plan(plan, eng)
        orep, ostore = oracle_c.execute(sp, co, cn, plan.text(), SEED, 1 << 16)
        assert rep["ok"] and orep["ok"], (seed, rep["error"])
        assert rep["bytes_moved"] == orep["bytes_moved"], seed
        for (ti, rank), want in ostore.entries.items():
            assert np.array_equal(eng.read(RS_DST, rank, ti), want), (seed, ti, rank)
        assert eng.verify_pattern(RS_DST, SEED)[0] == 0
        eng.close()
        n += 1
    assert n >= 20
    sp, co, cn = specs.sliced_case("c3zb", 4)
    eng = make_engine(sp, co, cn, m, 256 << 20, **({} if mode == "xfer-free" else {}))
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, SEED)[0] == 0
    assert eng.verify_pattern(RS_SRC, SEED)[0] == 0  # the source is untouched
    eng.close()
    sp = specs.llama("llama-mini-a16", 4, zero=True)
    co = dataclasses.replace(specs.iota_config(1, 2, 2, 2), dist_opt=2, bucket_elems=100_000)
    cn = dataclasses.replace(specs.iota_config(2, 4, 1, 2), dist_opt=2, bucket_elems=250_000)
    eng = make_engine(sp, co, cn, m, 1 << 20, **kw)
    plan = R.compute_transfer_plan(co, cn, sp)
    rep = R.execute_plan(plan, eng)
    assert rep["ok"], rep
    if mode == "staged":
        assert rep["ring_kernel"] == 2, rep  # aligned flat shards run the TMA stream lanes
    _, want = oracle_c.execute(sp, co, cn, plan.text(), SEED, 1 << 20)
    for (ti, rank), arr in want.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), arr), (ti, rank)
    eng.close()


def _random_aligned_resizes(n=10, seed=11):
    """Random TP/PP/DP resizes of the 16 B-aligned mini Llama (mixed bf16 /
    fp32 state), uneven stage splits included: every one runs on the TMA
    stream lanes."""
    import random
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        layers = rng.choice([2, 3, 4, 5])
        shapes = []
        for gen in (1, 2):
            tp, pp, dp = rng.choice([1, 2, 4]), rng.choice([1, 2]), rng.choice([1, 2])
            if tp * pp * dp > 8:
                break
            stages = None
            if pp == 2 and rng.random() < 0.5:
                first = rng.randrange(1, layers)
                stages = [0] * first + [1] * (layers - first)
            shapes.append(specs.iota_config(gen, tp, pp, dp, layer_stage=stages))
        if len(shapes) == 2:
            out.append((layers, shapes[0], shapes[1]))
    return out


@pytest.mark.parametrize("strict,lanes", [(False, 2), (True, 2), (False, 0), (True, 0)])
def test_stream_lanes_random_aligned_resizes(strict, lanes, oracle_c):
    """lanes 0: the engine's own allocation -- proportional + water-filled
    lanes, and under strict layers per-(layer, slot) lane caps with the local
    copies split into run-segmented roles (uneven PP stages included)."""
    for layers, co, cn in _random_aligned_resizes():
        sp = specs.llama("llama-mini-a16", layers)
        eng = make_engine(sp, co, cn, "staged", 1 << 20, lanes_per_link=lanes, ring_slot_kib=16, strict_layers=strict)
        plan = R.compute_transfer_plan(co, cn, sp)
        rep = R.execute_plan(plan, eng)
        assert rep["ok"], (co, cn, rep)
        assert rep["ring_kernel"] == (2 if rep["bytes_moved"] or strict else 0), (co, cn, rep)
        _, want = oracle_c.execute(sp, co, cn, plan.text(), SEED, 1 << 20)
        for (ti, rank), arr in want.entries.items():
            assert np.array_equal(eng.read(RS_DST, rank, ti), arr), (co, cn, ti, rank)
        eng.close()
