"""Runtime hook: the live-handoff lifecycle.

CPU tests drive ``LiveHandoff`` over a recording stand-in engine (the planner
is real host code) and check the reference's state machine rules
(generation.cpp:95-107 trigger/queue, :272-290 atomic switch, :300-304 lookup,
:315-362 abort / shadow loss).  GPU tests run chains of handoffs on a B200:
after every switch the *active* store (RS_SRC, the old destination) must hold
the analytic pattern -- the pattern is a function of global coordinates, so it
is layout independent and a chain of reshards must preserve it bit-exactly.
"""

import dataclasses

import pytest

from paper_2605_22014_b200 import specs
from paper_2605_22014_b200.handoff import HandoffError, LiveHandoff, LookupResult, Phase
from paper_2605_22014_b200.native import RS_DST, RS_SRC
from paper_2605_22014_b200.specs import iota_config

SEED = 42


class FakeEngine:
    """Records the calls LiveHandoff makes; no device."""

    def __init__(self, fail=False):
        self.configs, self.models, self.calls, self.fail = {}, {}, [], fail

    def layout(self, which, model, config, slots=None):
        self.calls.append(("layout", which, config.describe()))
        self.configs[which], self.models[which] = config, model

    def alloc(self, which):
        self.calls.append(("alloc", which))

    def free(self, which):
        self.calls.append(("free", which))

    def store_bytes(self, which):
        return 1000 + which

    def prepare(self, plan):
        self.calls.append(("prepare", plan.total_bytes()))

    def swap_stores(self):
        self.calls.append(("swap",))
        self.configs = {k ^ 1: v for k, v in self.configs.items()}

    def switch(self, plan, drain_events=None, swap=True):
        self.calls.append(("switch", drain_events))
        ok = not self.fail
        if ok and swap:
            self.configs = {k ^ 1: v for k, v in self.configs.items()}
        return {"drain_ms": 1.0, "transfer_ms": 2.0, "swap_ms": 0.01, "pause_ms": 3.01,
                "transfer_bytes": plan.total_bytes(), "swapped": ok and swap,
                "exec": {"ok": ok, "error": "" if ok else "ring wait timed out",
                         "failed_layer": None if ok else 0}}


def _mini(layers=2):
    return specs.llama("llama-mini", layers)


def test_lifecycle_transitions_and_lookup():
    model = _mini()
    c0, c1 = iota_config(1, 4, 2, 1), iota_config(2, 2, 2, 1)
    eng = FakeEngine()
    h = LiveHandoff(eng, model, c0)
    assert eng.configs[RS_SRC] == c0 and h.phase is Phase.STABLE
    with pytest.raises(ValueError, match="active\\+1"):
        h.trigger_resize(dataclasses.replace(c1, gen=5))
    with pytest.raises(HandoffError):
        h.switch()
    h.trigger_resize(c1)
    assert h.phase is Phase.PREPARE and h.shadow == c1
    h.prepare()
    assert h.phase is Phase.READY and h.extra_allocation_bytes() == 1001
    st = h.switch(drain_events=[None])
    assert h.phase is Phase.STABLE and h.active == c1 and h.shadow is None
    assert st.transfer_bytes == h.last_switch.transfer_bytes > 0
    assert (st.old_world, st.new_world, st.union_world) == (8, 4, 8)
    assert st.pause_s == pytest.approx(3.01e-3)
    assert h.extra_allocation_bytes() == 0
    assert [r.to for r in h.transition_log] == [Phase.PREPARE, Phase.READY, Phase.SWITCH,
                                                Phase.CLEANUP, Phase.STABLE]
    assert h.transition_log[2].gen_shadow == 2 and h.transition_log[3].gen_active == 2
    assert h.lookup(2) is LookupResult.ACTIVE
    assert h.lookup(1) is LookupResult.STALE
    assert h.lookup(3) is LookupResult.UNKNOWN
    assert ("free", RS_DST) in eng.calls  # old generation reclaimed in Cleanup


def test_queue_rebases_and_invalid_target_rejected():
    model = _mini()
    c0 = iota_config(1, 4, 2, 1)
    eng = FakeEngine()
    h = LiveHandoff(eng, model, c0)
    with pytest.raises(ValueError, match="invalid target"):
        h.trigger_resize(iota_config(2, 1, 3, 1))  # 3 stages for 2 layers: an empty stage
    h.trigger_resize(iota_config(2, 2, 2, 1))
    h.trigger_resize(iota_config(99, 2, 1, 2))  # queued while in flight; gen rebased later
    assert h.queued_events == 1
    h.prepare()
    h.switch()
    # queued target popped on return to Stable, rebased to active+1 = 3
    assert h.phase is Phase.PREPARE and h.shadow.gen == 3 and h.queued_events == 0
    h.prepare()
    h.switch()
    assert h.active.describe() == "TP2PP1DP2" and h.active.gen == 3


def test_failed_transfer_falls_back_to_active():
    model = _mini()
    c0, c1 = iota_config(1, 4, 2, 1), iota_config(2, 2, 2, 1)
    eng = FakeEngine(fail=True)
    h = LiveHandoff(eng, model, c0)
    h.trigger_resize(c1)
    h.prepare()
    with pytest.raises(HandoffError, match="timed out"):
        h.switch()
    assert h.phase is Phase.STABLE and h.active == c0 and h.shadow is None
    assert h.last_fallback.reason == "ring wait timed out" and h.last_fallback.failed_layer == 0
    assert eng.configs[RS_SRC] == c0  # no swap happened
    assert h.extra_allocation_bytes() == 0


def test_shadow_rank_lost_restarts_prepare():
    model = _mini()
    c0 = iota_config(1, 4, 2, 1)
    eng = FakeEngine()
    h = LiveHandoff(eng, model, c0)
    h.trigger_resize(iota_config(2, 2, 2, 2))
    h.prepare()
    h.shadow_rank_lost(100, iota_config(0, 2, 2, 1))  # not in the shadow: ignored
    assert h.phase is Phase.READY
    h.shadow_rank_lost(7, iota_config(0, 2, 2, 1))
    assert h.phase is Phase.PREPARE and h.shadow.describe() == "TP2PP2DP1" and h.shadow.gen == 2
    h.prepare()
    h.switch()
    assert h.active.world == 4


# ----------------------------------------------------------------------- GPU

@pytest.fixture
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CHAIN = [(4, 2, 1), (2, 2, 1), (2, 1, 2), (1, 4, 1), (4, 1, 2), (4, 2, 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_gpu_handoff_chain_preserves_state(_cuda, mode):
    """Six live handoffs in a row through rs_switch; the active store is
    checked against the analytic pattern after every one."""
    from paper_2605_22014_b200 import reshard as R
    model = _mini(4)
    eng = R.Engine([0], staging_bytes=1 << 20, mode=mode)
    h = LiveHandoff(eng, model, iota_config(1, *CHAIN[0]))
    eng.fill_pattern(RS_SRC, SEED)
    for gen, shape in enumerate(CHAIN[1:], start=2):
        h.trigger_resize(iota_config(gen, *shape))
        h.prepare()
        st = h.switch()
        assert h.active.gen == gen and h.phase is Phase.STABLE
        assert st.exec_report["ok"] and st.transfer_s > 0
        assert st.pause_s == pytest.approx(st.drain_s + st.transfer_s + st.swap_s)
        assert eng.configs[RS_SRC] == h.active
        assert eng.verify_pattern(RS_SRC, SEED)[0] == 0, (gen, shape)
    eng.close()


@pytest.mark.gpu
def test_gpu_switch_drains_training_stream(_cuda):
    """The transfer waits in stream order for the training stream's boundary
    event; drain time is device-measured from the switch call."""
    import torch
    from paper_2605_22014_b200 import reshard as R
    model = _mini(2)
    eng = R.Engine([0], staging_bytes=1 << 20)
    h = LiveHandoff(eng, model, iota_config(1, 4, 2, 1))
    eng.fill_pattern(RS_SRC, SEED)
    h.trigger_resize(iota_config(2, 2, 2, 1))
    h.prepare()
    train = torch.cuda.Stream()
    with torch.cuda.stream(train):
        torch.cuda._sleep(200_000_000)  # ~0.1 s of "training" in flight
        boundary = torch.cuda.Event()
        boundary.record(train)
    st = h.switch(drain_events=[boundary.cuda_event])
    assert st.drain_s > 0.02, st
    assert boundary.query()  # the transfer could not start before the boundary
    assert eng.verify_pattern(RS_SRC, SEED)[0] == 0
    eng.close()


@pytest.mark.gpu
def test_gpu_switch_failure_keeps_active_generation(_cuda):
    """A peer failure during the transfer (ring receivers drop out) aborts the
    handoff: the active store is untouched and still verifies, the machine is
    Stable on the old generation, and a new trigger can proceed."""
    from paper_2605_22014_b200 import reshard as R
    model = _mini(2)
    eng = R.Engine([0], staging_bytes=1 << 16, mode="staged", lanes_per_link=1,
                   spin_limit=200_000, fault_inject=1)
    c0 = iota_config(1, 4, 2, 1)
    h = LiveHandoff(eng, model, c0)
    eng.fill_pattern(RS_SRC, SEED)
    h.trigger_resize(iota_config(2, 2, 2, 1))
    h.prepare()
    with pytest.raises(HandoffError, match="timed out"):
        h.switch()
    assert h.phase is Phase.STABLE and h.active == c0
    assert eng.configs[RS_SRC] == c0
    assert eng.verify_pattern(RS_SRC, SEED)[0] == 0
    eng.close()
