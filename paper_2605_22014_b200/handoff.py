"""Runtime hook: the dual-world live handoff driving real device stores.

The reference's ``GenerationMachine`` (proj/include/reshard/generation.hpp:97-201,
proj/src/generation.cpp) is a time-driven simulator: its Switch phase prices
drain + transfer + swap with cost-model constants (``run_switch``,
generation.cpp:239-270, ``transfer_time_s``).  ``LiveHandoff`` keeps the same
lifecycle and vocabulary -- Stable -> Prepare -> Ready -> Switch -> Cleanup ->
Stable, FIFO queueing of triggers, generation lookup, abort edges -- but every
phase does the work on the GPU instead of pricing it:

* Prepare (overlapped with training): compute + verify the transfer plan, lay
  out and allocate the shadow generation's shard store, compile and upload
  the engine's descriptors (``rs_prepare``);
* Switch (training paused): ``rs_switch`` -- the reshard streams wait for the
  training streams' iteration-boundary events (drain), the plan runs on the
  device (transfer), the stores exchange roles (swap, the pointer swap of
  ``atomic_switch``, generation.cpp:272-290); the three are timed on the
  device and reported as ``SwitchStats`` (generation.hpp:78-91);
* Cleanup: the old generation's store is released (asynchronous in the
  reference, no pause).

Multi-process (one process per GPU): pass ``group``; every process drives its
own slots, shadow arenas are exchanged during Prepare (CUDA IPC handles over
the gloo/NCCL control group) and a barrier after the switch is the commit
point.  Out of scope: the cost model, mock warm-up, checkpoint
fallback bookkeeping beyond the state transitions.
"""

from __future__ import annotations

import dataclasses
import enum
import time
from collections import deque
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import reshard as R
from .native import RS_COMM, RS_DST, RS_SRC
from .specs import ModelSpec, ParallelConfig


class Phase(enum.Enum):
    STABLE = "Stable"
    PREPARE = "Prepare"
    READY = "Ready"
    SWITCH = "Switch"
    CLEANUP = "Cleanup"


class LookupResult(enum.Enum):
    ACTIVE = "active"
    STALE = "stale"
    UNKNOWN = "unknown"


@dataclass
class TransitionRecord:
    t: float
    from_: Phase
    to: Phase
    gen_active: int
    gen_shadow: Optional[int]


@dataclass
class SwitchStats:
    """generation.hpp:78-91 with measured pieces (seconds, like the reference)."""
    trigger_t: float = 0.0
    prepare_s: float = 0.0
    switch_start: float = 0.0
    drain_s: float = 0.0
    transfer_s: float = 0.0
    swap_s: float = 0.0
    pause_s: float = 0.0
    transfer_bytes: int = 0
    old_world: int = 0
    new_world: int = 0
    union_world: int = 0
    exec_report: dict = field(default_factory=dict)


@dataclass
class AllocationRecord:
    what: str
    bytes: int
    released: bool = False


@dataclass
class FallbackOutcome:
    """Abort edge (generation.cpp:315-340): the active store is untouched."""
    reason: str
    failed_layer: Optional[int] = None


class HandoffError(RuntimeError):
    pass


class LiveHandoff:
    def __init__(self, engine: R.Engine, model: ModelSpec, initial: ParallelConfig,
                 rank_device: Optional[Sequence[int]] = None, group=None,
                 plan_options: Optional[R.PlanOptions] = None, verify: bool = True):
        """``engine``'s RS_SRC store must hold (or be laid out here for) the
        initial generation; ``rank_device`` maps each rank-list position of a
        config to a device slot (default: all on slot 0)."""
        self.engine = engine
        self.model = model
        self.group = group
        self.plan_options = plan_options
        self.verify = verify
        self._placement = rank_device
        self._active = initial
        self._shadow: Optional[ParallelConfig] = None
        self._phase = Phase.STABLE
        self._queue: deque = deque()
        self._plan: Optional[R.TransferPlan] = None
        self._t0 = time.perf_counter()
        self._prepare_started = 0.0
        self._prepare_s = 0.0
        self.transition_log: List[TransitionRecord] = []
        self.allocation_ledger: List[AllocationRecord] = []
        self.last_switch: Optional[SwitchStats] = None
        self.last_fallback: Optional[FallbackOutcome] = None
        if engine.configs.get(RS_SRC) is None:
            engine.layout(RS_SRC, model, initial, self._slots(initial))
            engine.alloc(RS_SRC)
            self._connect((RS_SRC,))

    # -- state ---------------------------------------------------------------
    @property
    def phase(self) -> Phase:
        return self._phase

    @property
    def active(self) -> ParallelConfig:
        return self._active

    @property
    def shadow(self) -> Optional[ParallelConfig]:
        return self._shadow

    @property
    def queued_events(self) -> int:
        return len(self._queue)

    @property
    def plan(self) -> Optional[R.TransferPlan]:
        return self._plan

    def now(self) -> float:
        return time.perf_counter() - self._t0

    def lookup(self, generation_id: int) -> LookupResult:
        """generation.cpp:300-304: stale ids are rejected after the swap."""
        if generation_id == self._active.gen:
            return LookupResult.ACTIVE
        if generation_id < self._active.gen:
            return LookupResult.STALE
        return LookupResult.UNKNOWN

    def extra_allocation_bytes(self) -> int:
        return sum(a.bytes for a in self.allocation_ledger if not a.released)

    # -- transitions ---------------------------------------------------------
    def trigger_resize(self, target: ParallelConfig) -> None:
        """generation.cpp:95-107: queued FIFO while a handoff is in flight;
        otherwise the target must be generation active+1 and valid."""
        if self._phase != Phase.STABLE:
            self._queue.append(target)
            return
        if target.gen != self._active.gen + 1:
            raise ValueError("trigger_resize: target generation must be active+1")
        bad = R.validate_config(target, self.model)
        if bad:
            raise ValueError("trigger_resize: invalid target: " + bad[0])
        self._start_prepare(target)

    def prepare(self) -> None:
        """Prepare-phase work (overlaps training): plan, shadow store, compiled
        descriptors.  Prepare -> Ready."""
        if self._phase != Phase.PREPARE:
            raise HandoffError(f"prepare: phase is {self._phase.value}, not Prepare")
        t = time.perf_counter()
        plan = R.compute_transfer_plan(self._active, self._shadow, self.model, self.plan_options)
        if self.verify:
            bad = R.verify_plan(plan, self._active, self._shadow)
            if bad:
                self.abort_and_fallback("plan_verify: " + bad[0])
                raise HandoffError("prepare: plan verification failed: " + bad[0])
        eng = self.engine
        eng.layout(RS_DST, self.model, self._shadow, self._slots(self._shadow))
        eng.alloc(RS_DST)
        self._allocate("shadow_store", eng.store_bytes(RS_DST))
        if getattr(eng, "mode", "direct") == "staged":
            eng.comm_alloc(plan)  # plan-sized rings (<= B per dst rank): they follow the shadow layout
            self._connect((RS_DST, RS_COMM))
        else:
            self._connect((RS_DST,))
        eng.prepare(plan)
        self._plan = plan
        self._prepare_s = time.perf_counter() - t
        self._record(Phase.READY)

    def switch(self, drain_events: Optional[Sequence[int]] = None) -> SwitchStats:
        """Ready -> Switch -> Cleanup -> Stable at an iteration boundary.
        ``drain_events``: cudaEvent_t handles the training streams recorded at
        the boundary (one per local device).  On a failed transfer the machine
        falls back to Stable on the untouched active generation and raises."""
        if self._phase != Phase.READY:
            raise HandoffError(f"switch: phase is {self._phase.value}, not Ready")
        start = self.now()
        self._record(Phase.SWITCH)
        old, new = self._active, self._shadow
        st = self.engine.switch(self._plan, drain_events, swap=True)
        ok = st["exec"]["ok"]
        if self.group is not None:
            ok = self._all_ok(ok)
        if not ok:
            if st["swapped"]:  # a peer failed after we swapped: roll back our roles
                self.engine.swap_stores()
            self.abort_and_fallback(st["exec"]["error"] or "peer transfer failed",
                                    st["exec"]["failed_layer"])
            raise HandoffError("switch: transfer failed: " + (st["exec"]["error"] or "peer failure"))
        union = list(old.ranks) + [r for r in new.ranks if r not in set(old.ranks)]
        stats = SwitchStats(trigger_t=self._prepare_started, prepare_s=self._prepare_s,
                            switch_start=start, drain_s=st["drain_ms"] / 1e3,
                            transfer_s=st["transfer_ms"] / 1e3, swap_s=st["swap_ms"] / 1e3,
                            pause_s=st["pause_ms"] / 1e3, transfer_bytes=st["transfer_bytes"],
                            old_world=old.world, new_world=new.world, union_world=len(union),
                            exec_report=st["exec"])
        # atomic_switch (generation.cpp:272-290): routing moves to the new
        # generation; the old store (now RS_DST) is reclaimed in Cleanup.
        self._active, self._shadow, self._plan = new, None, None
        self.last_switch = stats
        self._record(Phase.CLEANUP)
        self.engine.free(RS_DST)
        self._release("shadow_store")
        self._enter_stable_and_pop_queue()
        return stats

    def abort_and_fallback(self, reason: str = "aborted", failed_layer: Optional[int] = None
                           ) -> FallbackOutcome:
        """Fail-stop before commit: the active store is untouched; the shadow
        store is released (generation.cpp:315-340)."""
        out = FallbackOutcome(reason, failed_layer)
        self._drop_shadow()
        if self._phase != Phase.STABLE:
            self._record(Phase.STABLE)
        self.last_fallback = out
        return out

    def shadow_rank_lost(self, rank: int, updated_target: ParallelConfig) -> None:
        """generation.cpp:342-362: restart Prepare with the updated target."""
        if self._phase == Phase.STABLE or self._shadow is None or rank not in self._shadow.ranks:
            return
        self._drop_shadow()
        self._record(Phase.STABLE)
        target = dataclasses.replace(updated_target, gen=self._active.gen + 1)
        bad = R.validate_config(target, self.model)
        if bad:
            raise ValueError("shadow_rank_lost: invalid updated target: " + bad[0])
        self._start_prepare(target)

    # -- internals -----------------------------------------------------------
    def _slots(self, cfg: ParallelConfig) -> List[int]:
        if self._placement is None:
            return [0] * cfg.world
        p = self._placement
        return list(p(cfg)) if callable(p) else list(p)[:cfg.world]

    def _connect(self, which) -> None:
        if self.group is None:
            return
        from .dist import connect
        connect(self.engine, self.group, which)

    def _all_ok(self, ok: bool) -> bool:
        import torch
        import torch.distributed as dist
        t = torch.tensor([0 if ok else 1], dtype=torch.int32)
        dist.all_reduce(t, group=self.group)  # the commit barrier
        return int(t.item()) == 0

    def _start_prepare(self, target: ParallelConfig) -> None:
        self._shadow = target
        self.last_fallback = None
        self._prepare_started = self.now()
        self._record(Phase.PREPARE)

    def _drop_shadow(self) -> None:
        if self._plan is not None or self.engine.configs.get(RS_DST) is not None:
            try:
                self.engine.free(RS_DST)
            except Exception:
                pass
        self._release("shadow_store")
        self._shadow, self._plan = None, None

    def _enter_stable_and_pop_queue(self) -> None:
        self._record(Phase.STABLE)
        if self._queue:  # rebase the queued target onto the new active generation
            target = dataclasses.replace(self._queue.popleft(), gen=self._active.gen + 1)
            if not R.validate_config(target, self.model):
                self._start_prepare(target)

    def _record(self, to: Phase) -> None:
        self.transition_log.append(TransitionRecord(self.now(), self._phase, to, self._active.gen,
                                                    self._shadow.gen if self._shadow else None))
        self._phase = to

    def _allocate(self, what: str, nbytes: int) -> None:
        self.allocation_ledger.append(AllocationRecord(what, int(nbytes)))

    def _release(self, what: str) -> None:
        for a in reversed(self.allocation_ledger):
            if a.what == what and not a.released:
                a.released = True
                return
