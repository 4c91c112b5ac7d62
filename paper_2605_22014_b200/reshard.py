"""Python mirror of the reference reshard API, over the C ABI.

Names, argument meaning and error behaviour follow the reference
(``proj/include/reshard/{planner,transfer_plan,topology,parallel_config,executor}.hpp``):

* ``compute_transfer_plan(c_old, c_new, model, options, stats)`` raises
  ``ValueError`` (``DomainError``) where the reference throws
  ``std::invalid_argument`` (planner.cpp:60-71);
* ``verify_plan`` returns the violation list (planner.cpp:194-303);
* ``write_plan`` / ``read_plan`` use the reference text format;
* ``execute_plan(plan, engine)`` replaces ``execute_plan(plan, src, dst,
  transport, staging_bytes, bpe)`` (executor.hpp:50-53): the engine holds the
  device shard stores, the transport (DIRECT peer stores or STAGED rings) and
  the staging budget; it returns an ExecutionReport dict with the reference's
  fields (ok, error, failed_layer, peak_staging_bytes, bytes_moved,
  local_copy_bytes, layers_processed) plus timing.

Every call goes to libreshard_b200.so; nothing here computes a plan or moves a
byte in Python.
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable, List, Optional, Sequence

from . import native as N
from .native import DomainError, IntegrityError, ReshardError  # noqa: F401
from .specs import ModelSpec, ParallelConfig


def _text(fn) -> str:
    need = C.c_size_t(0)
    fn(None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    fn(buf, need.value, C.byref(need))
    return buf.value.decode()


class PlanOptions:
    def __init__(self, balance_sources: bool = False):
        self.balance_sources = balance_sources


class PlannerStats:
    pairs_checked: int = 0


class TransferPlan:
    """Owning handle of a native plan."""

    def __init__(self, handle: int, model: ModelSpec):
        self._h = C.c_void_p(handle)
        self.model = model

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                N.lib().rs_plan_destroy(self._h)
            except Exception:
                pass
            self._h = C.c_void_p(0)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def text(self) -> str:
        L = N.lib()
        out = {}

        def call(buf, cap, need):
            N.check(L.rs_plan_write(self._h, buf, cap, need))
        return _text(call)

    def summary(self) -> dict:
        s = N.PlanSummary()
        N.check(N.lib().rs_plan_summary(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in N.PlanSummary._fields_}

    def total_bytes(self) -> int:
        return self.summary()["total_bytes"]


def compute_transfer_plan(c_old: ParallelConfig, c_new: ParallelConfig, model: ModelSpec,
                          options: Optional[PlanOptions] = None,
                          stats: Optional[PlannerStats] = None) -> TransferPlan:
    opts = N.PlanOptions(int(bool(options and options.balance_sources)))
    h = C.c_void_p()
    N.check(N.lib().rs_plan_compute(model.to_text().encode(),
                                    N.config_struct(c_old, model.num_layers),
                                    N.config_struct(c_new, model.num_layers), C.byref(opts),
                                    C.byref(h)))
    plan = TransferPlan(h.value, model)
    if stats is not None:
        stats.pairs_checked = plan.summary()["pairs_checked"]
    return plan


def write_plan(plan: TransferPlan) -> str:
    return plan.text()


def read_plan(text: str, model: ModelSpec) -> TransferPlan:
    h = C.c_void_p()
    N.check(N.lib().rs_plan_read(model.to_text().encode(), text.encode(), C.byref(h)))
    return TransferPlan(h.value, model)


def verify_plan(plan: TransferPlan, c_old: ParallelConfig, c_new: ParallelConfig) -> List[str]:
    L = N.lib()
    n = C.c_int32(0)
    co = N.config_struct(c_old, plan.model.num_layers)
    cn = N.config_struct(c_new, plan.model.num_layers)

    def call(buf, cap, need):
        N.check(L.rs_plan_verify(plan.handle, co, cn, buf, cap, need, C.byref(n)))
    return [l for l in _text(call).split("\n") if l]


def plan_cost_summary(plan: TransferPlan) -> dict:
    s = plan.summary()
    return {"total_bytes": s["total_bytes"], "max_link_bytes": s["max_link_bytes"],
            "task_count": s["task_count"]}


def validate_config(config: ParallelConfig, model: ModelSpec) -> List[str]:
    L = N.lib()
    n = C.c_int32(0)
    cs = N.config_struct(config, model.num_layers)

    def call(buf, cap, need):
        N.check(L.rs_validate_config(model.to_text().encode(), cs, buf, cap, need, C.byref(n)))
    return [l for l in _text(call).split("\n") if l]


def view(model: ModelSpec, tensor_index: int, config: ParallelConfig, rank: int):
    nd = len(model.tensors[tensor_index].shape)
    lo = (C.c_int64 * nd)(); hi = (C.c_int64 * nd)(); present = C.c_int32(0)
    N.check(N.lib().rs_view(model.to_text().encode(), N.config_struct(config, model.num_layers),
                            tensor_index, rank, lo, hi, C.byref(present)))
    return [(lo[i], hi[i]) for i in range(nd)] if present.value else None


def view_range(model: ModelSpec, tensor_index: int, config: ParallelConfig, rank: int):
    """(lo, hi, flat): the element range of the rank's view it holds, row
    major (flat-bucket distributed optimizer); flat False = the whole view."""
    lo = C.c_int64(0); hi = C.c_int64(0); flat = C.c_int32(0)
    N.check(N.lib().rs_view_range(model.to_text().encode(), N.config_struct(config, model.num_layers),
                                  tensor_index, rank, C.byref(lo), C.byref(hi), C.byref(flat)))
    return lo.value, hi.value, bool(flat.value)


def chunk_bounds(lo: Sequence[int], hi: Sequence[int], max_bytes: int, bpe: int):
    nd = len(lo)
    cap = 1 << 16
    olo = (C.c_int64 * (cap * nd))(); ohi = (C.c_int64 * (cap * nd))(); cnt = C.c_int64()
    N.check(N.lib().rs_chunk_bounds(nd, (C.c_int64 * nd)(*lo), (C.c_int64 * nd)(*hi), max_bytes,
                                    bpe, olo, ohi, cap, C.byref(cnt)))
    return [([olo[i * nd + k] for k in range(nd)], [ohi[i * nd + k] for k in range(nd)])
            for i in range(min(cnt.value, cap))]


class Engine:
    """Device engine: stores for C_old (RS_SRC) and C_new (RS_DST) + execution."""

    def __init__(self, devices: Iterable[int] = (0,), staging_bytes: int = 1 << 30,
                 mode: str = "direct", slots_per_link: int = 0, lanes_per_link: int = 0,
                 strict_layers: bool = False, item_bytes: int = 0, blocks_per_sm: int = 0,
                 copy_kernel: int = 0, world_slots: int = 0, first_local_slot: int = 0,
                 spin_limit: int = 0, fault_inject: int = 0, ring_slot_kib: int = 0,
                 ring_discard: int = 0, ring_cta_threads: int = 0, trace: bool = False,
                 ring_same_slot: int = 0, ring_kernel: int = 0, ring_stages: int = 0,
                 relay: bool = False):
        devs = list(devices)
        self._devs = (C.c_int32 * len(devs))(*devs)
        modes = {"direct": N.RS_MODE_DIRECT, "staged": N.RS_MODE_STAGED, "xfer": N.RS_MODE_XFER}
        o = N.EngineOptions(len(devs), self._devs, staging_bytes, modes[mode],
                            slots_per_link, lanes_per_link, int(strict_layers), item_bytes,
                            blocks_per_sm, copy_kernel, world_slots, first_local_slot,
                            spin_limit, fault_inject, ring_slot_kib, ring_discard, ring_cta_threads,
                            int(trace), ring_same_slot, ring_kernel, ring_stages, int(relay))
        h = C.c_void_p()
        N.check(N.lib().rs_engine_create(C.byref(o), C.byref(h)))
        self._h = h
        self.num_devices = len(devs)
        self.world_slots = world_slots or len(devs)
        self.first_local_slot = first_local_slot
        self.mode = mode
        self.models = {}
        self.configs = {}

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            N.lib().rs_engine_destroy(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def layout(self, which: int, model: ModelSpec, config: ParallelConfig,
               rank_device: Optional[Sequence[int]] = None):
        rd = list(rank_device) if rank_device is not None else [0] * config.world
        arr = (C.c_int32 * max(1, len(rd)))(*rd)
        N.check(N.lib().rs_store_layout(self._h, which, model.to_text().encode(),
                                        N.config_struct(config, model.num_layers), arr))
        self.models[which] = model
        self.configs[which] = config

    def alloc(self, which: int):
        N.check(N.lib().rs_store_alloc(self._h, which))

    def free(self, which: int):
        N.check(N.lib().rs_store_free(self._h, which))

    def bind(self, which: int, rank: int, tensor_index: int, dptr: int, nbytes: int):
        N.check(N.lib().rs_store_bind(self._h, which, rank, tensor_index, C.c_void_p(dptr), nbytes))

    def ptr(self, which: int, rank: int, tensor_index: int):
        p = C.c_void_p(); n = C.c_int64()
        N.check(N.lib().rs_store_ptr(self._h, which, rank, tensor_index, C.byref(p), C.byref(n)))
        return p.value, n.value

    def store_bytes(self, which: int) -> int:
        n = C.c_int64()
        N.check(N.lib().rs_store_bytes(self._h, which, C.byref(n)))
        return n.value

    def entries(self, which: int):
        """[(tensor_index, rank, nbytes)] in store order (tensor, ascending rank)."""
        L = N.lib()
        cnt = C.c_int64()
        N.check(L.rs_store_entries(self._h, which, None, None, None, 0, C.byref(cnt)))
        n = cnt.value
        ti = (C.c_int32 * max(1, n))(); rk = (C.c_int32 * max(1, n))(); nb = (C.c_int64 * max(1, n))()
        N.check(L.rs_store_entries(self._h, which, ti, rk, nb, n, C.byref(cnt)))
        return [(ti[i], rk[i], nb[i]) for i in range(n)]

    def read_to(self, which: int, rank: int, tensor_index: int, host_ptr: int, nbytes: int,
                offset: int = 0) -> None:
        N.check(N.lib().rs_store_read(self._h, which, rank, tensor_index, offset, nbytes,
                                      C.c_void_p(host_ptr)))

    def read(self, which: int, rank: int, tensor_index: int, offset: int = 0,
             nbytes: Optional[int] = None):
        import numpy as np
        if nbytes is None:
            nbytes = self.ptr(which, rank, tensor_index)[1] - offset
        out = np.empty(nbytes, np.uint8)
        N.check(N.lib().rs_store_read(self._h, which, rank, tensor_index, offset, nbytes,
                                      out.ctypes.data_as(C.c_void_p)))
        return out

    def write(self, which: int, rank: int, tensor_index: int, offset: int, data) -> None:
        import numpy as np
        a = np.ascontiguousarray(data, dtype=np.uint8)
        N.check(N.lib().rs_store_write(self._h, which, rank, tensor_index, offset, a.size,
                                       a.ctypes.data_as(C.c_void_p)))

    def comm_alloc(self, plan: Optional["TransferPlan"] = None):
        """STAGED staging arena: B per destination rank, or exactly ``plan``'s
        rings (rs_comm_alloc_plan)."""
        if plan is None:
            N.check(N.lib().rs_comm_alloc(self._h))
        else:
            N.check(N.lib().rs_comm_alloc_plan(self._h, plan.handle))

    # -- RS_MODE_XFER (comparator transport) -------------------------------
    def xfer_info(self):
        r, t, x = C.c_int32(), C.c_int32(), C.c_int32()
        N.check(N.lib().rs_xfer_info(self._h, C.byref(r), C.byref(t), C.byref(x)))
        return r.value, t.value, x.value

    def xfer_link(self, direction: int, index: int, rounds: int) -> dict:
        peer, s, d = C.c_int32(), C.c_int32(), C.c_int32()
        buf, nb = C.c_void_p(), C.c_int64()
        rb = (C.c_int64 * max(1, rounds))()
        N.check(N.lib().rs_xfer_link(self._h, direction, index, C.byref(peer), C.byref(s), C.byref(d),
                                     C.byref(buf), C.byref(nb), rb))
        return {"peer_slot": peer.value, "src_rank": s.value, "dst_rank": d.value, "ptr": buf.value or 0,
                "nbytes": nb.value, "round_bytes": [rb[i] for i in range(rounds)]}

    def xfer_step(self, what: int, rnd: int = 0, sync: bool = True):
        N.check(N.lib().rs_xfer_step(self._h, what | (0 if sync else N.RS_XFER_ASYNC), rnd))

    def xfer_stream(self) -> int:
        s = C.c_void_p()
        N.check(N.lib().rs_xfer_stream(self._h, C.byref(s)))
        return s.value or 0

    def trace(self, device: int = 0):
        """STAGED transport trace of the last run (engine built with trace=True):
        [{lane, batch, layer, role, bytes, t_begin, t_end}] (ns, globaltimer)."""
        cnt = C.c_int64()
        N.check(N.lib().rs_trace_read(self._h, device, None, 0, C.byref(cnt)))
        arr = (N.TraceRecord * max(1, cnt.value))()
        N.check(N.lib().rs_trace_read(self._h, device, arr, cnt.value, C.byref(cnt)))
        return [{f: getattr(arr[i], f) for f, _ in N.TraceRecord._fields_} for i in range(cnt.value)]

    def export_arena(self, which: int, slot: int):
        """(64-byte CUDA IPC handle, arena bytes) of a local slot's arena."""
        h = (C.c_char * N.RS_IPC_HANDLE_BYTES)(); n = C.c_int64()
        N.check(N.lib().rs_arena_export(self._h, which, slot, h, C.byref(n)))
        return bytes(h), n.value

    def import_arena(self, which: int, slot: int, handle: bytes, nbytes: int):
        buf = (C.c_char * N.RS_IPC_HANDLE_BYTES).from_buffer_copy(handle)
        N.check(N.lib().rs_arena_import(self._h, which, slot, buf, nbytes))

    def fill_pattern(self, which: int, seed: int):
        N.check(N.lib().rs_fill_pattern(self._h, which, seed))

    def verify_pattern(self, which: int, seed: int):
        bad = C.c_int64(); first = C.c_int64()
        N.check(N.lib().rs_verify_pattern(self._h, which, seed, C.byref(bad), C.byref(first)))
        return bad.value, first.value

    def prepare(self, plan: TransferPlan):
        N.check(N.lib().rs_prepare(self._h, plan.handle))

    def run(self, raise_on_failure: bool = False) -> dict:
        rep = N.ExecReport()
        rc = N.lib().rs_run(self._h, C.byref(rep))
        if rc not in (N.RS_OK, N.RS_EINTEGRITY) or (rc and raise_on_failure):
            N.check(rc)
        return rep.as_dict()

    def execute_host(self, plan: TransferPlan, host_src: Sequence[int], host_dst: Sequence[int],
                     window_layers: int = 0) -> dict:
        """Host shard stores in/out.  window_layers > 0: only that many layers'
        shards are device-resident at a time (bounded device memory); 0: the
        allocated / bound device stores are used."""
        rep = N.ExecReport()
        s = (C.c_void_p * len(host_src))(*host_src)
        d = (C.c_void_p * len(host_dst))(*host_dst)
        rc = N.lib().rs_execute_host(self._h, plan.handle, s, d, window_layers, C.byref(rep))
        if rc not in (N.RS_OK, N.RS_EINTEGRITY):
            N.check(rc)
        return rep.as_dict()

    def switch(self, plan: TransferPlan, drain_events: Optional[Sequence[int]] = None,
               swap: bool = True) -> dict:
        """Switch step of a live handoff (rs_switch): wait for the training
        streams' iteration-boundary events (cudaEvent_t handles, one per local
        device, None entries allowed), run the prepared plan, then swap the
        stores so RS_SRC is the new generation.  Returns SwitchStats as a
        dict; a failed transfer comes back with exec.ok False and no swap."""
        st = N.SwitchStats()
        ev = None
        if drain_events is not None:
            ev = (C.c_void_p * len(drain_events))(*[e or None for e in drain_events])
        rc = N.lib().rs_switch(self._h, plan.handle, ev, int(swap), C.byref(st))
        if rc not in (N.RS_OK, N.RS_EINTEGRITY):
            N.check(rc)
        out = st.as_dict()
        if out["swapped"]:
            self._swap_py()
        return out

    def swap_stores(self):
        N.check(N.lib().rs_store_swap(self._h))
        self._swap_py()

    def _swap_py(self):
        m, c = self.models, self.configs
        self.models = {k ^ 1: v for k, v in m.items() if k in (N.RS_SRC, N.RS_DST)}
        self.configs = {k ^ 1: v for k, v in c.items() if k in (N.RS_SRC, N.RS_DST)}


def plan_traffic(plan: TransferPlan, c_old: ParallelConfig, slot_old: Sequence[int],
                 c_new: ParallelConfig, slot_new: Sequence[int], nslots: int, relay: bool = False):
    """Per-slot [egress, ingress, intra-GPU task bytes, carryover bytes].
    relay=True: relay-chained DP broadcasts leave from the forwarding slot
    (the traffic an Engine(relay=True) STAGED run moves)."""
    out = (C.c_int64 * (4 * nslots))()
    so = (C.c_int32 * len(slot_old))(*slot_old)
    sn = (C.c_int32 * len(slot_new))(*slot_new)
    L = plan.model.num_layers
    N.check(N.lib().rs_plan_traffic_ex(plan.handle, N.config_struct(c_old, L), so, N.config_struct(c_new, L),
                                       sn, nslots, N.RS_TRAFFIC_RELAY if relay else 0, out))
    return [list(out[4 * s:4 * s + 4]) for s in range(nslots)]


def choose_placement(c_old: ParallelConfig, c_new: ParallelConfig, model: ModelSpec,
                     candidates: Optional[Sequence[int]] = None, nvlink_gbs: float = 900.0,
                     hbm_gbs: float = 6552.0, balance_sources: bool = False,
                     exhaustive_limit: int = 0):
    """Placement-aware rank ordering (extension, rs_plan_placement): the rank
    list for c_new's tp/pp/dp shape, drawn from ``candidates`` (default: the
    union of both configs' ranks), that minimises the per-GPU NVLink/HBM
    roofline of the resize.  Returns (ParallelConfig, stats dict)."""
    import dataclasses
    cand = sorted(set(c_old.ranks) | set(c_new.ranks)) if candidates is None else list(candidates)
    arr = (C.c_int32 * max(1, len(cand)))(*cand)
    out = (C.c_int32 * max(1, c_new.world))()
    o = N.PlacementOptions(nvlink_gbs, hbm_gbs, exhaustive_limit, int(balance_sources), 0)
    res = N.PlacementResult()
    L = model.num_layers
    N.check(N.lib().rs_plan_placement(model.to_text().encode(), N.config_struct(c_old, L),
                                      N.config_struct(c_new, L), arr, len(cand), C.byref(o), out,
                                      C.byref(res)))
    stats = {f: getattr(res, f) for f, _ in N.PlacementResult._fields_ if f != "reserved"}
    stats["exhaustive"] = bool(stats["exhaustive"])
    return dataclasses.replace(c_new, ranks=[out[i] for i in range(c_new.world)]), stats


def execute_plan(plan: TransferPlan, engine: Engine) -> dict:
    """Reference ``execute_plan`` on device stores: prepare + run, report dict.

    Integrity failures come back as ``ok=False`` with ``error`` and
    ``failed_layer`` (executor.cpp:210-215); CUDA / argument errors raise.
    """
    engine.prepare(plan)
    return engine.run()


class PinnedBuffer:
    """Page-locked host memory from rs_host_alloc (exact size, no rounding)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        N.check(N.lib().rs_host_alloc(nbytes, C.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes

    def free(self):
        if self.ptr:
            N.check(N.lib().rs_host_free(C.c_void_p(self.ptr)))
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
