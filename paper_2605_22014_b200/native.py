"""ctypes binding of libreshard_b200.so (include/rs_reshard.h).

This is the only way the Python side reaches the product: there is no Python
or CPU fallback for any reshard operation.  A missing library raises at import
of the calling function, never silently degrades.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libreshard_b200.so")

RS_OK, RS_EDOMAIN, RS_EINTEGRITY, RS_ESYSTEM = 0, 1, 2, 3
RS_SRC, RS_DST, RS_COMM = 0, 1, 2
RS_IPC_HANDLE_BYTES = 64
RS_MODE_DIRECT, RS_MODE_STAGED, RS_MODE_XFER = 0, 1, 2
RS_XFER_ASYNC = 16  # rs_xfer_step: enqueue only (rs_reshard.h)
RS_TRAFFIC_RELAY = 1

EXPORTS = [
    "rs_last_error", "rs_version", "rs_validate_config", "rs_view", "rs_view_range", "rs_plan_compute",
    "rs_plan_read", "rs_plan_write", "rs_plan_summary", "rs_plan_verify", "rs_plan_destroy",
    "rs_chunk_bounds", "rs_engine_create", "rs_engine_destroy", "rs_store_layout",
    "rs_store_alloc", "rs_store_bind", "rs_store_ptr", "rs_store_bytes", "rs_store_entries",
    "rs_store_read",
    "rs_store_write", "rs_store_free", "rs_fill_pattern", "rs_verify_pattern", "rs_prepare",
    "rs_run", "rs_execute", "rs_execute_host", "rs_host_alloc", "rs_host_free", "rs_comm_alloc",
    "rs_arena_export", "rs_arena_import", "rs_plan_traffic", "rs_plan_traffic_ex", "rs_xfer_info", "rs_xfer_link",
    "rs_xfer_step", "rs_xfer_stream", "rs_switch", "rs_store_swap", "rs_plan_placement", "rs_comm_alloc_plan", "rs_trace_read",
]


class ReshardError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class DomainError(ReshardError, ValueError):
    pass


class IntegrityError(ReshardError):
    pass


class SystemError_(ReshardError):
    pass


_ERRORS = {RS_EDOMAIN: DomainError, RS_EINTEGRITY: IntegrityError, RS_ESYSTEM: SystemError_}


class Config(C.Structure):
    _fields_ = [("generation_id", C.c_uint64), ("tp", C.c_int32), ("pp", C.c_int32),
                ("dp", C.c_int32), ("num_ranks", C.c_int32), ("ranks", C.POINTER(C.c_int32)),
                ("layer_stage", C.POINTER(C.c_int32)), ("distributed_optimizer", C.c_int32),
                ("dist_opt_bucket_elems", C.c_int32)]


class PlanOptions(C.Structure):
    _fields_ = [("balance_sources", C.c_int32)]


class PlanSummary(C.Structure):
    _fields_ = [("total_bytes", C.c_int64), ("max_link_bytes", C.c_int64),
                ("task_count", C.c_int64), ("remote_bytes", C.c_int64),
                ("local_bytes", C.c_int64), ("carryover_bytes", C.c_int64),
                ("carryover_count", C.c_int64), ("pairs_checked", C.c_int64),
                ("num_tensors", C.c_int32), ("num_layers_with_work", C.c_int32)]


class EngineOptions(C.Structure):
    _fields_ = [("num_devices", C.c_int32), ("device_ids", C.POINTER(C.c_int32)),
                ("staging_bytes", C.c_int64), ("mode", C.c_int32),
                ("slots_per_link", C.c_int32), ("lanes_per_link", C.c_int32),
                ("strict_layers", C.c_int32), ("item_bytes", C.c_int64),
                ("blocks_per_sm", C.c_int32), ("copy_kernel", C.c_int32),
                ("world_slots", C.c_int32), ("first_local_slot", C.c_int32),
                ("spin_limit", C.c_int64), ("fault_inject", C.c_int32),
                ("ring_slot_kib", C.c_int32), ("ring_discard", C.c_int32),
                ("ring_cta_threads", C.c_int32), ("trace", C.c_int32), ("ring_same_slot", C.c_int32),
                ("ring_kernel", C.c_int32), ("ring_stages", C.c_int32), ("relay", C.c_int32)]


class TraceRecord(C.Structure):
    _fields_ = [("lane", C.c_uint32), ("batch", C.c_uint32), ("layer", C.c_uint32), ("role", C.c_uint32),
                ("bytes", C.c_uint64), ("t_begin", C.c_uint64), ("t_end", C.c_uint64)]


class PlacementOptions(C.Structure):
    _fields_ = [("nvlink_gbs", C.c_double), ("hbm_gbs", C.c_double), ("exhaustive_limit", C.c_int64),
                ("balance_sources", C.c_int32), ("reserved", C.c_int32)]


class PlacementResult(C.Structure):
    _fields_ = [("roofline_ms", C.c_double), ("given_roofline_ms", C.c_double),
                ("remote_bytes", C.c_int64), ("local_bytes", C.c_int64), ("carryover_bytes", C.c_int64),
                ("max_link_bytes", C.c_int64), ("given_remote_bytes", C.c_int64),
                ("given_local_bytes", C.c_int64), ("given_carryover_bytes", C.c_int64),
                ("given_max_link_bytes", C.c_int64), ("evaluated", C.c_int64), ("exhaustive", C.c_int32),
                ("reserved", C.c_int32)]


class ExecReport(C.Structure):
    _fields_ = [("ok", C.c_int32), ("failed_layer", C.c_int32),
                ("peak_staging_bytes", C.c_int64), ("bytes_moved", C.c_int64),
                ("local_copy_bytes", C.c_int64), ("carryover_bytes", C.c_int64),
                ("layers_processed", C.c_int32), ("kernel_launches", C.c_int32),
                ("device_ms", C.c_double), ("host_ms", C.c_double), ("error", C.c_char * 512),
                ("copy_kernel", C.c_int32), ("ring_same_slot", C.c_int32),
                ("ring_kernel", C.c_int32), ("relay_routes", C.c_int32)]

    def as_dict(self) -> dict:
        return {"ok": bool(self.ok),
                "failed_layer": None if self.failed_layer < 0 else int(self.failed_layer),
                "peak_staging_bytes": int(self.peak_staging_bytes),
                "bytes_moved": int(self.bytes_moved),
                "local_copy_bytes": int(self.local_copy_bytes),
                "carryover_bytes": int(self.carryover_bytes),
                "layers_processed": int(self.layers_processed),
                "kernel_launches": int(self.kernel_launches),
                "device_ms": float(self.device_ms), "host_ms": float(self.host_ms),
                "error": self.error.decode(),
                "copy_kernel": int(self.copy_kernel), "ring_same_slot": int(self.ring_same_slot),
                "ring_kernel": int(self.ring_kernel), "relay_routes": int(self.relay_routes)}


class SwitchStats(C.Structure):
    _fields_ = [("drain_ms", C.c_double), ("transfer_ms", C.c_double),
                ("swap_ms", C.c_double), ("pause_ms", C.c_double),
                ("transfer_bytes", C.c_int64), ("swapped", C.c_int32),
                ("reserved", C.c_int32), ("exec", ExecReport)]

    def as_dict(self) -> dict:
        return {"drain_ms": float(self.drain_ms), "transfer_ms": float(self.transfer_ms),
                "swap_ms": float(self.swap_ms), "pause_ms": float(self.pause_ms),
                "transfer_bytes": int(self.transfer_bytes), "swapped": bool(self.swapped),
                "exec": self.exec.as_dict()}


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(make -C paper_2605_22014_b200/csrc); there is no fallback path")
        L = C.CDLL(LIB_PATH)
        P, VP, I32, I64, U64, SZ = C.POINTER, C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t
        L.rs_last_error.restype = C.c_char_p
        L.rs_version.restype = C.c_char_p
        L.rs_validate_config.argtypes = [C.c_char_p, P(Config), C.c_char_p, SZ, P(SZ), P(I32)]
        L.rs_view.argtypes = [C.c_char_p, P(Config), I32, I32, P(I64), P(I64), P(I32)]
        L.rs_view_range.argtypes = [C.c_char_p, P(Config), I32, I32, P(I64), P(I64), P(I32)]
        L.rs_plan_compute.argtypes = [C.c_char_p, P(Config), P(Config), P(PlanOptions), P(VP)]
        L.rs_plan_read.argtypes = [C.c_char_p, C.c_char_p, P(VP)]
        L.rs_plan_write.argtypes = [VP, C.c_char_p, SZ, P(SZ)]
        L.rs_plan_summary.argtypes = [VP, P(PlanSummary)]
        L.rs_plan_verify.argtypes = [VP, P(Config), P(Config), C.c_char_p, SZ, P(SZ), P(I32)]
        L.rs_plan_destroy.argtypes = [VP]
        L.rs_plan_destroy.restype = None
        L.rs_chunk_bounds.argtypes = [I32, P(I64), P(I64), I64, I64, P(I64), P(I64), I64, P(I64)]
        L.rs_engine_create.argtypes = [P(EngineOptions), P(VP)]
        L.rs_engine_destroy.argtypes = [VP]
        L.rs_engine_destroy.restype = None
        L.rs_store_layout.argtypes = [VP, I32, C.c_char_p, P(Config), P(I32)]
        L.rs_store_alloc.argtypes = [VP, I32]
        L.rs_store_free.argtypes = [VP, I32]
        L.rs_store_bind.argtypes = [VP, I32, I32, I32, VP, I64]
        L.rs_store_ptr.argtypes = [VP, I32, I32, I32, P(VP), P(I64)]
        L.rs_store_bytes.argtypes = [VP, I32, P(I64)]
        L.rs_store_entries.argtypes = [VP, I32, P(I32), P(I32), P(I64), I64, P(I64)]
        L.rs_store_read.argtypes = [VP, I32, I32, I32, I64, I64, VP]
        L.rs_store_write.argtypes = [VP, I32, I32, I32, I64, I64, VP]
        L.rs_fill_pattern.argtypes = [VP, I32, U64]
        L.rs_verify_pattern.argtypes = [VP, I32, U64, P(I64), P(I64)]
        L.rs_prepare.argtypes = [VP, VP]
        L.rs_run.argtypes = [VP, P(ExecReport)]
        L.rs_execute.argtypes = [VP, VP, P(ExecReport)]
        L.rs_execute_host.argtypes = [VP, VP, P(VP), P(VP), I32, P(ExecReport)]
        L.rs_host_alloc.argtypes = [SZ, P(VP)]
        L.rs_host_free.argtypes = [VP]
        L.rs_comm_alloc.argtypes = [VP]
        L.rs_comm_alloc_plan.argtypes = [VP, VP]
        L.rs_trace_read.argtypes = [VP, I32, P(TraceRecord), I64, P(I64)]
        L.rs_arena_export.argtypes = [VP, I32, I32, VP, P(I64)]
        L.rs_arena_import.argtypes = [VP, I32, I32, VP, I64]
        L.rs_plan_traffic.argtypes = [VP, P(Config), P(I32), P(Config), P(I32), I32, P(I64)]
        L.rs_plan_traffic_ex.argtypes = [VP, P(Config), P(I32), P(Config), P(I32), I32, I32, P(I64)]
        L.rs_xfer_info.argtypes = [VP, P(I32), P(I32), P(I32)]
        L.rs_xfer_link.argtypes = [VP, I32, I32, P(I32), P(I32), P(I32), P(VP), P(I64), P(I64)]
        L.rs_xfer_step.argtypes = [VP, I32, I32]
        L.rs_xfer_stream.argtypes = [VP, P(VP)]
        L.rs_switch.argtypes = [VP, VP, P(VP), I32, P(SwitchStats)]
        L.rs_store_swap.argtypes = [VP]
        L.rs_plan_placement.argtypes = [C.c_char_p, P(Config), P(Config), P(I32), I32, P(PlacementOptions),
                                        P(I32), P(PlacementResult)]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != RS_OK:
        msg = lib().rs_last_error().decode()
        raise _ERRORS.get(rc, ReshardError)(rc, msg)


def config_struct(cfg, num_layers: int) -> Config:
    ranks = (C.c_int32 * max(1, len(cfg.ranks)))(*cfg.ranks)
    stage = None
    if cfg.layer_stage is not None:
        stage = (C.c_int32 * max(1, num_layers))(*cfg.layer_stage)
    s = Config(cfg.gen, cfg.tp, cfg.pp, cfg.dp, len(cfg.ranks), ranks,
               C.cast(stage, C.POINTER(C.c_int32)) if stage is not None else None,
               int(getattr(cfg, "dist_opt", 0)), int(getattr(cfg, "bucket_elems", 0)))
    s._keep = (ranks, stage)
    return s
