"""ctypes front end for the two CPU oracles.  TEST INFRASTRUCTURE ONLY.

* ``Oracle("c")``   -- ``oracle/liboracle.so``: our C restatement (oracle.c).
* ``Oracle("ref")`` -- ``oracle/_ref/libreshard_ref.so``: the unmodified reference
  sources behind ``ref_harness.cpp``.

Both expose identical entry points, so every test can run against either and
the restatement is pinned against the reference on the same inputs.  Only
tests/, ``__graft_entry__.smoke()`` and bench.py's CPU arm import this module.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {"c": os.path.join(HERE, "liboracle.so"),
        "ref": os.path.join(HERE, "_ref", "libreshard_ref.so")}
PREFIX = {"c": "orc_", "ref": "ref_"}


class OracleError(RuntimeError):
    pass


class _Config(C.Structure):
    _fields_ = [("gen", C.c_uint64), ("tp", C.c_int32), ("pp", C.c_int32), ("dp", C.c_int32),
                ("nranks", C.c_int32), ("ranks", C.POINTER(C.c_int32)),
                ("layer_stage", C.POINTER(C.c_int32)), ("distributed_optimizer", C.c_int32),
                ("bucket_elems", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("ok", C.c_int32), ("failed_layer", C.c_int32),
                ("peak_staging_bytes", C.c_int64), ("bytes_moved", C.c_int64),
                ("local_copy_bytes", C.c_int64), ("layers_processed", C.c_int32),
                ("pad", C.c_int32), ("seconds", C.c_double), ("error", C.c_char * 512)]

    def as_dict(self) -> dict:
        return {"ok": bool(self.ok),
                "failed_layer": None if self.failed_layer < 0 else int(self.failed_layer),
                "peak_staging_bytes": int(self.peak_staging_bytes),
                "bytes_moved": int(self.bytes_moved),
                "local_copy_bytes": int(self.local_copy_bytes),
                "layers_processed": int(self.layers_processed),
                "error": self.error.decode(), "seconds": float(self.seconds)}


def build(kind: str = "all") -> None:
    subprocess.run(["make", "-s", "-C", HERE] + ([] if kind == "all" else
                   ["liboracle.so" if kind == "c" else "ref"]), check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def config_struct(cfg, num_layers: int):
    ranks = (C.c_int32 * max(1, len(cfg.ranks)))(*cfg.ranks)
    stage = None
    if cfg.layer_stage is not None:
        stage = (C.c_int32 * max(1, num_layers))(*cfg.layer_stage)
    s = _Config(cfg.gen, cfg.tp, cfg.pp, cfg.dp, len(cfg.ranks), ranks,
                C.cast(stage, C.POINTER(C.c_int32)) if stage is not None else None,
                int(getattr(cfg, "dist_opt", 0)), int(getattr(cfg, "bucket_elems", 0)))
    s._keep = (ranks, stage)
    return s


class Store:
    """Host shard store: ``entries[(ti, rank)]`` -> uint8 array (zero-copy)."""

    def __init__(self, lib, prefix: str, handle, num_tensors: int):
        self._lib, self._p, self.h = lib, prefix, handle
        self.entries: Dict[Tuple[int, int], np.ndarray] = {}
        count = getattr(lib, prefix + "store_count")
        entry = getattr(lib, prefix + "store_entry")
        for ti in range(num_tensors):
            for k in range(count(handle, ti)):
                rank = C.c_int(); ptr = C.POINTER(C.c_uint8)(); n = C.c_int64()
                entry(handle, ti, k, C.byref(rank), C.byref(ptr), C.byref(n))
                arr = (np.ctypeslib.as_array(ptr, shape=(n.value,)) if n.value
                       else np.zeros(0, np.uint8))
                self.entries[(ti, rank.value)] = arr

    def __del__(self):
        try:
            getattr(self._lib, self._p + "store_free")(self.h)
        except Exception:
            pass


class Oracle:
    def __init__(self, kind: str = "c"):
        if not available(kind):
            raise OracleError(f"oracle library missing: {LIBS[kind]} (run make -C oracle)")
        self.kind, self.p = kind, PREFIX[kind]
        lib = C.CDLL(LIBS[kind])
        cp = C.POINTER(C.c_char_p)
        f = lambda n: getattr(lib, self.p + n)
        f("plan_text").argtypes = [C.c_char_p, C.POINTER(_Config), C.POINTER(_Config), C.c_int,
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
        f("verify_plan").argtypes = [C.c_char_p, C.POINTER(_Config), C.POINTER(_Config), C.c_char_p,
                                     C.POINTER(C.c_void_p)]
        f("execute").restype = C.c_void_p
        f("execute").argtypes = [C.c_char_p, C.POINTER(_Config), C.POINTER(_Config), C.c_char_p,
                                 C.c_uint64, C.c_int64, C.POINTER(Report)]
        f("store_pattern").restype = C.c_void_p
        f("store_pattern").argtypes = [C.c_char_p, C.POINTER(_Config), C.c_uint64, C.c_int]
        f("store_count").argtypes = [C.c_void_p, C.c_int]
        f("store_entry").argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int),
                                     C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_int64)]
        f("store_free").argtypes = [C.c_void_p]
        f("free").argtypes = [C.c_void_p]
        f("pattern_byte").restype = C.c_uint8
        f("pattern_byte").argtypes = [C.c_uint32, C.c_int64, C.c_int64, C.c_uint64]
        if kind == "c":
            lib.orc_chunk_bounds.argtypes = [C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                             C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                                             C.POINTER(C.c_int64), C.c_int64,
                                             C.POINTER(C.c_int64), C.POINTER(C.c_void_p)]
            lib.orc_slice_local.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64), C.c_int64, C.c_void_p,
                                            C.POINTER(C.c_void_p)]
        self.lib = lib

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _take(self, ptr: C.c_void_p) -> str:
        s = C.string_at(ptr.value).decode() if ptr.value else ""
        self._fn("free")(ptr)
        return s

    def plan_text(self, spec, c_old, c_new, balance: bool = False) -> Tuple[str, int]:
        out = C.c_void_p(); pairs = C.c_int64(0)
        rc = self._fn("plan_text")(spec.to_text().encode(), config_struct(c_old, spec.num_layers),
                                   config_struct(c_new, spec.num_layers), int(balance),
                                   C.byref(out), C.byref(pairs))
        text = self._take(out)
        if rc:
            raise OracleError(text)
        return text, pairs.value

    def verify_plan(self, spec, c_old, c_new, plan_text: str) -> List[str]:
        out = C.c_void_p()
        rc = self._fn("verify_plan")(spec.to_text().encode(), config_struct(c_old, spec.num_layers),
                                     config_struct(c_new, spec.num_layers), plan_text.encode(),
                                     C.byref(out))
        text = self._take(out)
        if rc:
            raise OracleError(text)
        return [l for l in text.split("\n") if l]

    def execute(self, spec, c_old, c_new, plan_text: str, seed: int, staging: int):
        rep = Report()
        h = self._fn("execute")(spec.to_text().encode(), config_struct(c_old, spec.num_layers),
                                config_struct(c_new, spec.num_layers), plan_text.encode(),
                                seed, staging, C.byref(rep))
        if not h:
            raise OracleError(rep.error.decode())
        return rep.as_dict(), Store(self.lib, self.p, h, len(spec.tensors))

    def store_pattern(self, spec, cfg, seed: int, fill: bool = True) -> Store:
        h = self._fn("store_pattern")(spec.to_text().encode(), config_struct(cfg, spec.num_layers),
                                      seed, int(fill))
        if not h:
            raise OracleError("store_pattern failed")
        return Store(self.lib, self.p, h, len(spec.tensors))

    def pattern_byte(self, ti: int, element: int, b: int, seed: int) -> int:
        return int(self._fn("pattern_byte")(ti, element, b, seed))

    # -- C-oracle-only helpers -------------------------------------------------
    def chunk_bounds(self, lo, hi, max_bytes: int, bpe: int):
        nd = len(lo)
        L = (C.c_int64 * nd)(*lo); H = (C.c_int64 * nd)(*hi)
        cap = 1 << 16
        olo = (C.c_int64 * (cap * nd))(); ohi = (C.c_int64 * (cap * nd))()
        cnt = C.c_int64(); err = C.c_void_p()
        rc = self.lib.orc_chunk_bounds(nd, L, H, max_bytes, bpe, olo, ohi, cap, C.byref(cnt),
                                       C.byref(err))
        if rc:
            raise OracleError(self._take(err))
        return [([olo[i * nd + k] for k in range(nd)], [ohi[i * nd + k] for k in range(nd)])
                for i in range(min(cnt.value, cap))]

    def slice_local(self, buf: np.ndarray, owner_lo, owner_hi, lo, hi, bpe: int) -> np.ndarray:
        nd = len(lo)
        n = int(np.prod([h - l for l, h in zip(lo, hi)])) * bpe
        out = np.zeros(max(n, 1), np.uint8)
        arr = lambda v: (C.c_int64 * nd)(*v)
        err = C.c_void_p()
        b = np.ascontiguousarray(buf, dtype=np.uint8)
        rc = self.lib.orc_slice_local(b.ctypes.data, b.size, nd, arr(owner_lo), arr(owner_hi),
                                      arr(lo), arr(hi), bpe, out.ctypes.data, C.byref(err))
        if rc:
            raise OracleError(self._take(err))
        return out[:n]

    # -- reference-only: the timed CPU arm -------------------------------------
    def bench(self, spec, c_old, c_new, seed: int, fill_threads: int = 1) -> "RefBench":
        return RefBench(self, spec, c_old, c_new, seed, fill_threads)


class RefBench:
    """The reference's own execute_plan, planned and filled once, timed per step."""

    def __init__(self, orc: Oracle, spec, c_old, c_new, seed: int, fill_threads: int):
        lib = orc.lib
        lib.ref_bench_setup.restype = C.c_void_p
        lib.ref_bench_setup.argtypes = [C.c_char_p, C.POINTER(_Config), C.POINTER(_Config),
                                        C.c_uint64, C.c_int, C.POINTER(C.c_int64), C.POINTER(Report)]
        lib.ref_bench_step.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.POINTER(Report)]
        lib.ref_bench_check.restype = C.c_int64
        lib.ref_bench_check.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
        lib.ref_bench_free.argtypes = [C.c_void_p]
        self.lib, self.seed = lib, seed
        rep = Report(); nb = C.c_int64()
        self.h = lib.ref_bench_setup(spec.to_text().encode(), config_struct(c_old, spec.num_layers),
                                     config_struct(c_new, spec.num_layers), seed, fill_threads,
                                     C.byref(nb), C.byref(rep))
        if not self.h:
            raise OracleError(rep.error.decode())
        self.plan_bytes = nb.value

    def step(self, staging: int, threads: int) -> dict:
        rep = Report()
        self.lib.ref_bench_step(self.h, staging, threads, C.byref(rep))
        return rep.as_dict()

    def mismatches(self, threads: int) -> int:
        return int(self.lib.ref_bench_check(self.h, self.seed, threads))

    def close(self):
        if self.h:
            self.lib.ref_bench_free(self.h)
            self.h = None

    def __del__(self):
        self.close()
