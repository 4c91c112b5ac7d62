"""The NCCL send/recv comparator (RS_MODE_XFER).

The paper moves every chunk with NCCL isend/irecv.  Here the
same transport runs between our pack and unpack kernels, on the same chunk
schedule and staging budget as the ring path: per round, the engine packs each
cross-GPU link's chunks into that link's send buffer, NCCL moves the buffers,
the engine unpacks.  It is a measured comparison only -- the product moves
bytes GPU->GPU inside its own kernels (DIRECT / STAGED).

The link buffers are engine-owned device memory; they are exposed to
torch.distributed as uint8 tensors through DLPack (no copy).  With the gloo
backend (CPU tests, two processes on one GPU) the buffers are staged through
host memory.
"""

from __future__ import annotations

import ctypes as C
import time
from typing import List

import torch

_KEEP: List[object] = []  # DLPack structs must outlive the tensors built on them


class _DLDevice(C.Structure):
    _fields_ = [("device_type", C.c_int), ("device_id", C.c_int)]


class _DLDataType(C.Structure):
    _fields_ = [("code", C.c_uint8), ("bits", C.c_uint8), ("lanes", C.c_uint16)]


class _DLTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("device", _DLDevice), ("ndim", C.c_int),
                ("dtype", _DLDataType), ("shape", C.POINTER(C.c_int64)),
                ("strides", C.POINTER(C.c_int64)), ("byte_offset", C.c_uint64)]


_DELETER = C.CFUNCTYPE(None, C.c_void_p)


class _DLManagedTensor(C.Structure):
    _fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", C.c_void_p), ("deleter", _DELETER)]


@_DELETER
def _no_delete(_):  # the engine owns the memory
    return None


def device_bytes(ptr: int, nbytes: int, device: int) -> torch.Tensor:
    """A uint8 CUDA tensor aliasing engine-owned device memory (zero copy)."""
    shape = (C.c_int64 * 1)(nbytes)
    mt = _DLManagedTensor()
    mt.dl_tensor.data = ptr
    mt.dl_tensor.device = _DLDevice(2, device)  # kDLCUDA
    mt.dl_tensor.ndim = 1
    mt.dl_tensor.dtype = _DLDataType(1, 8, 1)  # kDLUInt, 8 bits
    mt.dl_tensor.shape = shape
    mt.dl_tensor.strides = None
    mt.dl_tensor.byte_offset = 0
    mt.manager_ctx = None
    mt.deleter = _no_delete
    _KEEP.append((mt, shape))
    new_capsule = C.pythonapi.PyCapsule_New
    new_capsule.restype = C.py_object
    new_capsule.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
    capsule = new_capsule(C.addressof(mt), b"dltensor", None)
    return torch.utils.dlpack.from_dlpack(capsule)


def run(engine, device: int, rank_of_slot=lambda s: s, host_staging: bool = False, group=None) -> dict:
    """One handoff over torch.distributed point-to-point (NCCL, or gloo with
    host staging).  Returns timing and traffic counters."""
    import torch.distributed as dist
    rounds, ntx, nrx = engine.xfer_info()
    tx = [engine.xfer_link(0, i, rounds) for i in range(ntx)]
    rx = [engine.xfer_link(1, i, rounds) for i in range(nrx)]
    for link in tx + rx:
        link["t"] = device_bytes(link["ptr"], link["nbytes"], device) if link["nbytes"] else None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    engine.xfer_step(0)  # local copies (same-GPU tasks, carryovers)
    moved = 0
    for r in range(rounds):
        engine.xfer_step(1, r)
        ops, stage_in = [], []
        for link in tx:
            n = link["round_bytes"][r]
            if n:
                buf = link["t"][:n]
                ops.append(dist.P2POp(dist.isend, buf.cpu() if host_staging else buf,
                                      rank_of_slot(link["peer_slot"]), group=group))
                moved += n
        for link in rx:
            n = link["round_bytes"][r]
            if n:
                buf = torch.empty(n, dtype=torch.uint8) if host_staging else link["t"][:n]
                ops.append(dist.P2POp(dist.irecv, buf, rank_of_slot(link["peer_slot"]), group=group))
                stage_in.append((link, buf, n))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if host_staging:
            for link, buf, n in stage_in:
                link["t"][:n].copy_(buf)
        torch.cuda.synchronize()
        engine.xfer_step(2, r)
    torch.cuda.synchronize()
    return {"rounds": rounds, "tx_links": ntx, "rx_links": nrx, "bytes_sent": moved,
            "seconds": time.perf_counter() - t0}
