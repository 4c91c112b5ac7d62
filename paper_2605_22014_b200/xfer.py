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


# --------------------------------------------------------------------------
# NCCL comparator on one GPU.
#
# NCCL refuses two ranks on one device, and torch.distributed refuses
# self-sends, so the 1-GPU comparator talks to libnccl directly: one
# single-rank communicator, every link's round buffer moved with
# ncclSend/ncclRecv to peer 0 (NCCL's self-loop, the path its all-to-all uses
# for the local block).  The job's "GPUs" are virtual slots on the same device:
# one RS_MODE_XFER engine per slot, so every cross-slot chunk is packed by our
# kernel into its link buffer, moved by NCCL into the receiving slot's buffer,
# and unpacked by our kernel -- the paper's pack -> isend/irecv -> unpack
# executor on the engine's chunk schedule and staging
# budget.

class _NcclUniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


class Nccl:
    """Minimal ctypes binding of the NCCL point-to-point API (test/bench only)."""

    UINT8 = 1  # ncclUint8

    def __init__(self, device: int):
        import os
        path = None
        try:
            import nvidia.nccl as _n  # the NCCL torch itself loads
            cand = os.path.join(list(_n.__path__)[0], "lib", "libnccl.so.2")
            path = cand if os.path.exists(cand) else None
        except Exception:
            pass
        self.lib = C.CDLL(path or "libnccl.so.2")
        L = self.lib
        L.ncclCommInitAll.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_int)]
        for f in (L.ncclSend, L.ncclRecv):
            f.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.ncclCommDestroy.argtypes = [C.c_void_p]
        L.ncclGetErrorString.restype = C.c_char_p
        L.ncclGetVersion.argtypes = [C.POINTER(C.c_int)]
        v = C.c_int()
        self._check(L.ncclGetVersion(C.byref(v)), "ncclGetVersion")
        self.version = v.value
        self.comm = C.c_void_p()
        devs = (C.c_int * 1)(device)
        self._check(L.ncclCommInitAll(C.byref(self.comm), 1, devs), "ncclCommInitAll")

    def _check(self, rc: int, what: str):
        if rc != 0:
            raise RuntimeError(f"{what}: {self.lib.ncclGetErrorString(rc).decode()}")

    def group(self, sends, recvs, stream: int):
        """sends/recvs: [(ptr, nbytes)] to / from peer 0, matched in order."""
        L = self.lib
        self._check(L.ncclGroupStart(), "ncclGroupStart")
        for p, n in sends:
            self._check(L.ncclSend(C.c_void_p(p), n, self.UINT8, 0, self.comm, C.c_void_p(stream)), "ncclSend")
        for p, n in recvs:
            self._check(L.ncclRecv(C.c_void_p(p), n, self.UINT8, 0, self.comm, C.c_void_p(stream)), "ncclRecv")
        self._check(L.ncclGroupEnd(), "ncclGroupEnd")

    def close(self):
        if self.comm.value:
            self.lib.ncclCommDestroy(self.comm)
            self.comm = C.c_void_p()


def run_local_slots(engines, nccl: Nccl, device: int, stream_ordered: bool = False) -> dict:
    """One handoff across virtual slots on one GPU: engines[k] drives slot k
    (RS_MODE_XFER, prepared); NCCL moves every link's round buffer.  Send and
    receive lists are both ordered by (src rank, dst rank), so the k-th send
    to peer 0 matches the k-th receive from peer 0.

    stream_ordered: the rounds are enqueued without a host round trip -- each
    engine's pack, the NCCL group and each engine's unpack are ordered by CUDA
    events (the strongest NCCL baseline; the default is the paper's
    host-driven loop)."""
    if stream_ordered:
        return _run_local_slots_events(engines, nccl, device)
    rounds = engines[0].xfer_info()[0]
    tx, rx = [], []
    for e in engines:
        _, ntx, nrx = e.xfer_info()
        tx += [e.xfer_link(0, i, rounds) for i in range(ntx)]
        rx += [e.xfer_link(1, i, rounds) for i in range(nrx)]
    key = lambda l: (l["src_rank"], l["dst_rank"])  # noqa: E731
    tx.sort(key=key)
    rx.sort(key=key)
    assert [key(l) for l in tx] == [key(l) for l in rx], "xfer links do not pair up"
    stream = torch.cuda.current_stream(device)
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for e in engines:
        e.xfer_step(0)
    moved = 0
    for r in range(rounds):
        for e in engines:
            e.xfer_step(1, r)
        sends = [(l["ptr"], l["round_bytes"][r]) for l in tx if l["round_bytes"][r]]
        recvs = [(l["ptr"], l["round_bytes"][r]) for l in rx if l["round_bytes"][r]]
        if sends:
            nccl.group(sends, recvs, stream.cuda_stream)
            stream.synchronize()
        moved += sum(n for _, n in sends)
        for e in engines:
            e.xfer_step(2, r)
    torch.cuda.synchronize(device)
    return {"rounds": rounds, "links": len(tx), "bytes_sent": moved, "seconds": time.perf_counter() - t0}


def _run_local_slots_events(engines, nccl: Nccl, device: int) -> dict:
    rounds = engines[0].xfer_info()[0]
    tx, rx = [], []
    for e in engines:
        _, ntx, nrx = e.xfer_info()
        tx += [e.xfer_link(0, i, rounds) for i in range(ntx)]
        rx += [e.xfer_link(1, i, rounds) for i in range(nrx)]
    key = lambda l: (l["src_rank"], l["dst_rank"])  # noqa: E731
    tx.sort(key=key)
    rx.sort(key=key)
    assert [key(l) for l in tx] == [key(l) for l in rx], "xfer links do not pair up"
    streams = [torch.cuda.ExternalStream(e.xfer_stream(), device=device) for e in engines]
    comm = torch.cuda.Stream(device)
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for e in engines:
        e.xfer_step(0, sync=False)
    moved = 0
    for r in range(rounds):
        sends = [(l["ptr"], l["round_bytes"][r]) for l in tx if l["round_bytes"][r]]
        recvs = [(l["ptr"], l["round_bytes"][r]) for l in rx if l["round_bytes"][r]]
        for e, st in zip(engines, streams):
            e.xfer_step(1, r, sync=False)
            ev = torch.cuda.Event()
            ev.record(st)
            comm.wait_event(ev)
        if sends:
            nccl.group(sends, recvs, comm.cuda_stream)
        done = torch.cuda.Event()
        done.record(comm)
        for e, st in zip(engines, streams):
            st.wait_event(done)  # the round's bytes landed (and its send buffers were read)
            e.xfer_step(2, r, sync=False)
        moved += sum(n for _, n in sends)
    torch.cuda.synchronize(device)
    return {"rounds": rounds, "links": len(tx), "bytes_sent": moved, "seconds": time.perf_counter() - t0,
            "stream_ordered": True}
