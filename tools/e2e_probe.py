#!/usr/bin/env python3
"""Where does the host-store (e2e) time go?  Diagnostic only.

Times, on the full C2 stores: all source entries H2D alone, all destination
entries D2H alone, both concurrently (two streams, per-entry copies), and
rs_execute_host, using the same pinned host buffers.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402

import ctypes  # noqa: E402

cudart = None
for cand in ("libcudart.so.12", "libcudart.so"):
    try:
        cudart = ctypes.CDLL(cand)
        break
    except OSError:
        pass
if cudart is None:
    import glob
    for p in glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*")):
        cudart = ctypes.CDLL(p)
        break
cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]


def main():
    sp, co, cn = specs.baseline_case("c2")
    plan = R.compute_transfer_plan(co, cn, sp)
    eng = R.Engine([0], staging_bytes=1 << 30)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 42)
    eng.prepare(plan)
    src = eng.entries(RS_SRC)
    dst = eng.entries(RS_DST)
    h2d = sum(n for *_, n in src)
    d2h = sum(n for *_, n in dst)
    hs = R.PinnedBuffer(h2d)
    win = R.PinnedBuffer(4 << 30)
    big = R.PinnedBuffer(d2h) if len(sys.argv) > 1 and sys.argv[1] == "bigdst" else None
    sp_, dp_ = [], []
    off = 0
    for ti, r, n in src:
        sp_.append((hs.ptr + off, eng.ptr(RS_SRC, r, ti)[0], n))
        eng.read_to(RS_SRC, r, ti, hs.ptr + off, n)
        off += n
    woff = 0
    doff = 0
    for ti, r, n in dst:
        if big is not None:
            dp_.append((big.ptr + doff, eng.ptr(RS_DST, r, ti)[0], n))
            doff += n
            continue
        if woff + n > win.nbytes:
            woff = 0
        dp_.append((win.ptr + woff, eng.ptr(RS_DST, r, ti)[0], n))
        woff += (n + 255) // 256 * 256
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run_h2d(stream):
        for h, d, n in sp_:
            cudart.cudaMemcpyAsync(ctypes.c_void_p(d), ctypes.c_void_p(h), n, 1, ctypes.c_void_p(stream.cuda_stream))

    def run_d2h(stream):
        for h, d, n in dp_:
            cudart.cudaMemcpyAsync(ctypes.c_void_p(h), ctypes.c_void_p(d), n, 2, ctypes.c_void_p(stream.cuda_stream))

    def timed(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t

    out = {"h2d_bytes": h2d, "d2h_bytes": d2h, "dst_target": "94GB pinned" if big else "4GiB window"}
    out["h2d_only_s"] = timed(lambda: run_h2d(s1))
    out["d2h_only_s"] = timed(lambda: run_d2h(s2))
    out["both_s"] = timed(lambda: (run_h2d(s1), run_d2h(s2)))
    srcp = [h for h, _, _ in sp_]
    dstp = [h for h, _, _ in dp_]
    out["execute_host_s"] = [round(timed(lambda: eng.execute_host(plan, srcp, dstp)), 3) for _ in range(2)]
    out["verify_mismatches"] = eng.verify_pattern(RS_DST, 42)[0]
    out["h2d_GBps"] = h2d / out["h2d_only_s"] / 1e9
    out["d2h_GBps"] = d2h / out["d2h_only_s"] / 1e9
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)


if __name__ == "__main__":
    main()
