#!/usr/bin/env python3
"""Per-shard vs coalesced host<->device copies on the full C2 stores
(diagnostic).  Host memory: one pinned mirror of the source arena (~94 GB)
plus a 4 GiB destination window -- bounded well under the 196 GB box.

  per_entry: one cudaMemcpyAsync per shard (what rs_execute_host issues)
  coalesced: one copy per run of consecutive shards (host mirror laid out
             exactly like the device arena, so a layer's shards are one run)
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402

cudart = torch.cuda.cudart()


def main():
    sp, co, cn = specs.baseline_case("c2")
    eng = R.Engine([0], staging_bytes=1 << 30)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    src = [(eng.ptr(RS_SRC, r, ti), n) for ti, r, n in eng.entries(RS_SRC)]
    dst = [(eng.ptr(RS_DST, r, ti), n) for ti, r, n in eng.entries(RS_DST)]
    s_base = min(p for (p, _), _ in src)
    s_end = max(p + n for (p, _), n in src)
    d_base = min(p for (p, _), _ in dst)
    mirror = R.PinnedBuffer(s_end - s_base)
    window = R.PinnedBuffer(4 << 30)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    import glob
    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                  "libcudart.so*")) + ["/usr/local/cuda/lib64/libcudart.so"]
    rt = ctypes.CDLL(libs[0])
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]

    def cpy(dst, src, n, kind, stream):
        rc = rt.cudaMemcpyAsync(dst, src, n, kind, stream)
        assert rc == 0, rc

    def per_entry():
        for (p, _), n in src:
            cpy(p, mirror.ptr + (p - s_base), n, 1, s1.cuda_stream)
        w = 0
        for (p, _), n in dst:
            if w + n > window.nbytes:
                w = 0
            cpy(window.ptr + w, p, n, 2, s2.cuda_stream)
            w += (n + 255) // 256 * 256

    def runs(entries):
        out = []
        for (p, _), n in sorted(entries):
            if out and out[-1][0] + out[-1][1] <= p <= out[-1][0] + out[-1][1] + 256:
                out[-1][1] = p + n - out[-1][0]
            else:
                out.append([p, n])
        return out

    src_runs, dst_runs = runs(src), runs(dst)

    def coalesced(chunk=1 << 30):
        for p, n in src_runs:
            for off in range(0, n, chunk):
                m = min(chunk, n - off)
                cpy(p + off, mirror.ptr + (p + off - s_base), m, 1, s1.cuda_stream)
        w = 0
        for p, n in dst_runs:
            for off in range(0, n, chunk):
                m = min(chunk, n - off)
                if w + m > window.nbytes:
                    w = 0
                cpy(window.ptr + w, p + off, m, 2, s2.cuda_stream)
                w += m

    def timed(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t

    total = sum(n for _, n in src) + sum(n for _, n in dst)
    out = {"copies_per_entry": len(src) + len(dst), "runs": len(src_runs) + len(dst_runs)}
    timed(per_entry)
    out["per_entry_s"] = timed(per_entry)
    timed(coalesced)
    out["coalesced_1GiB_s"] = timed(coalesced)
    out["coalesced_256MiB_s"] = timed(lambda: coalesced(256 << 20))
    for k in list(out):
        if k.endswith("_s"):
            out[k.replace("_s", "_GBps")] = total / out[k] / 1e9
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)
    mirror.free()
    window.free()


if __name__ == "__main__":
    main()
