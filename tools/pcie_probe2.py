#!/usr/bin/env python3
"""Host-transfer ceiling vs host buffer size and page size (diagnostic).

For each size: pinned via cudaHostAlloc, and anonymous mmap + MADV_HUGEPAGE
(2 MB transparent huge pages) + cudaHostRegister.  Measures H2D alone, D2H
alone and both concurrently, chunked in 1 GiB copies over the whole buffer.
"""
import ctypes
import json
import mmap
import sys
import time

import torch

libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
libc.munmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
MADV_HUGEPAGE = 14
cudart = torch.cuda.cudart()
GiB = 1 << 30


def host_tensor(nbytes, kind):
    if kind == "hostalloc":
        t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        return t, lambda: None
    p = libc.mmap(None, nbytes, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    if kind == "thp":
        libc.madvise(p, nbytes, MADV_HUGEPAGE)
    ctypes.memset(p, 0, nbytes)  # fault in (huge) pages
    rc = cudart.cudaHostRegister(p, nbytes, 0)
    assert int(rc) == 0, rc
    t = torch.frombuffer((ctypes.c_uint8 * nbytes).from_address(p), dtype=torch.uint8)

    def free():
        cudart.cudaHostUnregister(p)
        libc.munmap(p, nbytes)
    return t, free


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [8, 48]
    dev = torch.empty(8 * GiB, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for gib in sizes:
        for kind in ("hostalloc", "register4k", "thp"):
            n = gib * GiB
            a, fa = host_tensor(n, kind)
            b, fb = host_tensor(n, kind)

            def h2d():
                with torch.cuda.stream(s1):
                    for off in range(0, n, GiB):
                        dev[(off // GiB % 4) * GiB:(off // GiB % 4 + 1) * GiB].copy_(a[off:off + GiB], non_blocking=True)

            def d2h():
                with torch.cuda.stream(s2):
                    for off in range(0, n, GiB):
                        b[off:off + GiB].copy_(dev[(4 + off // GiB % 4) * GiB:(5 + off // GiB % 4) * GiB],
                                               non_blocking=True)

            def timed(fn):
                torch.cuda.synchronize()
                t = time.perf_counter()
                fn()
                torch.cuda.synchronize()
                return time.perf_counter() - t
            timed(h2d)
            r = {"GiB": gib, "kind": kind, "h2d": n / timed(h2d) / 1e9, "d2h": n / timed(d2h) / 1e9}
            t = timed(lambda: (h2d(), d2h()))
            r["both_total"] = 2 * n / t / 1e9
            print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
            del a, b
            fa()
            fb()


if __name__ == "__main__":
    main()
