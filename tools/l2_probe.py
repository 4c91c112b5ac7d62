#!/usr/bin/env python3
"""What the memory system sustains for the STAGED lanes' access shape
(tools/l2_probe.cu: 1-warp CTAs, 2 x 16 KB TMA stages, bulk load -> bulk
store).  Source / destination working sets small (L2-resident) or large
(HBM): L2->L2 is a ring slot written and read back, HBM->L2 a sender, L2->HBM
a receiver.  One JSON line per case; GB/s counts bytes read + written."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_l2_probe.so")


def lib():
    if not os.path.exists(SO):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                        os.path.join(HERE, "l2_probe.cu"), "-o", SO], check=True)
    L = ctypes.CDLL(SO)
    L.l2_probe.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                           ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    return L


def main():
    L = lib()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    MB, GB = 1 << 20, 1 << 30
    big_src = torch.empty(8 * GB, dtype=torch.uint8, device="cuda")
    big_dst = torch.empty(8 * GB, dtype=torch.uint8, device="cuda")
    small = [torch.empty(64 * MB, dtype=torch.uint8, device="cuda") for _ in range(2)]
    big_src.fill_(1)
    cases = [("L2->L2 32+32 MiB", small[0], 32 * MB, small[1], 32 * MB),
             ("L2->L2 16+16 MiB", small[0], 16 * MB, small[1], 16 * MB),
             ("L2->L2 48+48 MiB", small[0], 48 * MB, small[1], 48 * MB),
             ("HBM->L2 (sender shape)", big_src, 8 * GB, small[1], 32 * MB),
             ("L2->HBM (receiver shape)", small[0], 32 * MB, big_dst, 8 * GB),
             ("HBM->HBM", big_src, 8 * GB, big_dst, 8 * GB)]
    items = (16 * GB) // 16384
    for per_sm in (6, 3):
        for name, s, sb, d, db in cases:
            ms = ctypes.c_float(0)
            rc = L.l2_probe(s.data_ptr(), sb, d.data_ptr(), db, items, sms * per_sm, ctypes.byref(ms))
            moved = 2 * items * 16384
            print(json.dumps({"case": name, "ctas_per_sm": per_sm, "rc": rc, "ms": round(ms.value, 3),
                              "GBps_read_plus_write": round(moved / (ms.value / 1e3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    sys.exit(main())
