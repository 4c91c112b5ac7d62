#!/usr/bin/env python3
"""Lane-pair shape probe (tools/pair_probe.cu): payload GB/s of a sender
(HBM -> slot) + receiver (slot -> HBM) per CTA, receiver as a TMA warp
(mode 0, 64 KB smem per CTA) or a register warp (mode 1, 32 KB smem)."""
import ctypes
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_pair_probe.so")


def main():
    if not os.path.exists(SO):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                        os.path.join(HERE, "pair_probe.cu"), "-o", SO], check=True)
    L = ctypes.CDLL(SO)
    L.pair_probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                             ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                             ctypes.POINTER(ctypes.c_float)]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    GB, MB = 1 << 30, 1 << 20
    src = torch.empty(8 * GB, dtype=torch.uint8, device="cuda")
    dst = torch.empty(8 * GB, dtype=torch.uint8, device="cuda")
    slots = torch.empty(64 * MB, dtype=torch.uint8, device="cuda")
    items = (16 * GB) // 16384
    for mode in (0, 1):
        occ = L.pair_probe_occupancy(mode)
        for per_sm in sorted({occ, max(1, occ // 2)}):
            for sb in (32 * MB, 64 * MB):
                ms = ctypes.c_float(0)
                rc = L.pair_probe(mode, src.data_ptr(), 8 * GB, slots.data_ptr(), sb, dst.data_ptr(), 8 * GB, items,
                                  sms * per_sm, ctypes.byref(ms))
                print(json.dumps({"mode": ["tma+tma", "tma+registers"][mode], "ctas_per_sm": per_sm,
                                  "slot_MiB": sb >> 20, "rc": rc, "ms": round(ms.value, 3),
                                  "payload_GBps": round(items * 16384 / (ms.value / 1e3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
