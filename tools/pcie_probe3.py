#!/usr/bin/env python3
"""Host-transfer ceiling vs number of concurrent streams per direction
(diagnostic): pinned cudaHostAlloc buffers, 256 MiB copies dealt round-robin
over k streams per direction, H2D alone, D2H alone and both together."""
import json
import sys
import time

import torch

GiB = 1 << 30
CH = 256 << 20


def main():
    n = int(sys.argv[1]) * GiB if len(sys.argv) > 1 else 16 * GiB
    a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    b = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(8 * GiB, dtype=torch.uint8, device="cuda")
    for k in (1, 2, 4, 8):
        hs = [torch.cuda.Stream() for _ in range(k)]
        ds = [torch.cuda.Stream() for _ in range(k)]

        def h2d():
            for i, off in enumerate(range(0, n, CH)):
                with torch.cuda.stream(hs[i % k]):
                    d = (off // CH) % 16
                    dev[d * CH:(d + 1) * CH].copy_(a[off:off + CH], non_blocking=True)

        def d2h():
            for i, off in enumerate(range(0, n, CH)):
                with torch.cuda.stream(ds[i % k]):
                    d = 16 + (off // CH) % 16
                    b[off:off + CH].copy_(dev[d * CH:(d + 1) * CH], non_blocking=True)

        def both():
            h2d()
            d2h()

        def timed(fn):
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            return time.perf_counter() - t
        timed(h2d)
        r = {"streams_per_direction": k, "h2d_GBps": n / timed(h2d) / 1e9, "d2h_GBps": n / timed(d2h) / 1e9,
             "both_GBps": 2 * n / timed(both) / 1e9}
        print(json.dumps({x: (round(v, 1) if isinstance(v, float) else v) for x, v in r.items()}), flush=True)


if __name__ == "__main__":
    main()
