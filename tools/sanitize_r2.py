#!/usr/bin/env python3
"""Small cases for compute-sanitizer over the round-2 kernels: TMA stream
lanes (1-3 stages), strict layer barriers with the local
copies inside the lane launch, flat-bucket shards (DIRECT + STAGED).  Each
case checks its bytes against the C oracle; run under
`compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck}`."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle.pyoracle import Oracle  # noqa: E402
from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.native import RS_DST, RS_SRC  # noqa: E402

SEED = 42


def case(sp, co, cn, mode, **kw):
    eng = R.Engine([0], staging_bytes=1 << 20, mode=mode, **kw)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, SEED)
    eng.fill_pattern(RS_DST, 7)
    plan = R.compute_transfer_plan(co, cn, sp)
    for _ in range(2):
        rep = R.execute_plan(plan, eng)
        assert rep["ok"], rep
    _, want = Oracle("c").execute(sp, co, cn, plan.text(), SEED, 1 << 20)
    for (ti, rank), arr in want.entries.items():
        assert np.array_equal(eng.read(RS_DST, rank, ti), arr), (ti, rank)
    out = rep.get("ring_kernel")
    eng.close()
    return out


def main():
    sp = specs.llama("llama-mini-a16", 2)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 1)
    for stages in (2, 1, 3):
        print("stream lanes", stages, case(sp, co, cn, "staged", ring_stages=stages, lanes_per_link=2, ring_slot_kib=16))
    print("strict stream", case(sp, co, cn, "staged", strict_layers=True, lanes_per_link=2, ring_slot_kib=16))
    zp = specs.llama("llama-mini-a16", 2, zero=True)
    zo = dataclasses.replace(specs.iota_config(1, 2, 2, 2), dist_opt=2, bucket_elems=60_000)
    zn = dataclasses.replace(specs.iota_config(2, 4, 1, 2), dist_opt=2, bucket_elems=150_000)
    for mode in ("direct", "staged"):
        print("flat buckets", mode, case(zp, zo, zn, mode, lanes_per_link=2))
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
