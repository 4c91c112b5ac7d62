#!/usr/bin/env python3
"""Live handoff at full Llama-2-7B training-state size on one B200.

A chain of resize events through LiveHandoff (the GenerationMachine lifecycle,
proj/src/generation.cpp) with real device stores: every event is Prepare
(plan + verify + shadow store + descriptor compile, overlappable with
training) then Switch = drain (the reshard stream waits for a "training"
stream's iteration-boundary event) + transfer (the plan on the device) + swap
(store roles exchange), all device-timed by rs_switch.  The paper reports a
2-6 s live pause per event for 1.7B-30B models on A800s and
~2 s of state transfer for 14B; this prints the same
quantities per event.  After the chain the active store is checked against
the analytic pattern (every byte of the 94 GB state).  One JSON line per
event, then a summary line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_22014_b200 import reshard as R  # noqa: E402
from paper_2605_22014_b200 import specs  # noqa: E402
from paper_2605_22014_b200.handoff import LiveHandoff  # noqa: E402
from paper_2605_22014_b200.native import RS_SRC  # noqa: E402

SEED = 42
# TP/PP/DP shapes of the chain (8 -> 4 -> 8 -> 8 -> 4 ranks): scale-in (C2),
# scale-out (C5), a pure TP<->PP reshape, and a DP scale-in
CHAIN = [(4, 2, 1), (2, 2, 1), (4, 2, 1), (2, 4, 1), (2, 2, 1)]


def main():
    mode = os.environ.get("RS_HANDOFF_MODE", "direct")
    train_ms = float(os.environ.get("RS_HANDOFF_TRAIN_MS", "50"))
    model = specs.llama("llama2-7b")
    eng = R.Engine([0], staging_bytes=1 << 30, mode=mode)
    h = LiveHandoff(eng, model, specs.iota_config(1, *CHAIN[0]))
    t = time.perf_counter()
    eng.fill_pattern(RS_SRC, SEED)
    torch.cuda.synchronize()
    fill_s = time.perf_counter() - t
    train = torch.cuda.Stream()
    rows = []
    for gen, shape in enumerate(CHAIN[1:], start=2):
        target = specs.iota_config(gen, *shape)
        h.trigger_resize(target)
        t = time.perf_counter()
        h.prepare()
        prep_s = time.perf_counter() - t
        # an iteration of "training" still in flight when the switch is requested
        with torch.cuda.stream(train):
            torch.cuda._sleep(int(train_ms * 1e6 * 1.9))  # ~1.9 GHz SM clock
            boundary = torch.cuda.Event()
            boundary.record(train)
        st = h.switch(drain_events=[boundary.cuda_event])
        row = {"event": gen - 1, "from": "TP%dPP%dDP%d" % CHAIN[gen - 2], "to": "TP%dPP%dDP%d" % shape,
               "transfer_GB": round(st.transfer_bytes / 1e9, 3), "prepare_s": round(prep_s, 3),
               "drain_ms": round(st.drain_s * 1e3, 3), "transfer_ms": round(st.transfer_s * 1e3, 3),
               "swap_ms": round(st.swap_s * 1e3, 4), "pause_ms": round(st.pause_s * 1e3, 3),
               "pause_minus_drain_ms": round((st.pause_s - st.drain_s) * 1e3, 3),
               "reshard_GBps": round(st.transfer_bytes / st.transfer_s / 1e9, 1), "ok": st.exec_report["ok"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
    bad = eng.verify_pattern(RS_SRC, SEED)[0]
    print(json.dumps({"summary": True, "model": "Llama-2-7B bf16 params + fp32 master/m/v (94.3 GB state)",
                      "mode": mode, "events": len(rows), "state_fill_s": round(fill_s, 2),
                      "mean_transfer_ms": round(sum(r["transfer_ms"] for r in rows) / len(rows), 3),
                      "max_pause_minus_drain_ms": max(r["pause_minus_drain_ms"] for r in rows),
                      "simulated_training_ms": train_ms, "final_state_mismatches": bad,
                      "paper_live_pause_s": "2-6 (PAPER.md:433, A800 PCIe/IB)"}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
