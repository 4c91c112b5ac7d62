"""One process per GPU: control plane over torch.distributed (gloo, world 2).

* CPU: every rank computes the byte-identical plan, and the per-slot traffic
  (egress / ingress / intra-GPU / carryover) partitions it exactly.
* GPU: two processes on one B200, each driving one device slot; peer arenas
  mapped with CUDA IPC; DIRECT and STAGED handoffs across the process
  boundary, destination bytes checked against the analytic pattern.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(case, world=2, timeout=600):
    port = str(free_port())
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_workers.py"), case, str(r),
                               str(world), port], stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        assert p.returncode == 0, e[-3000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    return sorted(outs, key=lambda d: d["rank"])


def test_plan_agreement_and_partition():
    outs = launch("partition")
    for case in ("c1", "c2", "c5b"):
        rows = [o["result"][case] for o in outs]
        assert all(r["agree"] for r in rows)
        r = rows[0]
        assert r["egress_total"] == r["ingress_total"]
        assert r["egress_total"] + r["intra_total"] == r["plan_total"]
        assert r["carry_total"] == r["plan_carry"]
        # each rank's own share is the same row every rank computed for it
        assert [o["result"][case]["mine"] for o in outs] == [rows[0]["mine"], rows[1]["mine"]]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["direct", "direct-tma", "staged", "staged-strict", "xfer", "staged-a16",
                                  "staged-strict-a16", "staged-a16-auto", "staged-strict-a16-auto"])
def test_two_processes_one_gpu_ipc(mode):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    outs = launch(mode, timeout=900)
    for o in outs:
        assert o["result"]["ok"], o
        assert o["result"]["mismatches"] == 0, o


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["direct-a16", "staged-a16", "staged-strict-a16"])
def test_eight_processes_one_gpu_ipc(mode):
    """The 8-GPU process layout on one B200: eight processes, one slot each,
    every peer arena CUDA-IPC mapped into every process, the new ranks
    shifted one slot so every cross-rank byte crosses a process boundary
    (DIRECT peer stores incl. paired DP broadcasts, STAGED stream lanes with
    .sys handshakes, strict layer barriers over eight slots' done flags)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    outs = launch(mode, world=8, timeout=900)
    for o in outs:
        assert o["result"]["ok"], o
        assert o["result"]["mismatches"] == 0, o


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_two_processes_live_handoff_chain(mode):
    """Runtime hook across processes: three generations through LiveHandoff
    (shadow arenas exchanged in Prepare, commit barrier after each switch);
    every active store verifies against the analytic pattern."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    outs = launch("handoff-" + mode, timeout=900)
    for o in outs:
        assert o["result"]["ok"], o
        assert o["result"]["mismatches"] == 0, o
        assert len(o["result"]["pauses"]) == 3
