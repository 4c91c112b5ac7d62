"""Worker processes for the multi-process tests (launched as subprocesses).

    python tests/mp_workers.py <case> <rank> <world> <port> <device>

Rendezvous over gloo at 127.0.0.1 (control plane only); prints one JSON line.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def plan_partition(rank, world):
    """CPU: every rank computes the same plan; per-slot traffic partitions it."""
    import hashlib

    import torch.distributed as dist
    from paper_2605_22014_b200 import reshard as R, specs
    out = {}
    for case in ("c1", "c2", "c5b"):
        sp, co, cn = specs.baseline_case(case)
        plan = R.compute_transfer_plan(co, cn, sp)
        sha = hashlib.sha256(plan.text().encode()).hexdigest()
        so = [i * world // co.world for i in range(co.world)]
        sn = [i * world // cn.world for i in range(cn.world)]
        traffic = R.plan_traffic(plan, co, so, cn, sn, world)
        shas = [None] * world
        dist.all_gather_object(shas, sha)
        s = plan.summary()
        out[case] = {"agree": len(set(shas)) == 1, "mine": traffic[rank],
                     "egress_total": sum(t[0] for t in traffic), "ingress_total": sum(t[1] for t in traffic),
                     "intra_total": sum(t[2] for t in traffic), "carry_total": sum(t[3] for t in traffic),
                     "plan_total": s["total_bytes"], "plan_carry": s["carryover_bytes"]}
    return out


def ipc_reshard(rank, world, mode):
    """GPU: `world` processes share cuda:<device>; each drives one slot."""
    import torch
    import torch.distributed as dist
    from paper_2605_22014_b200 import reshard as R, specs
    from paper_2605_22014_b200.dist import connect
    from paper_2605_22014_b200.native import RS_DST, RS_SRC
    dev = int(os.environ.get("RS_TEST_DEVICE", "0"))
    torch.cuda.set_device(dev)
    auto_lanes = mode.endswith("-auto")  # the engine's own lane allocation (rings sized before prepare)
    mode = mode.replace("-auto", "")
    sp = specs.llama("llama-mini-a16" if mode.endswith("-a16") else "llama-mini", 4)
    mode = mode.replace("-a16", "")
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 2)
    so = [i * world // co.world for i in range(co.world)]
    sn = [(i + 1) * world // cn.world % world for i in range(cn.world)]  # shifted placement
    copy_kernel, strict = 0, False
    if mode == "direct-tma":  # TMA bulk stores into the peer process's IPC-mapped arena
        mode, copy_kernel = "direct", 17
    if mode == "staged-strict":  # layer barriers across the two slots (peer-mapped done flags)
        mode, strict = "staged", True
    eng = R.Engine([dev], staging_bytes=1 << 20, mode=mode, lanes_per_link=0 if auto_lanes else 1, world_slots=world,
                   first_local_slot=rank, copy_kernel=copy_kernel, strict_layers=strict)
    eng.layout(RS_SRC, sp, co, so)
    eng.layout(RS_DST, sp, cn, sn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    plan = R.compute_transfer_plan(co, cn, sp)
    eng.comm_alloc(plan if mode == "staged" else None)  # plan-sized rings, same on every process
    eng.fill_pattern(RS_SRC, 42)
    eng.fill_pattern(RS_DST, 7)
    connect(eng)
    dist.barrier()
    eng.prepare(plan)
    dist.barrier()
    rep = eng.run()
    torch.cuda.synchronize()
    dist.barrier()
    bad = eng.verify_pattern(RS_DST, 42)[0]
    rep2 = eng.run()  # idempotent second handoff over the same mappings
    dist.barrier()
    bad2 = eng.verify_pattern(RS_DST, 42)[0]
    dist.barrier()
    eng.close()
    return {"ok": rep["ok"] and rep2["ok"], "mismatches": bad + bad2, "error": rep["error"],
            "launches": rep["kernel_launches"]}


def relay_reshard(rank, world):
    """GPU: STAGED with relay chains for DP broadcasts across `world`
    processes on one GPU.  The case comes from RS_RELAY_CASE (JSON: spec
    group bytes, layers, old / new (tp, pp, dp), new-rank slots).  Returns the
    SHA-256 of every destination shard this process holds (the test combines
    them into the reference's digest order) and the traffic the run implies."""
    import hashlib

    import torch
    import torch.distributed as dist
    from paper_2605_22014_b200 import reshard as R, specs
    from paper_2605_22014_b200.dist import connect
    from paper_2605_22014_b200.native import RS_DST, RS_SRC
    case = json.loads(os.environ["RS_RELAY_CASE"])
    dev = int(os.environ.get("RS_TEST_DEVICE", "0"))
    torch.cuda.set_device(dev)
    sp = specs.group_spec(specs.llama("llama-mini-a16", case["layers"]), case["bpe"])
    co, cn = specs.iota_config(1, *case["old"]), specs.iota_config(2, *case["new"])
    so = [r % world for r in co.ranks] if "slot_old" not in case else case["slot_old"]
    sn = case["slot_new"]
    eng = R.Engine([dev], staging_bytes=case.get("staging", 1 << 20), mode="staged", lanes_per_link=case.get("lanes", 1),
                   world_slots=world, first_local_slot=rank, relay=case.get("relay", True),
                   strict_layers=case.get("strict", False))
    eng.layout(RS_SRC, sp, co, so)
    eng.layout(RS_DST, sp, cn, sn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    plan = R.compute_transfer_plan(co, cn, sp)
    eng.comm_alloc(plan)
    eng.fill_pattern(RS_SRC, 42)
    eng.fill_pattern(RS_DST, 7)
    connect(eng)
    dist.barrier()
    eng.prepare(plan)
    dist.barrier()
    rep = eng.run()
    torch.cuda.synchronize()
    dist.barrier()
    bad = eng.verify_pattern(RS_DST, 42)[0]
    digests = {}
    for ti, r, n in eng.entries(RS_DST):
        if sn[cn.ranks.index(r)] == rank:
            digests[f"{ti}:{r}"] = hashlib.sha256(eng.read(RS_DST, r, ti).tobytes()).hexdigest()
    eng.fill_pattern(RS_DST, 9)
    dist.barrier()
    rep2 = eng.run()  # a second handoff over the same rings (epochs advance)
    torch.cuda.synchronize()
    dist.barrier()
    bad2 = eng.verify_pattern(RS_DST, 42)[0]
    dist.barrier()
    eng.close()
    return {"ok": rep["ok"] and rep2["ok"], "mismatches": bad + bad2, "error": rep["error"] or rep2["error"],
            "digests": digests, "bytes_moved": rep["bytes_moved"], "launches": rep["kernel_launches"],
            "relay_routes": rep["relay_routes"], "ring_kernel": rep["ring_kernel"],
            "traffic": R.plan_traffic(plan, co, so, cn, sn, world, relay=True),
            "traffic_p2p": R.plan_traffic(plan, co, so, cn, sn, world)}


def xfer_reshard(rank, world):
    """GPU: the NCCL-style comparator transport across processes; with gloo
    (CPU test plumbing) the link buffers are staged through host memory."""
    import torch
    from paper_2605_22014_b200 import reshard as R, specs, xfer
    from paper_2605_22014_b200.native import RS_DST, RS_SRC
    dev = int(os.environ.get("RS_TEST_DEVICE", "0"))
    torch.cuda.set_device(dev)
    sp = specs.llama("llama-mini", 4)
    co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 2, 2)
    so = [i * world // co.world for i in range(co.world)]
    sn = [(i + 1) * world // cn.world % world for i in range(cn.world)]
    eng = R.Engine([dev], staging_bytes=64 << 10, mode="xfer", world_slots=world, first_local_slot=rank)
    eng.layout(RS_SRC, sp, co, so)
    eng.layout(RS_DST, sp, cn, sn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 42)
    eng.fill_pattern(RS_DST, 7)
    plan = R.compute_transfer_plan(co, cn, sp)
    eng.prepare(plan)
    info = xfer.run(eng, dev, host_staging=True)
    bad = eng.verify_pattern(RS_DST, 42)[0]
    eng.close()
    return {"ok": True, "mismatches": bad, "rounds": info["rounds"], "bytes_sent": info["bytes_sent"]}


def handoff_chain(rank, world, mode):
    """GPU: LiveHandoff across processes -- shadow arenas exchanged in
    Prepare, the commit barrier after every switch, a chain of generations."""
    import torch
    import torch.distributed as dist
    from paper_2605_22014_b200 import reshard as R, specs
    from paper_2605_22014_b200.handoff import LiveHandoff
    from paper_2605_22014_b200.native import RS_SRC
    dev = int(os.environ.get("RS_TEST_DEVICE", "0"))
    torch.cuda.set_device(dev)
    sp = specs.llama("llama-mini", 4)
    eng = R.Engine([dev], staging_bytes=1 << 20, mode=mode, lanes_per_link=1, world_slots=world,
                   first_local_slot=rank)

    def placement(cfg):  # alternate between blocked and shifted placements
        return [((i * world // cfg.world) + cfg.gen) % world for i in range(cfg.world)]

    h = LiveHandoff(eng, sp, specs.iota_config(1, 4, 2, 1), placement, group=dist.group.WORLD)
    eng.fill_pattern(RS_SRC, 42)
    dist.barrier()
    pauses, bad = [], 0
    for gen, shape in enumerate([(2, 2, 2), (2, 1, 2), (4, 2, 1)], start=2):
        h.trigger_resize(specs.iota_config(gen, *shape))
        h.prepare()
        st = h.switch()
        pauses.append(st.pause_s)
        dist.barrier()
        bad += eng.verify_pattern(RS_SRC, 42)[0]
    out = {"ok": h.active.gen == 4 and h.phase.value == "Stable", "mismatches": bad,
           "pauses": pauses, "launches": 0}
    dist.barrier()
    eng.close()
    return out


def main():
    case, rank, world, port = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port, RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "partition":
            res = plan_partition(rank, world)
        elif case == "xfer":
            res = xfer_reshard(rank, world)
        elif case == "relay":
            res = relay_reshard(rank, world)
        elif case.startswith("handoff-"):
            res = handoff_chain(rank, world, case.split("-", 1)[1])
        else:
            res = ipc_reshard(rank, world, case)
    finally:
        dist.destroy_process_group()
    print(json.dumps({"rank": rank, "result": res}), flush=True)


if __name__ == "__main__":
    main()
