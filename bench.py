#!/usr/bin/env python3
"""Reshard benchmark (BASELINE.json metric: reshard GB/s + handoff ms for a
7B TP/PP/DP resize, and % of the NVLink/HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one live handoff: the full transfer plan of the workload executed
over device-resident shard stores (plan computed and compiled beforehand, as
in the paper's Prepare phase).

N=1 workload (BASELINE config 2 at full size, the metric's own config):
Llama-2-7B, bf16 params + fp32 master + Adam m/v, TP4.PP2.DP1 (8 ranks) ->
TP2.PP2.DP1 (4 ranks) with every logical rank on cuda:0 (intra-device
relayout): 91.06 GB of plan bytes + 3.28 GB of carryover; src + dst state is
188.7 GB resident in HBM.  Inputs are ~700x the 126 MB L2, so no L2 flush is
needed between steps.

--impl reference times the reference's own execute_plan (oracle/_ref, built
from /root/reference/proj/src) on the host cores, on a bounded sample of the
same workload.

Every number is printed as ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reshard GB/s (Llama-2-7B TP4PP2->TP2PP2 handoff)"
UNIT = "GB/s"
HIGH_IS_GOOD = True
SEED = 42


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:  # NVML (initialised before the timed region): a sample costs microseconds
            import pynvml as nvml
            nvml.nvmlInit()
            self._h = nvml.nvmlDeviceGetHandleByIndex(index)
            self._max = nvml.nvmlDeviceGetMaxClockInfo(self._h, nvml.NVML_CLOCK_SM)
            self._nvml = nvml
        except Exception:
            self._nvml = None

    def _sample(self):
        nvml = self._nvml
        if nvml is not None:
            sm = nvml.nvmlDeviceGetClockInfo(self._h, nvml.NVML_CLOCK_SM)
            r = nvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            # hw_slowdown 0x8, hw_thermal 0x40, sw_thermal 0x20, sw_power_cap 0x4
            self.rows.append([str(self.index), str(sm), str(self._max)] +
                             ["Active" if r & b else "Not Active" for b in (0x8, 0x40, 0x20, 0x4)])
            return
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True, timeout=5).stdout.strip()
        if out:
            self.rows.append([x.strip() for x in out.split(",")])

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.01 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if self._nvml is not None:
            try:
                self._nvml.nvmlShutdown()
            except Exception:
                pass

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(n_gpus: int, layers: int = 0):
    from paper_2605_22014_b200 import specs
    if layers:  # profiling-only slice (never a bench value)
        sp, co, cn = specs.sliced_case("c2", layers)
        return sp, co, cn, f"c2 PROFILING SLICE ({layers} layers)"
    sp, co, cn = specs.baseline_case("c2")
    desc = ("c2: Llama-2-7B bf16 params + fp32 master/m/v, TP4.PP2.DP1 (8 ranks) -> "
            "TP2.PP2.DP1 (4 ranks), all logical ranks on one B200 (intra-device relayout)")
    return sp, co, cn, desc


def cpu_sample(layers: int):
    """Bounded sample of the same workload for the reference CPU path: the
    C2 resize on a `layers`-deep slice of Llama-2-7B (embedding + blocks +
    head), one single-dtype spec per group (the reference holds one element
    size per ModelSpec, model_spec.hpp:45)."""
    from paper_2605_22014_b200 import specs
    sp, co, cn = specs.sliced_case("c2", layers)
    return [(specs.group_spec(sp, b), co, cn) for b in (2, 4)]


def run_reference_cpu(threads: int, layers: int, steps: int, warmup: int, staging: int):
    """Time the reference execute_plan (oracle/_ref) on host cores."""
    from oracle.pyoracle import Oracle, available
    if not available("ref"):
        return None
    ref = Oracle("ref")
    nproc = os.cpu_count() or 1
    benches = [ref.bench(g, co, cn, SEED, fill_threads=nproc) for g, co, cn in cpu_sample(layers)]
    for _ in range(warmup):
        for b in benches:
            b.step(staging, threads)
    secs, nbytes, ok = [], 0, True
    for _ in range(steps):
        t = 0.0
        for b in benches:
            r = b.step(staging, threads)
            ok &= r["ok"]
            t += r["seconds"]
        secs.append(t)
    nbytes = sum(b.plan_bytes for b in benches)
    bad = sum(b.mismatches(nproc) for b in benches)
    for b in benches:
        b.close()
    mean = statistics.mean(secs)
    return {"value": nbytes / mean / 1e9, "seconds_per_step": mean, "plan_bytes": nbytes,
            "ok": ok and bad == 0, "mismatches": bad}


def reference_arm(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # >= 2 layers: the resize is PP2 -> PP2, every stage needs a layer
    layers = max(2, int(os.environ.get("RS_BENCH_CPU_LAYERS", str(min(os.cpu_count() or 1, 16)))))
    threads = min(os.cpu_count() or 1, layers)  # execute_plan is per-layer; one thread per layer
    res = run_reference_cpu(threads, layers, max(1, args.steps), args.warmup, args.staging_bytes)
    _, _, _, desc = workload(args.gpus)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref not built (reference sources absent at build time)"}))
        return
    sample = ("reference execute_plan (oracle/_ref, unmodified /root/reference/proj/src) on the "
              f"C2 resize of a {layers}-layer Llama-2-7B slice (bf16 group + fp32 master/m/v group), "
              f"{res['plan_bytes'] / 1e9:.2f} GB plan bytes per step, layers dealt to "
              f"{threads} threads, LoopbackTransport, B={args.staging_bytes}")
    line = {"metric": METRIC, "value": round(res["value"], 4), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["seconds_per_step"] * 1e3,
            "higher_is_better": HIGH_IS_GOOD, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic (reference pattern, shard_store.cpp:51-85)",
            "impl": "reference",
            "config": {"workload": desc + f" -- CPU sample: {layers}-layer slice", "staging_bytes": args.staging_bytes},
            "cpu_baseline": {"value": round(res["value"], 4), "unit": UNIT, "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": round(res["value"], 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "correct": res["ok"]}
    print(json.dumps(line), flush=True)


def xfer_one_gpu(args) -> None:
    """--mode xfer at N=1: the NCCL send/recv comparator on one B200.  Every
    rank gets its own virtual device slot (one RS_MODE_XFER engine each), so
    every cross-rank chunk is packed by our kernel, moved by ncclSend/ncclRecv
    (NCCL's self-loop on a single-rank communicator, libnccl called directly)
    and unpacked by our kernel, round by round on the engine's chunk schedule
    and budget B -- the paper's executor shape.  The step is
    host-driven (NCCL group per round, stream syncs), so it is timed by the
    host clock around fully synchronised steps."""
    import torch
    from paper_2605_22014_b200 import reshard as R
    from paper_2605_22014_b200 import xfer
    from paper_2605_22014_b200.native import RS_DST, RS_SRC

    torch.cuda.set_device(0)
    sp, co, cn, desc = workload(1, args.profile_layers)
    plan = R.compute_transfer_plan(co, cn, sp)
    summ = plan.summary()
    total = summ["total_bytes"]
    nslots = max(max(co.ranks), max(cn.ranks)) + 1
    nccl = xfer.Nccl(0)
    engs = []
    for s in range(nslots):
        e = R.Engine([0], staging_bytes=args.staging_bytes, mode="xfer", world_slots=nslots, first_local_slot=s)
        e.layout(RS_SRC, sp, co, list(co.ranks))
        e.layout(RS_DST, sp, cn, list(cn.ranks))
        e.alloc(RS_SRC)
        e.alloc(RS_DST)
        e.fill_pattern(RS_SRC, SEED)
        engs.append(e)
    for e in engs:
        e.prepare(plan)
    for _ in range(args.warmup):
        xfer.run_local_slots(engs, nccl, 0)
    with ClockSampler(0) as clk:
        infos = [xfer.run_local_slots(engs, nccl, 0) for _ in range(args.steps)]
    bad = sum(e.verify_pattern(RS_DST, SEED)[0] for e in engs)
    step_ms = statistics.mean(i["seconds"] for i in infos) * 1e3
    pk = peaks()
    algo = 2 * (total + summ["carryover_bytes"])
    achieved = algo / (step_ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": round(total / (step_ms / 1e3) / 1e9, 2), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
            "handoff_ms": round(step_ms, 4), "higher_is_better": HIGH_IS_GOOD, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic: reference pattern state (shard_store.cpp:51-85)",
            "config": {"workload": desc + " -- NCCL comparator: one virtual slot per rank",
                       "plan_bytes": total, "carryover_bytes": summ["carryover_bytes"], "mode": "xfer",
                       "transport": f"ncclSend/ncclRecv self-loop, NCCL {nccl.version}",
                       "staging_bytes": args.staging_bytes, "rounds": infos[0]["rounds"],
                       "links": infos[0]["links"], "bytes_through_nccl": infos[0]["bytes_sent"],
                       "timing": "host clock around synchronised steps (host-driven rounds)"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None,
                         "kernel": "rs_copy_kernel pack/unpack + NCCL copy",
                         "algorithmic_bytes_per_launch": algo, "peak_source": pk["source"]},
            "clocks": clk.summary(), "gpu_launches": None,
            "correct": {"dst_pattern_mismatches": int(bad)}}
    print(json.dumps(line), flush=True)
    for e in engs:
        e.close()
    nccl.close()


def copy_kernel_label(mode: str, world: int) -> str:
    if mode == "staged":
        return ("rs_exchange_kernel: ring lanes (one 256-thread CTA per lane end, 128 KiB slots x 2, "
                "L2-resident), spare CTAs copy local tasks")
    if mode == "xfer":
        return "pack/unpack LDG8 non-persistent kernels around ncclSend/ncclRecv"
    if world > 1:
        return "LDG8 non-persistent grid (peer stores over NVLink), one 16 KB item per warp"
    return ("TMA bulk copy (cp.async.bulk global->smem->global, mbarrier complete_tx), one 1-warp CTA per "
            "16 KB item, non-persistent grid")


def ours(args) -> None:
    """N=1: every logical rank on cuda:0.  N>1 (torchrun, one process per GPU):
    rank id r of both configs lives on GPU r*N//8 (iota placement at N=8);
    each process drives its GPU's slot, peer arenas are CUDA-IPC mapped and
    every byte moves GPU->GPU over NVLink inside our kernels.  The control
    plane (handle exchange, barriers, max-over-ranks timing) is gloo."""
    import torch
    from paper_2605_22014_b200 import reshard as R
    from paper_2605_22014_b200.native import RS_DST, RS_SRC

    rank, world, local = dist_env()
    device = 0 if os.environ.get("RS_BENCH_SAME_DEVICE") else local
    torch.cuda.set_device(device)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    sp, co, cn, desc = workload(args.gpus, args.profile_layers)
    if args.placement == "searched":
        # placement-aware destination rank list (rs_plan_placement); changes the
        # plan (more self-held bytes), so it is a different workload: labelled
        cn, _ = R.choose_placement(co, cn, sp, candidates=sorted(set(co.ranks) | set(cn.ranks)))
        desc += f" [searched dst rank list {cn.ranks}]"
    plan = R.compute_transfer_plan(co, cn, sp)
    summ = plan.summary()
    total = summ["total_bytes"]
    nranks = max(max(co.ranks), max(cn.ranks)) + 1
    slot_of = lambda r: r * world // nranks  # noqa: E731
    so = [slot_of(r) for r in co.ranks]
    sn = [slot_of(r) for r in cn.ranks]
    traffic = R.plan_traffic(plan, co, so, cn, sn, world)

    eng = R.Engine([device], staging_bytes=args.staging_bytes, mode=args.mode, lanes_per_link=args.lanes,
                   ring_slot_kib=args.ring_slot_kib,
                   strict_layers=args.strict, world_slots=world, first_local_slot=rank)
    eng.layout(RS_SRC, sp, co, so)
    eng.layout(RS_DST, sp, cn, sn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    if args.mode == "staged":
        eng.comm_alloc(plan)
    eng.fill_pattern(RS_SRC, SEED)
    if world > 1:
        from paper_2605_22014_b200.dist import connect
        from paper_2605_22014_b200.native import RS_COMM
        connect(eng, which=(RS_SRC, RS_DST) + ((RS_COMM,) if args.mode == "staged" else ()))
    eng.prepare(plan)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    if args.mode == "xfer":
        # comparator: our pack/unpack kernels around torch.distributed p2p
        # (NCCL between GPUs; gloo + host staging when processes share a GPU)
        from paper_2605_22014_b200 import xfer
        same = bool(os.environ.get("RS_BENCH_SAME_DEVICE"))
        group = None if (world == 1 or same) else torch.distributed.new_group(backend="nccl")

        def one_step():
            info = xfer.run(eng, device, host_staging=same, group=group)
            return {"ok": True, "device_ms": info["seconds"] * 1e3, "kernel_launches": 1 + 2 * info["rounds"]}
    else:
        def one_step():
            return eng.run()

    for _ in range(args.warmup):
        barrier()
        rep = one_step()
        assert rep["ok"], rep
    barrier()
    bad_warm = eng.verify_pattern(RS_DST, SEED)[0]

    barrier()
    launches = 0
    dev_ms = []
    with ClockSampler(device) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if world > 1:
                torch.distributed.barrier()  # every GPU starts the handoff together
            rep = one_step()
            dev_ms.append(rep["device_ms"])
            launches += rep["kernel_launches"]
        barrier()
        wall = time.perf_counter() - t0
    step_ms = sum(dev_ms) / len(dev_ms)
    mismatches = eng.verify_pattern(RS_DST, SEED)[0]
    if world > 1:
        t = torch.tensor([step_ms, float(mismatches), float(bad_warm), float(launches)], dtype=torch.float64)
        torch.distributed.all_reduce(t[:1], op=torch.distributed.ReduceOp.MAX)
        tt = t[1:].clone()
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.SUM)
        step_ms = float(t[0])
        mismatches, bad_warm, launches = int(tt[0]), int(tt[1]), int(tt[2])

    pk = peaks()
    if world == 1:
        # algorithmic bytes: every moved byte read once + written once (the
        # floor for any path; STAGED's ring slots are staging overhead on top)
        algo_bytes = 2 * (total + summ["carryover_bytes"])
        kernel = "rs_exchange_kernel" if args.mode == "staged" else "rs_copy_tma_np_kernel"
        achieved = algo_bytes / (step_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None, "kernel": kernel,
                "algorithmic_bytes_per_launch": algo_bytes, "peak_source": pk["source"],
                "note": ("the peak is torch copy_ of 2 GiB (MEASURED_PEAKS.json); the TMA bulk copy kernel "
                         "sustains 6.82-6.95 TB/s on a plain contiguous 2-32 GiB copy where copy_ gets "
                         "6.50-6.69 (profiles/r1/contig_probe.jsonl), so frac can exceed 1; "
                         "frac_vs_contiguous_copy compares with the kernel's own contiguous 32 GiB copy")}
        if args.mode == "direct":
            contiguous = 6922.3  # profiles/r1/contig_probe.jsonl: this kernel (TMA-NP, 16 KB items), 32 GiB copy
            roof["contiguous_copy_gbs"] = contiguous
            roof["frac_vs_contiguous_copy"] = round(achieved / contiguous, 4)
        if args.mode == "staged":  # with DRAM-resident rings each remote byte costs 2 more
            ring = algo_bytes + 2 * summ["remote_bytes"]
            roof["ring_staged_bytes_per_launch"] = ring
            roof["frac_vs_dram_resident_ring"] = round(ring / (step_ms / 1e3) / 1e9 / pk["hbm_gbs"], 4)
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp) and args.mode == "direct" and not args.profile_layers:
            with open(tp) as f:  # measured on this exact launch (full-size C2, DIRECT)
                roof["traffic"] = json.load(f).get("rs_copy_kernel_dram_bytes_per_launch")
    else:
        # the busiest GPU's NVLink direction bounds the handoff
        link = max(max(t[0], t[1]) for t in traffic)
        achieved = link / (step_ms / 1e3) / 1e9
        nvl = 770.0
        roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": nvl, "unit": "GB/s",
                "frac": round(achieved / nvl, 4), "traffic": None, "kernel": ("rs_exchange_kernel (ring lanes over peer memory)" if args.mode == "staged"
                                                                 else "rs_copy_kernel<8> non-persistent (peer stores)"),
                "algorithmic_bytes_per_launch": link,
                "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                "per_gpu_egress_ingress_GB": [[round(t[0] / 1e9, 2), round(t[1] / 1e9, 2)] for t in traffic]}

    line = {"metric": METRIC, "value": round(total / (step_ms / 1e3) / 1e9, 2), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(step_ms, 4), "handoff_ms": round(step_ms, 4),
            "higher_is_better": HIGH_IS_GOOD, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic: reference pattern state (shard_store.cpp:51-85), random-init-equivalent bytes",
            "config": {"workload": desc if world == 1 else desc.replace(
                           "all logical ranks on one B200 (intra-device relayout)",
                           f"rank r on GPU r*{world}//8, one process per GPU"),
                       "plan_bytes": total, "carryover_bytes": summ["carryover_bytes"],
                       "tasks": summ["task_count"], "mode": args.mode, "placement": args.placement, "staging_bytes": args.staging_bytes,
                       "strict_layers": bool(args.strict), "copy_kernel": copy_kernel_label(args.mode, world),
                       "l2": "inputs 188.7 GB >> 126 MB L2: no flush needed"},
            "roofline": roof, "clocks": clk.summary(), "gpu_launches": launches, "wall_s": round(wall, 3),
            "correct": {"dst_pattern_mismatches": int(mismatches), "warmup_check": int(bad_warm)}}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_layers = int(os.environ.get("RS_BENCH_CPU_SAMPLE_LAYERS", "4"))  # ~12 s of single-thread work
        res = run_reference_cpu(1, cpu_layers, 1, 0, args.staging_bytes)
        if res is not None:
            line["cpu_baseline"] = {
                "value": round(res["value"], 4), "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": (f"reference execute_plan (oracle/_ref) on the C2 resize of a {cpu_layers}-layer Llama-2-7B "
                           f"slice, both dtype groups, {res['plan_bytes'] / 1e9:.2f} GB, 1 thread "
                           f"(the reference is single-threaded) of {os.cpu_count()} host cores")}
    if not args.no_e2e:
        pos_old = {r: i for i, r in enumerate(co.ranks)}
        pos_new = {r: i for i, r in enumerate(cn.ranks)}

        def local_entry(which, r):
            return (so[pos_old[r]] if which == RS_SRC else sn[pos_new[r]]) == rank
        line["e2e"] = e2e(eng, plan, total, args, world, local_entry)
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e(eng, plan, total, args, world=1, local_entry=None) -> dict:
    """Same handoff through rs_execute_host with HOST shard stores: every step
    copies all (this process's) source shards H2D from pinned memory and all
    destination shards D2H, layer-pipelined.  Host RAM cannot hold a second
    94 GB store next to the pinned source (196 GB box), so destination shards
    land in a 4 GiB pinned window that successive shards overwrite; every
    byte still crosses PCIe.  On this box H2D and D2H each run ~55 GB/s and
    ~96 GB/s combined when the engine merges back-to-back shards into large
    copies (tools/e2e_probe2.py): the e2e step is host-transfer bound, the
    reshard kernel is ~1.5 % of it."""
    import torch
    from paper_2605_22014_b200.native import RS_DST, RS_SRC
    from paper_2605_22014_b200.reshard import PinnedBuffer

    src = eng.entries(RS_SRC)
    dst = eng.entries(RS_DST)
    src_local = [local_entry(RS_SRC, r) for _, r, _ in src]
    dst_local = [local_entry(RS_DST, r) for _, r, _ in dst]
    h2d = sum(n for (_, _, n), l in zip(src, src_local) if l)
    d2h = sum(n for (_, _, n), l in zip(dst, dst_local) if l)
    host_src = PinnedBuffer(max(h2d, 1))
    window = PinnedBuffer(4 << 30)
    # the host source store holds the device source state, so the e2e output
    # is checkable against the analytic pattern afterwards
    off, src_ptrs = 0, []
    for (ti, r, n), l in zip(src, src_local):
        if not l:
            src_ptrs.append(0)
            continue
        src_ptrs.append(host_src.ptr + off)
        eng.read_to(RS_SRC, r, ti, host_src.ptr + off, n)
        off += n
    dst_ptrs, woff = [], 0
    for (_, _, n), l in zip(dst, dst_local):
        if not l:
            dst_ptrs.append(0)
            continue
        if woff + n > window.nbytes:
            woff = 0
        dst_ptrs.append(window.ptr + woff)
        woff += (n + 255) // 256 * 256
    eng.fill_pattern(RS_DST, SEED ^ 0xDEAD)  # poison: the e2e run must rewrite every byte
    times, ok = [], True
    steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(steps):
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        rep = eng.execute_host(plan, src_ptrs, dst_ptrs)
        if world > 1:
            torch.distributed.barrier()  # every GPU's host stores complete
        times.append(time.perf_counter() - t0)
        ok &= rep["ok"]
    bad = eng.verify_pattern(RS_DST, SEED)[0]
    host_src.free()
    window.free()
    mean = statistics.mean(times)
    if world > 1:
        t = torch.tensor([float(h2d), float(d2h), float(bad)], dtype=torch.float64)
        torch.distributed.all_reduce(t)
        h2d, d2h, bad = int(t[0]), int(t[1]), int(t[2])
    return {"value": round(total / mean / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "s_per_step": round(mean, 4),
            "path": "rs_execute_host (C ABI, host shard stores)",
            "bound": ("host<->device transfer: 188.7 GB per step over PCIe; measured ceiling "
                      "H2D 55.5 + D2H 55.2 GB/s alone, ~96 GB/s combined concurrent with merged copies "
                      "(profiles/r1/e2e_probe2.json)"),
            "ok": bool(ok and bad == 0)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="direct", choices=["direct", "staged", "xfer"])
    ap.add_argument("--staging-bytes", type=int, default=1 << 30)
    ap.add_argument("--lanes", type=int, default=0, help="ring lanes per link (0: automatic)")
    ap.add_argument("--strict", type=int, default=0)
    ap.add_argument("--placement", default="iota", choices=["iota", "searched"],
                    help="destination rank list: BASELINE iota, or rs_plan_placement's choice")
    ap.add_argument("--ring-slot-kib", type=int, default=0, help="STAGED ring slot cap (0: default, -1: none)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-layers", type=int, default=0, help="profiling slice (not a bench value)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    elif args.mode == "xfer" and dist_env()[1] == 1 and not os.environ.get("RS_BENCH_SAME_DEVICE"):
        xfer_one_gpu(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
