"""Drop-in for C++ callers of the reference's *execution* API: a program
written against proj/include/reshard/{executor,shard_store,transport}.hpp
(tools/cpp_exec_example.cpp: ShardStore::allocate / fill_pattern,
RecordingTransport, execute_plan(plan, src, dst, transport, B, bpe))
compiles against include/reshard/*.hpp unchanged, links libreshard_b200.so,
and runs the plan on the B200.  Its ExecutionReport fields and destination
digests must equal the reference executor's own (tests/golden, produced by
oracle/_ref)."""
import hashlib
import json
import os
import subprocess

import pytest

from paper_2605_22014_b200 import specs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(tmp_path):
    exe = tmp_path / "cpp_exec_example"
    libdir = os.path.join(ROOT, "paper_2605_22014_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tools", "cpp_exec_example.cpp"), "-L", libdir, "-lreshard_b200",
                        f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def cfg_file(path, c):
    stages = "-" if c.layer_stage is None else ",".join(map(str, c.layer_stage))
    path.write_text(f"{c.gen} {c.tp} {c.pp} {c.dp} {','.join(map(str, c.ranks))} {stages}\n")
    return str(path)


def run(exe, tmp_path, sp, co, cn, B, mode):
    spec = tmp_path / "spec.txt"
    spec.write_text(sp.to_text())
    out = tmp_path / "dst.bin"
    r = subprocess.run([str(exe), str(spec), cfg_file(tmp_path / "old.cfg", co), cfg_file(tmp_path / "new.cfg", cn),
                        str(B), str(sp.bytes_per_element), mode, str(out)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, (r.stdout, r.stderr)
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    return rep, hashlib.sha256(out.read_bytes()).hexdigest()


def test_cpp_exec_example_compiles(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["staged", "direct"])
def test_cpp_execute_plan_matches_reference(mode, tmp_path, golden):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = build(tmp_path)
    rows = {r["seed"]: r for r in golden["random_pairs"]["cases"]}
    n = 0
    for seed, sp, co, cn in specs.iter_random_cases(24, golden["random_pairs"]["base_seed"]):
        for B in ("4096", "64"):
            want = rows[seed]["exec"][B]
            rep, sha = run(exe, tmp_path, sp, co, cn, int(B), mode)
            assert rep["ok"] == want["ok"], (seed, B, rep)
            for k in ("bytes_moved", "local_copy_bytes", "layers_processed"):
                assert rep[k] == want[k], (seed, B, k, rep)
            assert (rep["failed_layer"] if rep["failed_layer"] >= 0 else None) == want["failed_layer"]
            assert rep["peak_staging_bytes"] <= int(B)
            assert sha == want["dst_sha"], (seed, B)
            # transport accounting: every cross-rank byte as reference-sized frames
            assert rep["event_bytes"] == rep["bytes_moved"] == rep["bytes_sent"]
            assert rep["pattern_bad"] == 0
            n += 1
    assert n == 48
    # full GPT-2 C1 (8 ranks, 12 layers, 1.57 GB) at B = 1 GiB
    sp, co, cn = specs.baseline_case("c1")
    want = golden["c1_exec"]["1073741824"]
    rep, sha = run(exe, tmp_path, sp, co, cn, 1 << 30, mode)
    assert rep["ok"] and sha == want["dst_sha"]
    assert (rep["bytes_moved"], rep["local_copy_bytes"], rep["layers_processed"]) == \
        (want["bytes_moved"], want["local_copy_bytes"], want["layers_processed"])
