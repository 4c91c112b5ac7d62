"""Drop-in for C++ callers: a program written against the reference's
planning API (tools/cpp_api_example.cpp) compiles against
include/reshard_b200/reshard.hpp, links libreshard_b200.so, and produces the
reference's plan text (golden SHA-256 from oracle/_ref, tests/golden) plus the
reference's error behaviour.  CPU only."""
import hashlib
import json
import os
import subprocess

from paper_2605_22014_b200 import specs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(tmp_path):
    exe = tmp_path / "cpp_api_example"
    libdir = os.path.join(ROOT, "paper_2605_22014_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tools", "cpp_api_example.cpp"), "-L", libdir, "-lreshard_b200",
                        f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_caller_plans_like_the_reference(tmp_path, golden):
    """Every BASELINE resize with iota ranks and the default layer split
    (C1, C2, C3, C5, C5b), per element-size group as the reference's
    single-bpe ModelSpec expresses it: the C++ caller's write_plan output has
    the SHA-256 of the reference's own plan (golden from oracle/_ref)."""
    exe = build(tmp_path)
    n = 0
    for case in ("c1", "c2", "c3", "c5", "c5b"):
        sp, co, cn = specs.baseline_case(case)
        for bpe in sorted({t.bpe for t in sp.tensors}):
            key = f"{case}_{bpe}B"
            spec = tmp_path / f"{key}.spec"
            spec.write_text(specs.group_spec(sp, bpe).to_text())
            plan_out = tmp_path / f"{key}.plan"
            out = subprocess.run([str(exe), str(spec), str(co.tp), str(co.pp), str(co.dp), str(cn.tp),
                                  str(cn.pp), str(cn.dp), str(plan_out)], capture_output=True, text=True)
            assert out.returncode == 0, (key, out.stdout, out.stderr)
            got = json.loads(out.stdout)
            want = golden["baseline_plans"][key]
            assert got["identical_gen_throws"] and got["bad_config_violations"] > 0 and got["violations"] == 0
            assert hashlib.sha256(plan_out.read_bytes()).hexdigest() == want["plan_sha"], key
            assert got["pairs_checked"] == want["pairs_checked"], key
            assert got["total_bytes"] == want["total_bytes"] and got["task_count"] == want["tasks"], key
            assert got["reread_task_count"] == got["task_count"] and got["first_remote_task_chunks_1MiB"] > 0
            n += 1
    assert n == 9
