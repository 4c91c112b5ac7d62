"""A plain C99 program (tools/capi_example.c) links libreshard_b200.so through
include/rs_reshard.h and plans BASELINE config 2 -- no Python on its path.
CPU only (planning is host code)."""
import json
import os
import subprocess

from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_plans_through_the_abi(tmp_path):
    exe = tmp_path / "capi_example"
    libdir = os.path.join(ROOT, "paper_2605_22014_b200")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tools", "capi_example.c"), "-L", libdir, "-lreshard_b200",
                        f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    sp, co, cn = specs.baseline_case("c2")
    spec = tmp_path / "c2.spec"
    spec.write_text(sp.to_text())
    out = subprocess.run([str(exe), str(spec), "4", "2", "1", "2", "2", "1"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    got = json.loads(out.stdout)
    want = R.compute_transfer_plan(co, cn, sp)
    s = want.summary()
    assert got["violations"] == 0
    for k in ("total_bytes", "remote_bytes", "local_bytes", "carryover_bytes", "task_count"):
        assert got[k] == s[k], k
    assert got["plan_text_bytes"] == len(want.text()) + 1
