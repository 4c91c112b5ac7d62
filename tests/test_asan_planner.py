"""Host planner under AddressSanitizer + UndefinedBehaviorSanitizer
(SURVEY.md §5): csrc/host/*.cpp built standalone with -fsanitize, driven over
random resizes (plan, verify, text round trip, chunk_bounds, placement).
CPU only."""
import os
import subprocess

import pytest

from paper_2605_22014_b200 import specs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = ["model.cpp", "layout.cpp", "planner.cpp", "plan_text.cpp", "placement.cpp"]


def test_planner_is_sanitizer_clean(tmp_path):
    exe = tmp_path / "asan_planner"
    srcs = [os.path.join(ROOT, "paper_2605_22014_b200", "csrc", "host", f) for f in HOST]
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-g", "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
                        "-fno-sanitize-recover=all", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tools", "asan_planner.cpp"), *srcs, "-o", str(exe)],
                       capture_output=True, text=True)
    if r.returncode != 0 and "sanitize" in r.stderr and "cannot find" in r.stderr:
        pytest.skip("sanitizer runtime not installed")
    assert r.returncode == 0, r.stderr[-3000:]
    lines = []
    for i, (seed, sp, co, cn) in enumerate(specs.iter_random_cases(60)):
        f = tmp_path / f"s{seed}.spec"
        f.write_text(sp.to_text())
        lines.append(f"{f} {co.tp} {co.pp} {co.dp} {cn.tp} {cn.pp} {cn.dp} {i % 2}")
    for case in ("c1",):
        sp, co, cn = specs.baseline_case(case)
        f = tmp_path / f"{case}.spec"
        f.write_text(sp.to_text())
        lines.append(f"{f} {co.tp} {co.pp} {co.dp} {cn.tp} {cn.pp} {cn.dp} 0")
    out = subprocess.run([str(exe)], input="\n".join(lines) + "\n", capture_output=True, text=True, timeout=600,
                         env={**os.environ, "ASAN_OPTIONS": "detect_leaks=1", "UBSAN_OPTIONS": "print_stacktrace=1"})
    assert out.returncode == 0, (out.stdout, out.stderr[-4000:])
    assert '"violations": 0' in out.stdout and '"plans": ' in out.stdout
