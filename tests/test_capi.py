"""The C-ABI library loads and exports every symbol include/rs_reshard.h declares.

CPU only: no compute call is made (engine creation needs a GPU).
"""

import ctypes
import os
import re
import subprocess

from paper_2605_22014_b200 import native as N
from paper_2605_22014_b200 import specs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rs_reshard.h")).read()
    return sorted(set(re.findall(r"\b(rs_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_version_and_error_codes():
    lib = N.lib()
    assert b"sm_100a" in lib.rs_version()
    h = ctypes.c_void_p()
    sp = specs.gpt2_124m(2)
    c = N.config_struct(specs.iota_config(1, 1, 1, 1), sp.num_layers)
    rc = lib.rs_plan_compute(sp.to_text().encode(), c, c, None, ctypes.byref(h))
    assert rc == N.RS_EDOMAIN
    assert lib.rs_last_error() == b"compute_transfer_plan: identical generation ids"
    rc = lib.rs_plan_read(sp.to_text().encode(), b"bogus line\n", ctypes.byref(h))
    assert rc == N.RS_EINTEGRITY and b"unknown record" in lib.rs_last_error()


def test_include_dir_has_only_boundary_headers():
    inc = os.path.join(ROOT, "include")
    assert os.path.exists(os.path.join(inc, "rs_reshard.h"))
    # the header is plain C: compiles as C99 with no CUDA / torch includes
    r = subprocess.run(["gcc", "-std=c99", "-fsyntax-only", "-x", "c", os.path.join(inc, "rs_reshard.h")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_engine_rejects_duplicate_devices_before_touching_cuda():
    """Two slots of one process on one GPU could deadlock STAGED rings; the
    engine refuses the option struct (checked before any CUDA call)."""
    from paper_2605_22014_b200 import reshard as R
    import pytest
    with pytest.raises(N.DomainError, match="listed twice"):
        R.Engine([0, 0])


def test_strict_layers_option_checks():
    """strict_layers is a DIRECT / STAGED schedule (XFER rounds are host
    driven); STAGED barriers need the classic lanes.  Checked before CUDA."""
    from paper_2605_22014_b200 import reshard as R
    import pytest
    with pytest.raises(N.DomainError, match="strict_layers"):
        R.Engine([0], mode="xfer", strict_layers=True)
    with pytest.raises(N.DomainError, match="strict_layers"):
        R.Engine([0], mode="staged", strict_layers=True, ring_discard=8 | 5)


def test_ring_same_slot_is_validated():
    """a typo in ring_same_slot must not silently select a policy."""
    from paper_2605_22014_b200 import reshard as R
    import pytest
    for bad in (3, -1):
        with pytest.raises(N.DomainError, match="ring_same_slot"):
            R.Engine([0], mode="staged", ring_same_slot=bad)
