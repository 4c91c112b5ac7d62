"""CUDA error propagation through the C ABI (SURVEY §4 fault tests): device
failures come back as RS_ESYSTEM (SystemError_) with the CUDA error text,
never as a crash or a silent success."""
import os
import subprocess
import sys

import pytest

from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs
from paper_2605_22014_b200.native import RS_DST, RS_SRC, SystemError_

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_out_of_memory_is_a_system_error_and_recoverable():
    sp = specs.llama("llama-mini", 2)
    co, cn = specs.iota_config(1, 2, 1, 1), specs.iota_config(2, 1, 1, 1)
    eng = R.Engine([0], staging_bytes=1 << 50)  # B far beyond HBM: the B-sized comm arena cannot exist
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    with pytest.raises(SystemError_, match="cudaMalloc"):
        eng.comm_alloc()
    eng.alloc(RS_SRC)  # the engine (and the context) stay usable
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 1)
    rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, 1)[0] == 0
    eng.close()


CHILD = r"""
import sys
sys.path.insert(0, sys.argv[1])
from paper_2605_22014_b200 import reshard as R, specs
from paper_2605_22014_b200.native import RS_DST, RS_SRC, SystemError_
sp = specs.llama("llama-mini", 2)
co, cn = specs.iota_config(1, 2, 1, 1), specs.iota_config(2, 1, 1, 1)
eng = R.Engine([0], staging_bytes=1 << 20)
eng.layout(RS_SRC, sp, co)
eng.layout(RS_DST, sp, cn)
eng.alloc(RS_SRC)
for ti, rank, nbytes in eng.entries(RS_DST):
    eng.bind(RS_DST, rank, ti, 0x1000, nbytes)  # not device memory: the copy faults
try:
    R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    print("NO ERROR")
except SystemError_ as e:
    print("SYSTEM ERROR:", e)
"""


def test_device_fault_is_reported_not_crashed():
    """An illegal address inside the copy kernel (a bound destination that is
    not device memory) surfaces as RS_ESYSTEM from rs_run.  Run in a child
    process: the fault poisons that CUDA context."""
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=300)
    assert "SYSTEM ERROR:" in out.stdout, (out.stdout, out.stderr[-2000:])
    assert "illegal" in out.stdout.lower() or "invalid" in out.stdout.lower(), out.stdout
