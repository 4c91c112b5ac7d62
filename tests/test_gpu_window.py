"""Bounded-device-memory layer streaming of host shard stores (GPU).

rs_execute_host with window_layers = W keeps only W layers' shards on the
device (layer l in slot l % W, a slot refilled after its previous layer's
D2H).  Host stores come from the C oracle's pattern fill of C_old; the host
destination must equal the oracle's analytic pattern of C_new byte for byte.
"""
import numpy as np
import pytest

from paper_2605_22014_b200 import reshard as R
from paper_2605_22014_b200 import specs
from paper_2605_22014_b200.native import RS_DST, RS_SRC

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_windowed(sp, co, cn, window, oracle_c, repeat=2):
    src = oracle_c.store_pattern(sp, co, 11)
    want = oracle_c.store_pattern(sp, cn, 11)
    eng = R.Engine([0], staging_bytes=1 << 30)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    ks, kd = sorted(src.entries), sorted(want.entries)
    assert [(t, r) for t, r, _ in eng.entries(RS_SRC)] == ks
    outs = {k: np.zeros_like(want.entries[k]) for k in kd}
    plan = R.compute_transfer_plan(co, cn, sp)
    for _ in range(repeat):  # second call reuses the compiled program and window
        rep = eng.execute_host(plan, [src.entries[k].ctypes.data for k in ks], [outs[k].ctypes.data for k in kd],
                               window_layers=window)
        assert rep["ok"], rep
    for k in kd:
        assert np.array_equal(outs[k], want.entries[k]), (window, k)
    with pytest.raises(ValueError, match="windowed"):
        eng.verify_pattern(RS_DST, 11)
    eng.close()


@pytest.mark.parametrize("window", [1, 2, 3])
def test_windowed_mini_llama(window, oracle_c):
    sp = specs.llama("llama-mini", 6)
    run_windowed(sp, specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 3, 1), window, oracle_c)


def test_windowed_gpt2_c1(oracle_c):
    sp, co, cn = specs.baseline_case("c1")
    run_windowed(sp, co, cn, 2, oracle_c, repeat=1)
