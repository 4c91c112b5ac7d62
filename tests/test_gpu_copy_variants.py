"""Every copy-engine variant is bit-exact (GPU): LDG x4/x8/x16, CTA-cooperative,
evict-first stores, TMA bulk single-issuer and multi-issuer rings, and the
copy-engine comparator (RS_COPY_CE, cudaMemcpy2DAsync planes)."""
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


@pytest.mark.parametrize("copy_kernel", [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18])
@pytest.mark.parametrize("case", ["c1", "mini"])
def test_copy_variant_bitexact(copy_kernel, case):
    if case == "c1":
        sp, co, cn = specs.sliced_case("c1", 2)
    else:
        sp = specs.llama("llama-mini", 4)
        co, cn = specs.iota_config(1, 4, 2, 1), specs.iota_config(2, 2, 1, 2)
    eng = R.Engine([0], staging_bytes=1 << 30, copy_kernel=copy_kernel)
    eng.layout(RS_SRC, sp, co)
    eng.layout(RS_DST, sp, cn)
    eng.alloc(RS_SRC)
    eng.alloc(RS_DST)
    eng.fill_pattern(RS_SRC, 5)
    eng.fill_pattern(RS_DST, 6)
    rep = R.execute_plan(R.compute_transfer_plan(co, cn, sp), eng)
    assert rep["ok"] and eng.verify_pattern(RS_DST, 5)[0] == 0
    eng.close()
