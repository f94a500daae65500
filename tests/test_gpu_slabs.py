"""The multi-GPU slab path (tp_create_slab + halo pack/unpack + split-step C ABI)
on one GPU: several slab contexts exchanging halos in-process must reproduce the
single-context device run — and hence the reference — bit for bit."""
import numpy as np
import pytest

from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.distributed import CudaSlab, LocalComm, SlabRunner, assemble, decompose
from tests.util import assert_bitwise

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("make", [lambda: scenarios.c1_hill(64),
                                  lambda: scenarios.c3_channel(80, 48, t_end=30.0, dt_out=0.5),
                                  lambda: scenarios.wet_valley(96, 70)])
def test_cuda_slabs_equal_single_device(gpu, oracle_kind, make, parts):
    import torch
    from oracle.oracle import OracleSim
    sc = make()
    steps = 30
    t_next = 0.5 / sc.config.scaling.t_unit() if sc.config.inflow else 1e9
    ref = OracleSim(sc, oracle_kind)
    t1, d1, _ = ref.steps(0.0, t_next, steps, t_end=1e9)
    stream = torch.cuda.Stream()
    slabs = [CudaSlab(sc, r, stream=stream) for r in decompose(sc.nrows, parts)]
    run = SlabRunner(slabs, LocalComm())
    t2, d2, _ = run.steps(0.0, t_next, steps, t_end=1e9)
    assert_bitwise(d2, d1, "dts")
    assert t2 == t1
    assert_bitwise(assemble([s.state() for s in slabs]), ref.state()[:, 3:-3, 3:-3], "interior")
    np.testing.assert_allclose(run.audit(), ref.audit(), rtol=1e-12, atol=1e-300)
