"""Multi-rank row-slab decomposition on CPU (no GPU): the orchestration that drives
the GPUs (paper_2104_06784_b200.distributed: halo exchange at the two ghost-refill
points + exact lambda all-reduce) run over the C-oracle slabs, in-process and as a
world_size-2 gloo job.  The decomposed run must equal the single-domain run bit
for bit (dt sequence and every interior value)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle.oracle import OracleSim, OracleSlab
from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.distributed import LocalComm, SlabRunner, TorchComm, assemble, decompose
from tests.util import assert_bitwise


def test_decompose():
    assert decompose(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert decompose(4, 2) == [(0, 2), (2, 4)]
    with pytest.raises(ValueError):
        decompose(5, 3)


def _single(sc, steps, t_next=1e9):
    o = OracleSim(sc, "port")
    t, dts, _ = o.steps(0.0, t_next, steps, t_end=1e9)
    return t, dts, o.state()[:, 3:-3, 3:-3], o.audit()


@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("make", [lambda: scenarios.c1_hill(40),
                                  lambda: scenarios.c3_channel(48, 30, t_end=30.0, dt_out=0.5)])
def test_local_slabs_equal_single_domain(make, parts):
    sc = make()
    steps = 40
    t_next = 0.5 / sc.config.scaling.t_unit() if sc.config.inflow else 1e9
    t1, d1, s1, a1 = _single(sc, steps, t_next)
    slabs = [OracleSlab(sc, r) for r in decompose(sc.nrows, parts)]
    run = SlabRunner(slabs, LocalComm())
    t2, d2, _ = run.steps(0.0, t_next, steps, t_end=1e9)
    assert_bitwise(d2, d1, "dts")
    assert t2 == t1
    assert_bitwise(assemble([s.state() for s in slabs]), s1, "interior state")
    np.testing.assert_allclose(run.audit(), a1, rtol=1e-12, atol=1e-300)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, steps):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = scenarios.c1_hill(36)
    slab = OracleSlab(sc, decompose(sc.nrows, world)[rank])
    run = SlabRunner([slab], TorchComm())
    t, dts, _ = run.steps(0.0, 1e9, steps, t_end=1e9)
    audit = run.audit()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), t=t, dts=dts, state=slab.state(), audit=audit)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_equals_single_domain(tmp_path):
    steps = 25
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), steps), nprocs=2, join=True,
                       start_method="spawn")
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(2)]
    t1, d1, s1, a1 = _single(scenarios.c1_hill(36), steps)
    for x in r:
        assert_bitwise(x["dts"], d1, "dts")
        assert float(x["t"]) == t1
    assert_bitwise(assemble([x["state"] for x in r]), s1, "gloo interior state")
    np.testing.assert_allclose(r[0]["audit"], a1, rtol=1e-12, atol=1e-300)
