"""Row-block (slab) decomposition of the time-stepping core across devices.

SURVEY.md §8(e): the padded grid is split into contiguous row blocks (j is the
slow index, field.hpp:23).  Each slab owns its rows plus two halo rows per side
and exchanges them exactly where the reference refills ghosts:

  1. after apply_boundaries(u, t)        (solver.cpp:639)  — rows of u^n
  2. after apply_boundaries(u*, t + dt)  (solver.cpp:523)  — rows of u*

plus one all-reduce(MAX) of the local wave-speed bound per step, which is exact
and partition independent, so dt and every state value are bitwise those of the
single-device run (tests/test_distributed_*.py check that).  Halo rows are
exchanged at full padded width after the owner's W/E ghost fill, which keeps
the reference's corner semantics; inflow cells are applied by the owning slab.

Slab backends (same method set):
  * CudaSlab — one tp_create_slab context (include/tpflow_b200.h) on one GPU,
    buffers are CUDA tensors; halos move with NCCL send/recv (TorchComm) or
    device copies (LocalComm, several slabs in one process).
  * oracle.oracle.OracleSlab — the CPU checker's slab (tests only, gloo).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np


def row_work(sc, tx: int = 16, halo: int = 2) -> np.ndarray:
    """Per-row work estimate of a Mode-I scenario for the stage kernels: the number of
    16-column tiles in which the row's radius-2 neighbourhood holds wet cells (dry tiles are
    bitwise no-ops and skipped).  Mode-II / no release: uniform."""
    if sc.h0 is None or sc.hydrograph is not None:
        return np.ones(sc.nrows)
    wet = np.asarray(sc.h0) > 0.0
    if sc.vx0 is not None:
        wet |= (np.asarray(sc.vx0) != 0.0) | (np.asarray(sc.vy0) != 0.0)
    nr, nc = wet.shape
    ntx = (nc + tx - 1) // tx
    pad = np.zeros((nr, ntx * tx), dtype=bool)
    pad[:, :nc] = wet
    # columns dilated by the radius-2 box (a tile's box reads 2 cells of each neighbour tile)
    colw = pad.copy()
    colw[:, 2:] |= pad[:, :-2]
    colw[:, 1:] |= pad[:, :-1]
    colw[:, :-1] |= pad[:, 1:]
    colw[:, :-2] |= pad[:, 2:]
    tiles = colw.reshape(nr, ntx, tx).any(axis=2)           # [rows, tile columns]
    rows = tiles.copy()
    for d in range(1, halo + 1):                            # rows dilated the same way
        rows[d:] |= tiles[:-d]
        rows[:-d] |= tiles[d:]
    return rows.sum(axis=1).astype(np.float64)


def decompose_balanced(work: np.ndarray, parts: int, floor: float = 0.05, min_rows: int = 2) -> List[tuple]:
    """Contiguous row blocks [row0, row1) with near-equal work (strong scaling): `work` per
    row (row_work), plus `floor` x its mean per row so dry rows are not free (boundary
    fill, tile lists, later spreading).  Every slab keeps >= min_rows rows."""
    nrows = len(work)
    if parts < 1 or nrows < min_rows * parts:
        raise ValueError(f"cannot split {nrows} rows into {parts} slabs of >= {min_rows} rows")
    w = np.asarray(work, dtype=np.float64)
    w = w + floor * max(w.mean(), 1e-300)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    out, r = [], 0
    for k in range(parts):
        if k == parts - 1:
            r1 = nrows
        else:
            target = cum[-1] * (k + 1) / parts
            r1 = int(np.searchsorted(cum, target))
            r1 = max(r1, r + min_rows)
            r1 = min(r1, nrows - min_rows * (parts - 1 - k))
        out.append((r, r1))
        r = r1
    return out


def decompose(nrows: int, parts: int) -> List[tuple]:
    """Balanced contiguous row blocks [row0, row1) (each >= 2 rows)."""
    if parts < 1 or nrows < 2 * parts:
        raise ValueError(f"cannot split {nrows} rows into {parts} slabs of >= 2 rows")
    base, extra = divmod(nrows, parts)
    out, r = [], 0
    for k in range(parts):
        n = base + (1 if k < extra else 0)
        out.append((r, r + n))
        r += n
    return out


class CudaSlab:
    """One slab on one GPU, driven through the C ABI's split-step entry points."""

    def __init__(self, scenario, rows: Sequence[int], device: int = 0, stream=None, fastdiv: bool = True):
        import torch
        from .simulator import Simulator
        self.torch = torch
        self.device = device
        self.sim = Simulator.from_scenario(scenario, device=device, rows=tuple(rows), fastdiv=fastdiv)
        self.L, self.h = self.sim.L, self.sim.h
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        self.sim.set_stream(self.stream.cuda_stream)
        n = int(self.L.tp_halo_bytes(self.h)) // 8
        mk = lambda: torch.empty(n, dtype=torch.float64, device=f"cuda:{device}")  # noqa: E731
        self.send = [mk(), mk()]
        self.recv = [mk(), mk()]
        self.lam = torch.zeros(1, dtype=torch.float64, device=f"cuda:{device}")
        self.row0, self.row1 = rows

    def _ptr(self, t):
        return C.c_void_p(t.data_ptr())

    def pack(self, buf: int, side: int):
        self.sim._check(self.L.tp_halo_pack(self.h, buf, side, self._ptr(self.send[side])))
        return self.send[side]

    def unpack(self, buf: int, side: int, src=None):
        src = self.recv[side] if src is None else src
        self.sim._check(self.L.tp_halo_unpack(self.h, buf, side, self._ptr(src)))

    def step_begin(self, t: float, t_next: float, t_end: float):
        self.sim._check(self.L.tp_step_begin(self.h, t, t_next, t_end))

    def bc(self, buf: int):
        self.sim._check(self.L.tp_bc(self.h, buf))

    def lambda_local(self):
        self.sim._check(self.L.tp_lambda_local(self.h, self._ptr(self.lam)))
        return self.lam

    def dt_from(self, lam):
        self.sim._check(self.L.tp_dt_from(self.h, self._ptr(lam)))

    def stage(self, corrector: int):
        self.sim._check(self.L.tp_stage(self.h, corrector))

    def step_end(self):
        t, hit, dt = C.c_double(), C.c_int(), C.c_double()
        self.sim._check(self.L.tp_step_end(self.h, C.byref(t), C.byref(hit), C.byref(dt)))
        return t.value, bool(hit.value), dt.value

    def state(self) -> np.ndarray:
        return self.sim.state()

    def audit(self) -> np.ndarray:
        return self.sim.audit_array()

    def synchronize(self):
        self.stream.synchronize()


class LocalComm:
    """All slabs live in this process (e.g. several contexts on one GPU)."""

    def exchange(self, slabs, buf: int):
        for lo, hi in zip(slabs[:-1], slabs[1:]):
            lo_n = lo.pack(buf, 1)       # lo's top interior rows -> hi's south halo
            hi_s = hi.pack(buf, 0)       # hi's bottom interior rows -> lo's north halo
            _sync_between(lo, hi)
            _sync_between(hi, lo)
            hi.unpack(buf, 0, lo_n)
            lo.unpack(buf, 1, hi_s)
            _sync_between(lo, hi)
            _sync_between(hi, lo)

    def allreduce_max(self, slabs, lams):
        import torch
        if isinstance(lams[0], torch.Tensor):
            # the lambdas were written on the slabs' streams; torch works on its current
            # stream: order both ways with host synchronisation (test-path backend)
            for s in slabs:
                s.synchronize()
            m = lams[0].clone()
            for x in lams[1:]:
                m = torch.maximum(m, x.to(m.device))
            out = [m.to(x.device) for x in lams]
            torch.cuda.synchronize()
            return out
        m = max(lams)
        return [m] * len(lams)

    def allreduce_sum(self, arrs):
        s = np.sum(np.stack(arrs), axis=0)
        return s


def _on_stream(slab):
    """torch's current stream = the slab's stream (device slabs); no-op otherwise."""
    import contextlib
    st = getattr(slab, "stream", None)
    if st is None:
        return contextlib.nullcontext()
    return slab.torch.cuda.stream(st)


def _sync_between(a, b):
    """Order b's stream after a's (device slabs); no-op on the CPU oracle."""
    sa, sb = getattr(a, "stream", None), getattr(b, "stream", None)
    if sa is not None and sb is not None and sa is not sb:
        ev = a.torch.cuda.Event()
        ev.record(sa)
        sb.wait_event(ev)


class TorchComm:
    """One slab per rank; torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, slabs, buf: int):
        (s,) = slabs
        with _on_stream(s):
            self._exchange(s, buf)

    def _exchange(self, s, buf: int):
        dist = self.dist
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, s.pack(buf, 0), self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, s.recv[0], self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, s.pack(buf, 1), self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, s.recv[1], self.rank + 1, self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if self.rank > 0:
            s.unpack(buf, 0)
        if self.rank < self.world - 1:
            s.unpack(buf, 1)

    def allreduce_max(self, slabs, lams):
        import torch
        (lam,) = lams
        t = lam if isinstance(lam, torch.Tensor) else torch.tensor([lam], dtype=torch.float64)
        with _on_stream(slabs[0]):  # collectives on the stream that wrote lambda
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return [t if isinstance(lam, torch.Tensor) else float(t.item())]

    def allreduce_sum(self, arrs):
        import torch
        (a,) = arrs
        t = torch.tensor(a, dtype=torch.float64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()


class SlabRunner:
    """Simulator::run's loop body (solver.cpp:637-649) over decomposed slabs."""

    def __init__(self, slabs, comm):
        self.slabs = list(slabs)
        self.comm = comm

    def step(self, t: float, t_next: float, t_end: float):
        S, comm = self.slabs, self.comm
        for s in S:
            s.step_begin(t, t_next, t_end)
            s.bc(0)                                      # apply_boundaries(u, t)
        comm.exchange(S, 0)
        lams = comm.allreduce_max(S, [s.lambda_local() for s in S])   # compute_dt
        for s, lam in zip(S, lams):
            s.dt_from(lam)
            s.stage(0)                                   # predictor
            s.bc(1)                                      # apply_boundaries(u*, t+dt)
        comm.exchange(S, 1)
        for s in S:
            s.stage(1)                                   # corrector
        res = [s.step_end() for s in S]
        t_new, hit, dt = res[0]
        assert all(r == res[0] for r in res), res       # dt is exact across slabs
        return t_new, hit, dt

    def steps(self, t: float, t_next: float, max_steps: int, t_end: Optional[float] = None):
        t_end = t_next if t_end is None else t_end
        dts, hit = [], False
        while t < t_end and len(dts) < max_steps:
            t, hit, dt = self.step(t, t_next, t_end)
            dts.append(dt)
            if hit:
                break
        return t, np.array(dts), hit

    def audit(self) -> np.ndarray:
        return self.comm.allreduce_sum([s.audit() for s in self.slabs]) if len(self.slabs) == 1 else \
            np.sum([s.audit() for s in self.slabs], axis=0)


class PeerGroup:
    """Slabs of one process joined by the device-resident exchange (tp_peer_connect_local):
    halo rows are stored straight into the neighbour's buffers and lambda is reduced in
    device memory inside the step graphs (tp_peer.cu), no host round trip per step.
    Every slab needs its own CUDA stream (a slab's waits must not block its neighbour)."""

    def __init__(self, slabs):
        self.slabs = list(slabs)
        n = len(self.slabs)
        streams = {id(s.stream) for s in self.slabs}
        if len(streams) != n:
            raise ValueError("PeerGroup: every slab needs its own stream")
        self.L = self.slabs[0].L
        self._hs = (C.c_void_p * n)(*[s.h.value for s in self.slabs])
        for r, s in enumerate(self.slabs):
            s.sim._check(self.L.tp_peer_connect_local(s.h, r, n, self._hs))

    def steps(self, t: float, t_next: float, max_steps: int, t_end: Optional[float] = None):
        tt, n, hit = C.c_double(t), C.c_long(), C.c_int()
        te = t_next if t_end is None else t_end
        self.slabs[0].sim._check(self.L.tp_steps_group(self._hs, len(self.slabs), t_next, te, int(max_steps),
                                                       C.byref(tt), C.byref(n), C.byref(hit)))
        return tt.value, n.value, bool(hit.value)

    def audit(self) -> np.ndarray:
        return np.sum([s.audit() for s in self.slabs], axis=0)


def peer_connect_ranks(slab: "CudaSlab", group=None) -> None:
    """One slab per process: all-gather the CUDA-IPC blobs (include/tpflow_b200.h
    TP_PEER_BLOB_BYTES) over torch.distributed and connect; afterwards every rank calls
    slab.sim.steps(...) with identical arguments."""
    import torch
    import torch.distributed as dist
    nb = 256
    blob = (C.c_ubyte * nb)()
    slab.sim._check(slab.L.tp_peer_export(slab.h, blob))
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    mine = torch.tensor(list(bytes(blob)), dtype=torch.uint8, device=dev)
    allb = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(allb, mine, group=group)
    flat = bytes(torch.cat(allb).cpu().tolist())
    buf = (C.c_ubyte * len(flat)).from_buffer_copy(flat)
    slab.sim._check(slab.L.tp_peer_connect(slab.h, rank, world, buf))


def assemble(states: Sequence[np.ndarray]) -> np.ndarray:
    """Interior rows of per-slab padded states -> the interior of the whole grid."""
    return np.concatenate([s[:, 3:-3, 3:-3] for s in states], axis=1)


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun): weak scaling, one slab per rank, device-resident exchange
# ---------------------------------------------------------------------------
def bench_scenario(args, world: int):
    """The grid bench.py runs at N = world GPUs, and the `stack` argument of the CPU
    reference on it (oracle/cpu_bench.py).  weak: one copy of the N=1 workload per GPU,
    stacked along the rows (Mode-II C3 stretches the channel instead); strong: the one
    N=1 grid split N ways."""
    from . import scenarios
    if args.config == "c1":
        base = scenarios.c1_hill(args.ncols)
    elif args.config == "c3":
        base = scenarios.SCENARIOS["c3"](args.ncols, args.nrows * (world if args.scaling == "weak" else 1))
    else:
        base = scenarios.SCENARIOS[args.config](args.ncols, args.nrows)
    if args.scaling == "strong":
        return base, 1
    if args.config == "c3":
        return base, world
    return scenarios.stacked(base, world), world


def bench_decomposition(sc, world: int, scaling: str) -> List[tuple]:
    """weak: equal rows (every slab is one copy of the workload); strong: equal work
    (wet-tile count from the initial state, decompose_balanced)."""
    if scaling == "strong":
        return decompose_balanced(row_work(sc), world)
    return decompose(sc.nrows, world)


def _peak_hbm():
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pp = os.path.join(root, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        with open(pp) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def bench_main(args, metric: str, clock_sampler=None) -> None:
    """One slab per rank of the bench grid (bench_scenario), joined by the device-resident
    exchange (tp_peer.cu over CUDA IPC / NVLink).  Timed: K steps of the device loop on
    every rank along the run's output schedule, CUDA events on the launching stream, max
    over ranks.  Also: the stage kernels' roofline per rank (processed-tile bytes, max over
    ranks of the kernel time), e2e through the C ABI with pinned host buffers, and the CPU
    reference on the same grid (rank 0)."""
    import json
    import time
    import torch
    import torch.distributed as dist
    import bench as B

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    dev = local % ndev  # one GPU per rank; fewer GPUs than ranks only for functional runs
    torch.cuda.set_device(dev)
    nccl = ndev >= world
    if not dist.is_initialized():
        dist.init_process_group("nccl" if nccl else "gloo",
                                **({"device_id": torch.device(f"cuda:{dev}")} if nccl else {}))

    def reduce_max(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        if nccl:
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu()]

    def reduce_sum(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        if nccl:
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return [float(x) for x in t.cpu()]

    sc, stack = bench_scenario(args, world)
    parts = bench_decomposition(sc, world, args.scaling)
    rows = parts[rank]
    stream = torch.cuda.Stream()
    slab = CudaSlab(sc, rows, device=dev, stream=stream)
    peer_connect_ranks(slab)
    sim = slab.sim
    sim.set_option("graph_steps", args.graph_steps)
    clock = B.RunClock(sim)

    clock.advance(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = clock_sampler(dev) if clock_sampler else None
    if clocks:
        clocks.__enter__()
    ms_local = B.timed_steps(sim, clock, stream, args.steps)
    if clocks:
        clocks.__exit__(None, None, None)
    launches = sim.kernel_launches()
    act_p, act_c, ntiles = sim.active_tiles()
    ms, = reduce_max([ms_local])
    cells = sc.ncols * sc.nrows
    value = cells * args.steps / (ms / 1e3) / 1e9

    # roofline of the stage kernels on this rank's slab; whole-job: processed bytes of all
    # ranks over the slowest rank's kernel time, against world x the per-GPU peak
    peak, peak_src = _peak_hbm()
    slab_cells = sc.ncols * (rows[1] - rows[0])
    rl = B.stage_roofline(sim, clock, slab_cells, args.roofline_reps, peak)
    kms, = reduce_max([rl["kernel_ms_per_step"]])
    alg_all, = reduce_sum([rl["alg_bytes_per_step"]])
    achieved = alg_all / (kms / 1e3) / 1e9 / world
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "kernel": "stage_kernel<pred>+stage_kernel<corr> per step, per GPU: processed-tile "
                          "algorithmic bytes of all ranks / N / the slowest rank's kernel time",
                "peak_source": peak_src, "kernel_ms_per_step_max": round(kms, 4),
                "rank0": {k: rl[k] for k in ("frac", "kernel_ms_per_step", "processed_tile_frac")}}
    nt = B.ncu_traffic()
    if nt:
        for cand in (nt, nt.get("wet"), nt.get("c5")):
            if cand and cand.get("grid") == [sc.ncols, (rows[1] - rows[0])] and cand.get("config") == args.config:
                roofline["traffic"] = cand["dram_bytes_per_step"]

    # e2e: the same steps through the C ABI with this rank's state from / to pinned host memory
    import ctypes as Cc
    nbytes = 6 * sim.ny * sim.nx * 8
    h_in = torch.empty(6 * sim.ny * sim.nx, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty_like(h_in, pin_memory=True)  # empty_like alone is pageable
    assert h_in.is_pinned() and h_out.is_pinned()
    dp = Cc.POINTER(Cc.c_double)
    sim._check(sim.L.tp_get_state(sim.h, Cc.cast(h_in.data_ptr(), dp)))
    sim._check(sim.L.tp_get_state(sim.h, Cc.cast(h_out.data_ptr(), dp)))
    torch.cuda.synchronize()
    dist.barrier()
    w0 = time.perf_counter()
    sim._check(sim.L.tp_set_state(sim.h, Cc.cast(h_in.data_ptr(), dp)))
    ne = clock.advance(args.steps)
    sim._check(sim.L.tp_get_state(sim.h, Cc.cast(h_out.data_ptr(), dp)))
    w, = reduce_max([time.perf_counter() - w0])
    e2e_v = cells * ne / w / 1e9
    h2d_all, = reduce_sum([float(nbytes)])

    cpu = None
    if rank == 0 and not args.no_cpu:
        lanes = os.cpu_count() or 1
        try:
            c = B.cpu_reference(args.config, args.ncols, args.nrows, max(1, args.cpu_steps // max(stack, 1)),
                                lanes, stack=stack)
            cpu = {"value": round(c["value"] / 1e9, 6), "unit": "GCUPS", "cores": c["lanes"],
                   "kind": "reference" if c["kind"] == "ref" else "port",
                   "sample": f"{c['steps']} steps of the same {sc.ncols}x{sc.nrows} grid from t=0 "
                             f"(after 1 untimed step), BackendConfig::parallel({c['lanes']})",
                   "seconds": round(c["seconds"], 3)}
        except Exception as e:  # noqa: BLE001 - reported, not fatal to the GPU arm
            cpu = {"unavailable": str(e)[:200]}
    if rank == 0:
        cfg = B.workload_config(sc)
        cfg.update({"parallelism": f"slab{world}", "scaling_mode": args.scaling,
                    "slab_rows": [int(r1 - r0) for r0, r1 in parts],
                    "decomposition": ("equal work: wet-tile rows of the initial state (decompose_balanced)"
                                      if args.scaling == "strong" else "equal rows: one workload copy per GPU"),
                    "exchange": "halo rows stored into the neighbour's buffers over peer memory, "
                                "lambda all-reduce in device memory (tp_peer.cu)",
                    "gpus_visible": ndev, "graph_steps": args.graph_steps,
                    "l2": ("per-rank inputs larger than L2" if 18 * sim.ny * sim.nx * 8 > 126e6 else
                           "per-rank inputs fit in L2 (functional size)"),
                    "active_tiles_last_step_rank0": [act_p, act_c, ntiles]})
        out = {"metric": metric, "value": round(value, 4), "unit": "GCUPS", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
               "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
               "data": f"synthetic (deterministic {sc.name} generator in scenarios.py; no network data)",
               "config": cfg,
               "e2e": {"value": round(e2e_v, 4), "unit": "GCUPS",
                       "h2d_bytes_per_step": int(h2d_all) // max(ne, 1),
                       "d2h_bytes_per_step": int(h2d_all) // max(ne, 1),
                       "mode": f"every rank: tp_set_state(pinned host) + tp_steps({ne}) + tp_get_state, "
                               f"wall clock, max over ranks"},
               "roofline": roofline, "cpu_baseline": cpu,
               "clocks": clocks.summary() if clocks else None,
               "gpu_launches": launches}
        print(json.dumps(out))
    dist.barrier()
