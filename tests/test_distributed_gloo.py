"""world_size-2/4 gloo tests of the multi-rank control plane (CPU, no GPU).

Real processes, real torch.distributed collectives; the device is the numpy
stand-in of tests/fake_backend.py.  Checks: remapped multi-rank execution is
bit-identical to the oracle, reports match, reference ledgers match the
reference's accounting.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, outq):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_03359_b200.distributed import run_circuit_distributed
        from tests.circuits import random_circuit, to_product
        from tests.fake_backend import NumpyBackend
        from oracle.ref_builders import benchmark
        if case == "random":
            circ = random_circuit(np.random.default_rng(7), 7, 40)
        else:
            circ = benchmark(9)
        res = run_circuit_distributed(to_product(circ), dist, backend_factory=NumpyBackend)
        state = res.gathered_state(dist)
        if rank == 0:
            outq.put((state, res.report.qx, res.report.qy, res.report.qz, res.report.norm_deviation,
                      [l.snapshot() for l in res.ledgers], res.device_stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "random"), (4, "random"), (2, "bench"), (4, "bench")])
def test_distributed_control_plane_gloo(world, case):
    from oracle import ref_engine
    from oracle.ref_builders import benchmark
    from tests.circuits import random_circuit
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    state, qx, qy, qz, dev, ledgers, stats = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    circ = random_circuit(np.random.default_rng(7), 7, 40) if case == "random" else benchmark(9)
    want = ref_engine.run_circuit(circ, ranks=world)
    assert np.array_equal(state, want.gathered_state())
    wx, wy, wz, wd = want.report
    assert max(np.max(np.abs(np.array(qx) - wx)), np.max(np.abs(np.array(qy) - wy)),
               np.max(np.abs(np.array(qz) - wz))) < 1e-12
    assert ledgers == want.ledgers
    assert stats["swaps"] >= 0


class _CountingDist:
    """Stand-in process group: all_gather_object reports this rank's object for every rank,
    except the ranks listed in `peer_objs` (to simulate a peer whose cache differs)."""

    def __init__(self, rank=0, world=2):
        self.rank, self.world, self.barriers = rank, world, 0
        self.peer_objs = {}

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.world

    def barrier(self):
        self.barriers += 1

    def all_gather_object(self, out, obj):
        for r in range(self.world):
            out[r] = self.peer_objs.get(r, obj) if r != self.rank else obj


def test_peer_map_cache_decisions(monkeypatch):
    """Cached peer mappings (distributed.py _PEER_MAPS): same shape on every rank keeps
    them with no barrier; another shape, a BYTE run, or ANY rank reporting a stale cache
    closes every mapping on every rank, holds a barrier and drops the IPC export marks."""
    from paper_2511_03359_b200 import distributed as D
    closed, unexports = [], []

    class _Lib:
        def sv_ipc_close(self, device, p):
            closed.append((device, p))
            return 0

        def sv_ipc_unexport_all(self, out):
            unexports.append(1)
            return 0
    monkeypatch.setattr(D.nat, "load", lambda *a, **k: _Lib())
    monkeypatch.setattr(D, "_PEER_MAPS", {})
    d = _CountingDist()
    maps = D._prepare_peer_maps(d, 0, (30, 1))          # empty cache: collective close path
    assert maps == {} and d.barriers == 1 and len(unexports) == 1
    maps[1] = (b"h1", "p1")
    again = D._prepare_peer_maps(d, 0, (30, 1))
    assert again is maps and d.barriers == 1 and not closed
    d.peer_objs[1] = (True, (30, 1))                      # the peer's cache is stale: we follow
    again = D._prepare_peer_maps(d, 0, (30, 1))
    assert again == {} and d.barriers == 2 and closed == [(0, "p1")] and len(unexports) == 2
    d.peer_objs.clear()
    again[1] = (b"h1", "p1")
    other = D._prepare_peer_maps(d, 0, (29, 1))
    assert other == {} and d.barriers == 3 and closed[-1] == (0, "p1")
    other[1] = (b"h2", "p2")
    D._prepare_peer_maps(d, 0, ("byte", 29))
    assert d.barriers == 4 and closed[-1] == (0, "p2")
    D.release_peer_maps(d)
    assert D._PEER_MAPS == {} and d.barriers == 5 and len(unexports) == 5


def _gather_worker(rank, world, port, outq):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_03359_b200.distributed import all_gather_candidates
        rng = np.random.default_rng(100 + rank)
        mine = []
        for r in range(world):      # ragged, empty and -0.0 entries
            nm, npp = int(rng.integers(0, 5)) * (r != rank), int(rng.integers(0, 4))
            mags = rng.random(nm)
            ph = rng.normal(size=npp) + 1j * rng.normal(size=npp)
            if npp:
                ph[0] = complex(-0.0, 0.0)
            mine.append((mags, ph))
        fast = all_gather_candidates(dist, mine)
        ref = [None] * world
        dist.all_gather_object(ref, mine)
        same = all(len(a) == len(b) and all(
            x[0].tobytes() == y[0].tobytes() and x[1].tobytes() == y[1].tobytes() and x[1].dtype == y[1].dtype
            for x, y in zip(a, b)) for a, b in zip(fast, ref))
        outq.put((rank, same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_candidate_all_gather_equals_all_gather_object(world):
    """The BYTE barrier's tensor all-gather returns exactly what all_gather_object does."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(same for _, same in got), got
