"""Probe (torchrun): where run_circuit_distributed's time goes for one C2 layer + M at
2^n amplitudes per GPU: backend setup (alloc + zero + IPC maps), gates, measure, close."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed as dist

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import distributed as D
from paper_2511_03359_b200.device import jit_wait
from tests.circuits import to_product
from oracle.ref_builders import OCircuit
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
which = sys.argv[2] if len(sys.argv) > 2 else "layer"
remap = (sys.argv[3] != "ref") if len(sys.argv) > 3 else True
N = n + (world.bit_length() - 1)
if which == "bench":
    circ = pb.build_benchmark(N)
else:
    layer = to_product(OCircuit(N, tuple(bench.workload_layers(N, 2)[1]))).gates
    circ = pb.Circuit(N, tuple(layer) + (pb.gates.measure_all(),))
orig_init = D.CudaBackend.__init__
orig_measure = D._measure
marks = {}


def timed_init(self, *a, **k):
    t0 = time.perf_counter()
    orig_init(self, *a, **k)
    self.dev.synchronize()
    marks["setup"] = time.perf_counter() - t0


def timed_measure(be, *a, **k):
    be.dev.synchronize()
    marks["gates_end"] = time.perf_counter()
    r = orig_measure(be, *a, **k)
    marks["measure"] = time.perf_counter() - marks["gates_end"]
    return r


D.CudaBackend.__init__ = timed_init
for name in ("measure_local", "pair_dot", "close", "swap", "swap_group", "apply_local"):
    orig = getattr(D.CudaBackend, name)

    def wrap(self, *a, _orig=orig, _name=name, **k):
        self.dev.synchronize()
        t = time.perf_counter()
        r = _orig(self, *a, **k)
        self.dev.synchronize()
        marks.setdefault("calls", []).append((_name, round(time.perf_counter() - t, 4)))
        return r
    setattr(D.CudaBackend, name, wrap)
D._measure = timed_measure
for rep in range(3):
    dist.barrier()
    t0 = time.perf_counter()
    from paper_2511_03359_b200 import _native as nat
    nat.pass_timing(True)
    nat.pass_timing_read()
    res = D.run_circuit_distributed(circ, dist, device=rank, remap=remap)
    passes, pass_ms, _ = nat.pass_timing_read()
    nat.pass_timing(False)
    t1 = time.perf_counter()
    res.backend.close()
    res.backend.dev.free()
    t2 = time.perf_counter()
    if rank == 0:
        print("calls", marks.pop("calls", []), flush=True)
    marks.pop("calls", None)
    if rank == 0:
        print(f"rep {rep}: total {t1 - t0:.3f}s setup {marks['setup']:.3f}s measure {marks['measure']:.3f}s "
              f"gates {t1 - t0 - marks['setup'] - marks['measure']:.3f}s close {t2 - t1:.3f}s passes {passes} "
              f"pass_ms {pass_ms:.1f} stats {res.device_stats}",
              flush=True)
    del res
    jit_wait()
dist.destroy_process_group()
