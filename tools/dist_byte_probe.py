"""Probe (torchrun): BYTE benchmark through run_circuit_distributed with per-phase timing
of the backend's gate loop (device passes vs host barrier)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed as dist

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import distributed as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = n + (world.bit_length() - 1)
acc = {}
for name in ("apply_gate", "swap", "swap_group", "measure_local", "pair_dot"):
    orig = getattr(D.CudaByteBackend, name)

    def wrap(self, *a, _orig=orig, _name=name, **k):
        t = time.perf_counter()
        r = _orig(self, *a, **k)
        self.st.synchronize()
        acc[_name] = acc.get(_name, 0.0) + time.perf_counter() - t
        return r
    setattr(D.CudaByteBackend, name, wrap)
orig_pass = D.CudaByteBackend._pass


def timed_pass(self, *a, **k):
    self.st.synchronize()
    t = time.perf_counter()
    r = orig_pass(self, *a, **k)
    acc["_pass"] = acc.get("_pass", 0.0) + time.perf_counter() - t
    return r


D.CudaByteBackend._pass = timed_pass
orig_ct = D.ByteDeviceState.collect_tagged if hasattr(D, "ByteDeviceState") else None
from paper_2511_03359_b200.byte_state import ByteDeviceState
orig_ct = ByteDeviceState.collect_tagged


def timed_ct(self, *a, **k):
    self.synchronize()
    t = time.perf_counter()
    r = orig_ct(self, *a, **k)
    acc["collect_tagged"] = acc.get("collect_tagged", 0.0) + time.perf_counter() - t
    return r


ByteDeviceState.collect_tagged = timed_ct
circ = pb.build_benchmark(N)
for rep in range(2):
    acc.clear()
    dist.barrier()
    t0 = time.perf_counter()
    res = D.run_circuit_distributed(circ, dist, mode=pb.PrecisionMode.BYTE, device=rank)
    t = time.perf_counter() - t0
    if rank == 0:
        print(f"rep {rep}: total {t:.3f}s gates {len(circ.gates) - 1} stats {res.device_stats} "
              + " ".join(f"{k}={v:.3f}" for k, v in sorted(acc.items())), flush=True)
    res.backend.close()
    res.backend.st.free()
    del res
dist.destroy_process_group()
