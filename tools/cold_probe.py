"""Where the first run_circuit of a fresh process spends its time (N=33 C2 layer + M):
allocation, planning + disk-cache lookup, fused passes (module loads), measure-all.
Run twice on one box: the first process fills the on-disk cubin cache."""
import json
import os
import sys
import time

t_start = time.perf_counter()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes  # noqa: E402

import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200 import _native as nat  # noqa: E402
from paper_2511_03359_b200.device import DeviceState, jit_prepare, jit_stats  # noqa: E402
from paper_2511_03359_b200.engine import gate_to_op  # noqa: E402
from oracle.ref_builders import OCircuit  # noqa: E402
from tests.circuits import to_product  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
lay = bench.workload_layers(n, 9)[1]
ops = [gate_to_op(g) for g in to_product(OCircuit(n, tuple(lay))).gates]
c = ctypes.c_int(0)
nat.check(nat.load().sv_device_count(ctypes.byref(c)))
t = {"import": time.perf_counter() - t_start}
t0 = time.perf_counter()
free, tot = ctypes.c_uint64(0), ctypes.c_uint64(0)
nat.check(nat.load().sv_mem_info(0, ctypes.byref(free), ctypes.byref(tot)))
t["context"] = time.perf_counter() - t0
for rep in range(2):
    r = {}
    t0 = time.perf_counter()
    dev = DeviceState(n, pb.PrecisionMode.FP64)
    dev.zero(0, lazy=True)
    dev.synchronize()
    r["alloc"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    jit_prepare(n, ops)
    r["jit_prepare"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev.apply_fused(ops)
    dev.synchronize()
    r["passes"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev.measure()
    r["measure"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev.free()
    r["free"] = time.perf_counter() - t0
    t[f"rep{rep}"] = {k: round(v * 1e3, 1) for k, v in r.items()}
t["jit"] = jit_stats()
print(json.dumps(t))
