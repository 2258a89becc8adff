"""Probe: where the end-to-end run_circuit time goes at N (default 33): create, zero,
fused layer, measure, destroy -- each timed with a device sync."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat
from paper_2511_03359_b200.device import DeviceState, jit_prepare, jit_wait
from paper_2511_03359_b200.engine import gate_to_op
from tests.circuits import to_product
from oracle.ref_builders import OCircuit
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
layer = to_product(OCircuit(n, tuple(bench.workload_layers(n, 2)[1]))).gates
ops = [gate_to_op(g) for g in layer]
jit_prepare(n, ops)
jit_wait()
for rep in range(3):
    t = [time.perf_counter()]
    dev = DeviceState(n, pb.PrecisionMode.FP64)
    dev.synchronize(); t.append(time.perf_counter())
    dev.zero(0)
    dev.synchronize(); t.append(time.perf_counter())
    dev.apply_fused(ops)
    dev.synchronize(); t.append(time.perf_counter())
    dev.measure()
    t.append(time.perf_counter())
    dev.free()
    t.append(time.perf_counter())
    circ = pb.Circuit(n, tuple(layer) + (pb.gates.measure_all(),))
    t0 = time.perf_counter()
    res = pb.run_circuit(circ)
    t_rc = time.perf_counter() - t0
    del res
    d = [round((b - a) * 1e3, 1) for a, b in zip(t, t[1:])]
    print(f"rep {rep}: create {d[0]} zero {d[1]} layer {d[2]} measure {d[3]} free {d[4]} ms; "
          f"run_circuit {t_rc * 1e3:.1f} ms", flush=True)
