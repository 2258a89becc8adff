"""Probe: fused C2 layers in FP32 storage vs FP64 at N (default 32): ms per layer and the
effective GB/s of the passes (algorithmic bytes 2 * bpe * 2^N per pass)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat
from paper_2511_03359_b200.device import DeviceState, jit_prepare, jit_wait
from paper_2511_03359_b200.engine import gate_to_op
from tests.circuits import to_product
from oracle.ref_builders import OCircuit
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
layers = [[gate_to_op(g) for g in to_product(OCircuit(n, tuple(l))).gates] for l in bench.workload_layers(n, 4)]
for mode in (pb.PrecisionMode.FP64, pb.PrecisionMode.FP32):
    for o in layers:
        jit_prepare(n, o, 12, nat.mode_code(mode))
    jit_wait()
    dev = DeviceState(n, mode)
    dev.zero(0)
    for o in layers:
        dev.apply_fused(o)
    dev.synchronize()
    nat.pass_timing(True)
    nat.pass_timing_read()
    e0, e1 = nat.Event(), nat.Event()
    e0.record(dev.stream)
    for o in layers[1:]:
        dev.apply_fused(o)
    e1.record(dev.stream)
    dev.synchronize()
    p, ms, by = nat.pass_timing_read()
    nat.pass_timing(False)
    print(f"{mode.name}: {e0.elapsed_ms(e1) / (len(layers) - 1):.1f} ms/layer, {p} passes, "
          f"{by / (ms / 1e3) / 1e9:.0f} GB/s per pass", flush=True)
    dev.free()
print("done", flush=True)
