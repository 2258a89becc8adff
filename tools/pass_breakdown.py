"""Per-pass timing of the C2 bench layers: ops, segments and ms of every fused pass."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat
from paper_2511_03359_b200.device import DeviceState
from paper_2511_03359_b200.engine import gate_to_op
from tests.circuits import to_product
from oracle.ref_builders import OCircuit
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 6
nat.check(nat.load().sv_fused_variant(cfg))
layers_o = bench.workload_layers(n, 4)
dev = DeviceState(n, pb.PrecisionMode.FP64)
dev.zero(0)
for li, lo in enumerate(layers_o):
    gates = to_product(OCircuit(n, tuple(lo))).gates
    kinds = {}
    for g in gates:
        kinds[g.kind] = kinds.get(g.kind, 0) + 1
    nat.pass_timing(True)
    nat.pass_timing_read()
    # one apply per gate prefix to learn the pass split: time the whole layer, then per pass
    dev.apply_fused([gate_to_op(g) for g in gates])
    dev.synchronize()
    p, ms, by = nat.pass_timing_read()
    nat.pass_timing(False)
    print(f"layer {li}: {len(gates)} gates {kinds} -> {p} passes, {ms:.2f} ms, "
          f"{by / (ms / 1e3) / 1e9:.0f} GB/s per pass", flush=True)
