"""Run ONE fused pass of the C2 bench layers (the library's own split), for ncu.

    python tools/one_pass.py N LAYER PASS [cfg=9] [reps=1]
    ncu --set full --profile-from-start off -k sv_pass -c 1 python tools/one_pass.py 32 1 2

The pass is compiled (specialised) and run once untimed, then `reps` launches run
between cudaProfilerStart/Stop; it prints the pass's ops and its event time.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200 import _native as nat  # noqa: E402
from paper_2511_03359_b200.device import DeviceState, jit_prepare, jit_wait, ops_array  # noqa: E402
from paper_2511_03359_b200.engine import gate_to_op  # noqa: E402
from oracle.ref_builders import OCircuit  # noqa: E402
from tests.circuits import to_product  # noqa: E402

n, li, pi = (int(x) for x in sys.argv[1:4])
cfg = int(sys.argv[4]) if len(sys.argv) > 4 else 9
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
lib = nat.load()
if li < 0:     # LAYER -1: build_adder(N // 2, ...) (BASELINE config 3 at N=32)
    circ = pb.build_adder(n // 2, [47302 % (1 << (n // 2)), 18233 % (1 << (n // 2))])[0]
    ops = [gate_to_op(g) for g in circ.gates if g.kind != "M"]
else:
    lay = bench.workload_layers(n, 9)[li]
    ops = [gate_to_op(g) for g in to_product(OCircuit(n, tuple(lay))).gates]


def plan(c):
    nat.check(lib.sv_fused_variant(c))
    ends = (ctypes.c_int * 256)()
    k = lib.sv_plan_passes(n, nat.SV_FP64, ops_array(ops), len(ops), 12, ends, 256)
    return [ends[i] for i in range(k)]


if cfg == 9:
    cfg = 8 if len(plan(8)) < len(plan(6)) else 6
ends = plan(cfg)
a = 0 if pi == 0 else ends[pi - 1]
sub = ops[a:ends[pi]]
dev = DeviceState(n, pb.PrecisionMode.FP64)
dev.zero(0)
jit_prepare(n, sub, 12)
jit_wait()
dev.apply_fused(sub)
dev.synchronize()
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
e0, e1 = nat.Event(), nat.Event()
if cudart:
    cudart.cudaProfilerStart()
e0.record(dev.stream)
for _ in range(reps):
    dev.apply_fused(sub)
e1.record(dev.stream)
dev.synchronize()
if cudart:
    cudart.cudaProfilerStop()
kinds = [{1: "1q", 2: "2q"}.get(o.kind, "diag") for o in sub]
print(f"N={n} layer {li} pass {pi} cfg {cfg}: {len(sub)} ops {kinds} {e0.elapsed_ms(e1) / reps:.2f} ms")
