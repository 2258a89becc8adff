"""Time single fused passes with chosen op mixes (GPU microbenchmark, not a test)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat, gates as g
from paper_2511_03359_b200.device import DeviceState
from paper_2511_03359_b200.engine import gate_to_op
from tests.circuits import haar_unitary

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(1)
dev = DeviceState(n, pb.PrecisionMode.FP64)
dev.zero(0)
u2 = lambda q: g.u2(q, haar_unitary(rng, 2))
u4 = lambda a, b: g.u4(a, b, haar_unitary(rng, 4))
cases = {
    "diag-only(Z@20)": [g.z(20)],
    "1xH@0": [g.h(0)],
    "1xH@20": [g.h(20)],
    "4xH@20-23": [g.h(q) for q in (20, 21, 22, 23)],
    "7xH@20-26": [g.h(q) for q in range(20, 27)],
    "12xH@0-11": [g.h(q) for q in range(12)],
    "4xU2@20-23": [u2(q) for q in (20, 21, 22, 23)],
    "8xU2@20-27": [u2(q) for q in range(20, 28)],
    "2xU4": [u4(20, 21), u4(22, 23)],
    "4xU4": [u4(20, 21), u4(22, 23), u4(24, 25), u4(26, 20)],
    "8xU2@20-23x2": [u2(q) for q in (20, 21, 22, 23)] * 2,
    "8xH@20-27": [g.h(q) for q in range(20, 28)],
    "16xU2@20-23x4": [u2(q) for q in (20, 21, 22, 23)] * 4,
    "6xH@20-25": [g.h(q) for q in range(20, 26)],
    "6xU2@20-25": [u2(q) for q in range(20, 26)],
    "6xH@20-25x2": [g.h(q) for q in range(20, 26)] * 2,
    "3xU4@20-25": [u4(20, 21), u4(22, 23), u4(24, 25)],
    "mix8": [g.h(20), u2(21), g.cnot(22, 23), u4(24, 20), g.cphase(21, 25, 3), g.x(26), g.phase(22, 2), u2(25)],
}
if len(sys.argv) > 3:
    cases = {k: v for k, v in cases.items() if k in sys.argv[3].split(",")}
bytes_pass = 2 * 16 * (1 << n)
variants = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "3"])]
for variant in variants:
    nat.check(nat.load().sv_fused_variant(variant))
    for name, gl in cases.items():
        ops = [gate_to_op(x) for x in gl]
        dev.apply_fused(ops)  # warm
        e0, e1 = nat.Event(), nat.Event()
        e0.record(dev.stream)
        reps = 5
        for _ in range(reps):
            dev.apply_fused(ops)
        e1.record(dev.stream)
        ms = e0.elapsed_ms(e1) / reps
        print(f"{variant} {name:18s} {ms:8.3f} ms  {bytes_pass / ms / 1e6:8.1f} GB/s per pass", flush=True)
