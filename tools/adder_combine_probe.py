"""Adder N=32: exact (bit-identical) vs combined diagonal runs (within 1e-12): wall time
of run_circuit (second call) and the reports' largest difference."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200 import _native as nat  # noqa: E402
from paper_2511_03359_b200.device import jit_wait  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 16
circ, regs = pb.build_adder(w, [47302 % (1 << w), 18233 % (1 << w)])
out = {}
for exact in (True, False):
    pb.run_circuit(circ, exact_diagonals=exact)
    jit_wait()
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        res = pb.run_circuit(circ, exact_diagonals=exact)
        ts.append(time.perf_counter() - t0)
    nat.pass_timing(True)
    nat.pass_timing_read()
    res = pb.run_circuit(circ, exact_diagonals=exact)
    nat.pass_timing(False)
    cnt, ms, _ = nat.pass_timing_read()
    out[exact] = res.report
    kat = all(abs(res.report.qz[q] - 1.0) < 1e-12 for q in regs["R2"])
    print(f"exact={exact}: {min(ts):.4f} s, {cnt} passes {ms:.1f} ms, R2 all ones {kat}, "
          f"launches {res.device_stats['kernel_launches']}", flush=True)
print("report max difference:", out[True].max_difference(out[False]))
