"""Probe: wall time of the all-qubit measurement (sv_measure) on a 2^n FP64 state."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200.device import DeviceState

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dev = DeviceState(n, pb.PrecisionMode.FP64)
dev.zero(0)
for q in range(n):
    dev.apply_1q(q, pb.gates.H_MATRIX)
dev.synchronize()
norm, ones, cross = dev.measure()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    norm, ones, cross = dev.measure()
    ts.append(time.perf_counter() - t0)
t = min(ts)
print(f"n={n} measure {t * 1e3:.2f} ms  read-equivalent {2 ** n * 16 / t / 1e9:.0f} GB/s per state read  "
      f"norm={norm:.15f} max|ones-0.5|={np.max(np.abs(ones - 0.5)):.2e} "
      f"max|cross.re-0.5|={np.max(np.abs(cross.real - 0.5)):.2e}", flush=True)
