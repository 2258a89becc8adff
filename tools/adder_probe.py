"""Probe: time the QFT adder through run_circuit and report launches / pass timing."""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat

w = int(sys.argv[1]) if len(sys.argv) > 1 else 16
circ, regs = pb.build_adder(w, [47302 % (1 << w), 18233 % (1 << w)])
pb.run_circuit(pb.build_adder(4, [3, 12])[0])
for rep in range(3):
    l0 = nat.launch_count()
    nat.pass_timing(True)
    nat.pass_timing_read()
    t0 = time.perf_counter()
    res = pb.run_circuit(circ)
    t = time.perf_counter() - t0
    nat.pass_timing(False)
    passes, ms, byts = nat.pass_timing_read()
    print(f"N={circ.n_qubits} gates={len(circ.gates)} wall={t:.4f}s launches={nat.launch_count() - l0} "
          f"fused passes={passes} pass_ms={ms:.2f} stats={res.device_stats}", flush=True)
    del res
    from paper_2511_03359_b200.device import jit_stats, jit_wait
    t0 = time.perf_counter()
    jit_wait()
    print(f"jit_wait {time.perf_counter() - t0:.3f}s {jit_stats()}", flush=True)
