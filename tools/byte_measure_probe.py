"""Probe: repeated BYTE measure-all timings on a Hadamard-benchmark state (one GPU)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200.byte_state import ByteEngineState
from paper_2511_03359_b200.layout import PartitionLayout

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
circ = pb.build_benchmark(n)
st = ByteEngineState(n, PartitionLayout(n, n))
st.zero(0)
for g in circ.gates[:-1]:
    st.apply_gate(g)
st.synchronize()
for rep in range(4):
    t0 = time.perf_counter()
    norm, ones, cross = st.measure_sums()
    print(f"n={n} BYTE measure {1e3 * (time.perf_counter() - t0):.2f} ms norm={norm:.15f}", flush=True)
