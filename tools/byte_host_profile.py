"""Host side of the BYTE per-gate barrier: cProfile of gates 40..80 of the BYTE adder
(the CPHASE runs) after the first 40 gates, next to their wall time."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200.byte_state import ByteEngineState  # noqa: E402
from paper_2511_03359_b200.layout import PartitionLayout  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
w = n // 2
circ, _ = pb.build_adder(w, [(1 << w) - 1 - 0x55 % (1 << w), 0x55 % (1 << w)])
st = ByteEngineState(n, PartitionLayout(n, n))
st.zero(0)
gates = [g for g in circ.gates if g.kind != "M"]
for g in gates[:40]:
    st.apply_gate(g)
st.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for g in gates[40:80]:
    st.apply_gate(g)
st.synchronize()
pr.disable()
dt = time.perf_counter() - t0
print(f"gates 40..80: {dt * 1e3 / 40:.3f} ms/gate")
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
