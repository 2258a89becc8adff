"""Where the first BYTE gate of a process spends its time (cProfile of apply_gate)."""
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
circ = pb.build_benchmark(n)
t0 = time.perf_counter()
st = ByteEngineState(n, PartitionLayout(n, n))
st.zero(0)
st.synchronize()
print(f"create+zero {1e3 * (time.perf_counter() - t0):.1f} ms")
for k in range(3):
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    st.apply_gate(circ.gates[k])
    st.synchronize()
    pr.disable()
    print(f"gate {k}: {1e3 * (time.perf_counter() - t0):.2f} ms")
    if k == 0:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
