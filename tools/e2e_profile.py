"""Where an e2e run_circuit call's time goes (GPU box): the bench's e2e circuit (H layer +
random layer + measure-all, N=33), one warm-up call, then timed calls with the fused
passes' device time (sv_pass_timing) and a cProfile of the host side.

    python tools/e2e_profile.py [N=33] [layer=1]
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200 import _native as nat  # noqa: E402
from tests.circuits import to_product  # noqa: E402
from oracle.ref_builders import OCircuit  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
li = int(sys.argv[2]) if len(sys.argv) > 2 else 1
layers = bench.workload_layers(n, 9)
circ = to_product(OCircuit(n, tuple(layers[0]) + tuple(layers[li]) + (pb.gates.measure_all(),)))
gates_only = to_product(OCircuit(n, tuple(layers[0]) + tuple(layers[li])))
for c in (circ, gates_only):
    pb.run_circuit(c)
for label, c in (("gates+M", circ), ("gates only", gates_only)):
    for rep in range(2):
        nat.pass_timing(True)
        nat.pass_timing_read()
        t0 = time.perf_counter()
        res = pb.run_circuit(c)
        _ = res.report.qz[0] if res.report else None
        wall = time.perf_counter() - t0
        nat.pass_timing(False)
        passes, ms, by = nat.pass_timing_read()
        print(f"{label}: wall {wall * 1e3:.1f} ms, {passes} fused passes {ms:.1f} ms device, "
              f"stats {res.device_stats.get('support')}", flush=True)
        del res
pr = cProfile.Profile()
pr.enable()
res = pb.run_circuit(circ)
pr.disable()
del res
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
