"""Time BYTE-mode gates (single GPU): benchmark H sweep and adder phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2511_03359_b200 as pb
from paper_2511_03359_b200.byte_state import ByteEngineState
from paper_2511_03359_b200.layout import PartitionLayout

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
which = sys.argv[2] if len(sys.argv) > 2 else "bench"
if which == "bench":
    circ = pb.build_benchmark(n)
else:
    w = n // 2
    circ, _ = pb.build_adder(w, [(1 << w) - 1 - 0x55 % (1 << w), 0x55 % (1 << w)])
layout = PartitionLayout(circ.n_qubits, circ.n_qubits)
st = ByteEngineState(circ.n_qubits, layout)
st.zero(0)
st.time_passes = True
st.pass_events = []
times = []
for gate in circ.gates:
    if gate.kind == "M":
        t0 = time.perf_counter()
        norm, ones, cross = st.measure_sums()
        tm = time.perf_counter() - t0
        continue
    t0 = time.perf_counter()
    ne = len(st.pass_events)
    prof = os.environ.get("BYTE_PROBE_PROFILE_GATE") == str(len(times))   # ncu --profile-from-start off
    if prof:
        import torch
        torch.cuda.cudart().cudaProfilerStart()
    st.apply_gate(gate)
    st.synchronize()
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    times.append((gate.kind, time.perf_counter() - t0))
    if os.environ.get("BYTE_PROBE_VERBOSE"):
        ev = [("s" if sc else "w") + f"{a.elapsed_ms(b):.2f}" for sc, a, b in st.pass_events[ne:]]
        print(f"  {gate.kind}{tuple(gate.qubits) if hasattr(gate, 'qubits') else ''} {times[-1][1]*1e3:.2f} ms "
              f"passes {' '.join(ev)} mags {len(st.codebook.mags)}", flush=True)
byt = 4 * (1 << circ.n_qubits)
ts = np.array([t for _, t in times])
scan = [a.elapsed_ms(b) for sc, a, b in st.pass_events if sc]
wr = [a.elapsed_ms(b) for sc, a, b in st.pass_events if not sc]
print(f"  device: scan passes {len(scan)} median {np.median(scan) if scan else 0:.2f} ms; "
      f"write passes {len(wr)} median {np.median(wr):.2f} ms -> {byt / (np.median(wr) / 1e3) / 1e9:.0f} GB/s")
print(f"BYTE {which} N={circ.n_qubits}: {len(ts)} gates, median {np.median(ts)*1e3:.2f} ms/gate "
      f"({byt / np.median(ts) / 1e9:.0f} GB/s eff), mean {ts.mean()*1e3:.2f} ms, max {ts.max()*1e3:.1f} ms; "
      f"passes {st.passes} reencodes {st.reencodes} host fixes {st.host_fixes}; measure {tm*1e3:.1f} ms "
      f"norm {norm:.15f} mags {len(st.codebook.mags)} phases {len(st.codebook.thetas)}", flush=True)
