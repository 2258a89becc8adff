"""Host-memory tier on one B200: build_benchmark(N) FP64 larger than HBM.

    python tools/tier_bench.py [N] [fast_capacity_GiB] [chunk_GiB]

Runs run_circuit(build_benchmark(N), tier_config=TierConfig(fast, chunk),
tier_execute=True): the reference's staging plan executed with the slow chunks in
pinned host memory.  Prints one JSON line: setup (pinning) and run seconds, the
reference tier ledger (model) bytes, the physical host-link bytes and GB/s, and the
parity-pattern known answer of the benchmark (test_builders.py:21-33).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200.tier import TierConfig  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 34
fast_gib = float(sys.argv[2]) if len(sys.argv) > 2 else 168
chunk_gib = float(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = TierConfig(int(fast_gib * (1 << 30)), int(chunk_gib * (1 << 30)))
circ = pb.build_benchmark(N)
t0 = time.perf_counter()
res = pb.run_circuit(circ, tier_config=cfg, tier_execute=True)
wall = time.perf_counter() - t0
st = res.device_stats["tier"]
rep = res.report
# known answer: qubits hit twice by H read Qz = 0, Qx = 0.5; once-hit read Qx = 0, Qz = 0.5
twice = {N - 5, N - 6, N - 1, 0, N - 2, 1}
dev = 0.0
for q in range(N):
    qx, qz = (0.5, 0.0) if q in twice else (0.0, 0.5)
    dev = max(dev, abs(rep.qx[q] - qx), abs(rep.qz[q] - qz))
link = st["h2d_bytes"] + st["d2h_bytes"] + st["zero_copy_bytes"]
acct = res.tier_accounts[0]
out = {"what": f"build_benchmark({N}) FP64 on 1 B200, tier_execute", "n_qubits": N,
       "state_GiB": (16 << N) / 2**30, "fast_capacity_GiB": fast_gib, "chunk_GiB": chunk_gib,
       "hbm_fast_GiB": st["hbm_fast_bytes"] / 2**30, "slow_GiB": acct.slow_bytes / 2**30,
       "groups": st["groups"], "gates": len(circ.gates), "wall_s": round(wall, 2),
       "setup_s": st["setup_seconds"], "run_s": st["run_seconds"],
       "model_tier_bytes": res.total_tier_bytes, "model_transfers": res.total_tier_transfers,
       "physical_link_bytes": link, "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"],
       "zero_copy_bytes": st["zero_copy_bytes"], "slot_memsets": st["slot_memsets"],
       "link_GBps": round(link / st["run_seconds"] / 1e9, 2) if st["run_seconds"] else None,
       "sec_per_gate": round(st["run_seconds"] / len(circ.gates), 4),
       "kat_parity_max_dev": dev, "norm_deviation": rep.norm_deviation,
       "high_water_GiB": acct.high_water_bytes / 2**30}
print(json.dumps(out), flush=True)
