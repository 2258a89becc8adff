"""Probe (torchrun): time run_circuit_distributed on the N=32 adder, three runs, with
the device stats of each; rank 0 prints."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed as dist

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat
from paper_2511_03359_b200.device import jit_stats, jit_wait
from paper_2511_03359_b200.distributed import run_circuit_distributed

w = int(sys.argv[1]) if len(sys.argv) > 1 else 16
circ, regs = pb.build_adder(w, [47302 % (1 << w), 18233 % (1 << w)])
for rep in range(3):
    dist.barrier()
    nat.pass_timing(True)
    nat.pass_timing_read()
    t0 = time.perf_counter()
    res = run_circuit_distributed(circ, dist, device=rank)
    t1 = time.perf_counter()
    passes, ms, _ = nat.pass_timing_read()
    nat.pass_timing(False)
    kat = all(abs(res.report.qz[q] - 1.0) < 1e-12 for q in regs["R2"])
    res.backend.close()
    res.backend.dev.free()
    t2 = time.perf_counter()
    if rank == 0:
        print(f"rep {rep}: run {t1 - t0:.3f}s close+free {t2 - t1:.3f}s fused passes {passes} pass_ms {ms:.1f} "
              f"kat {kat} stats {res.device_stats} jit {jit_stats()}", flush=True)
    del res
    jit_wait()
dist.destroy_process_group()
