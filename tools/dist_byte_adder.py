"""Probe (torchrun): the BYTE-encoded QFT adder (BASELINE config 5's second circuit) through
run_circuit_distributed; prints wall time, passes, host fixes and the R2 read-out."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed as dist

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200.distributed import run_circuit_distributed

w = int(sys.argv[1]) if len(sys.argv) > 1 else 14
a, b = 374982 % (1 << w), 149305 % (1 << w)
circ, regs = pb.build_adder(w, [a, b])
dist.barrier()
prof = None
if rank == 0 and os.environ.get("BYTE_ADDER_PROFILE"):
    import cProfile
    prof = cProfile.Profile()
    prof.enable()
t0 = time.perf_counter()
res = run_circuit_distributed(circ, dist, mode=pb.PrecisionMode.BYTE, device=rank)
t = time.perf_counter() - t0
if prof is not None:
    import pstats
    prof.disable()
    pstats.Stats(prof).sort_stats("tottime").print_stats(25)
if rank == 0:
    qz = res.report.qz
    bits = "".join("1" if qz[q] > 0.5 else "0" for q in regs["R2"])
    print(f"BYTE adder w={w} N={circ.n_qubits} on {world} GPUs: {t:.1f} s, {len(circ.gates)} gates, "
          f"stats {res.device_stats}, codebook {len(res.codebook.mags)}/{len(res.codebook.thetas)}, "
          f"R2 bits {bits} (a+b mod 2^w = {format((a + b) % (1 << w), f'0{w}b')}), norm dev "
          f"{res.report.norm_deviation:.3e}", flush=True)
ev = getattr(res.backend.st, "pass_events", None)
if rank == 0 and ev:
    import numpy as np
    scan = [a.elapsed_ms(b) for sc, a, b in ev if sc]
    wr = [a.elapsed_ms(b) for sc, a, b in ev if not sc]
    print(f"passes: scan {len(scan)} sum {sum(scan):.0f} ms median {np.median(scan):.2f}; "
          f"write {len(wr)} sum {sum(wr):.0f} ms median {np.median(wr):.2f}", flush=True)
res.backend.close()
dist.destroy_process_group()
