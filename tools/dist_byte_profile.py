"""Host-side profile of a distributed BYTE run (torchrun, one rank per GPU): where the
per-gate time of run_circuit_distributed(mode=BYTE) goes once the passes are support-
restricted (the codebook barrier: candidate reads, all-gather, merge, table upload).

    torchrun --nproc-per-node 2 tools/dist_byte_profile.py [width=18]
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch.distributed as dist  # noqa: E402

import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200.distributed import run_circuit_distributed  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 18
    circ, _ = pb.build_adder(w, [112838 % (1 << w), 149305 % (1 << w)])
    res = run_circuit_distributed(circ, dist, mode=pb.PrecisionMode.BYTE, device=rank)
    res.backend.close()
    del res
    pr = cProfile.Profile()
    dist.barrier()
    t0 = time.perf_counter()
    pr.enable()
    res = run_circuit_distributed(circ, dist, mode=pb.PrecisionMode.BYTE, device=rank)
    pr.disable()
    wall = time.perf_counter() - t0
    res.backend.close()
    if rank == 0:
        print(f"wall {wall:.3f} s for {len(circ.gates)} gates", flush=True)
        pstats.Stats(pr).sort_stats("tottime").print_stats(30)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
