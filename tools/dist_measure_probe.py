"""Probe (torchrun): the distributed measurement's two halves at 2^n amplitudes per GPU --
local measurement passes alone, global-qubit pair dots alone (NVLink), both concurrent
(what _measure does)."""
import os
import sys
import threading
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed as dist

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import distributed as D

n_local = int(sys.argv[1]) if len(sys.argv) > 1 else 33
be = D.CudaBackend(dist, n_local, pb.PrecisionMode.FP64, rank)
for q in range(3):
    be.apply_local([D.gate_op(D.nat.SV_OP_1Q, qa=q, data=D.nat.mat_buffer(pb.gates.H_MATRIX))])
gpos = list(range(n_local, n_local + world.bit_length() - 1))


def timed(fn):
    be._sync_all()
    dist.barrier()
    t0 = time.perf_counter()
    fn()
    be.dev.synchronize()
    dist.barrier()
    return time.perf_counter() - t0


def both():
    box = {}
    th = threading.Thread(target=lambda: box.update(v=be.pair_dots(gpos)))
    prev = D.nat.load().sv_measure_reserve(be.MEASURE_RESERVE)
    th.start()
    be.measure_local()
    th.join()
    D.nat.load().sv_measure_reserve(prev)


for rep in range(3):
    tm = timed(be.measure_local)
    tp = timed(lambda: be.pair_dots(gpos))
    tb = timed(both)
    if rank == 0:
        half = (1 << n_local) // 2 * 16
        print(f"blocks {be.PAIR_DOT_BLOCKS} reserve {be.MEASURE_RESERVE} rep {rep}: measure_local {tm * 1e3:.1f} ms  pair_dots {tp * 1e3:.1f} ms "
              f"({len(gpos) * half / tp / 1e9:.0f} GB/s over the link)  concurrent {tb * 1e3:.1f} ms", flush=True)
be.close()
dist.destroy_process_group()
