"""Multi-GPU parity check, launched by torchrun (one process per GPU).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tests/dist_gpu_check.py

Runs random circuits, the Hadamard benchmark and the QFT adder through
run_circuit_distributed (CUDA IPC + NVLink kernels) and compares the
gathered state (bit for bit), the report and the reference ledgers with the
CPU oracle on rank 0.  Exit code 0 = all checks passed.
"""
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    # SVB200_DEVICES=k: ranks share k GPUs (rank % k) -- 8-rank runs on a 4-GPU box
    ndev = int(os.environ.get("SVB200_DEVICES", "0")) or world
    dev = rank % ndev
    from paper_2511_03359_b200.distributed import run_circuit_distributed
    from oracle import ref_engine
    from oracle.ref_builders import adder, benchmark
    from tests.circuits import random_circuit, sparse_circuit, to_product
    cases = [("random14", random_circuit(np.random.default_rng(11), 14, 80)),
             ("random18", random_circuit(np.random.default_rng(12), 18, 60)),
             ("bench20", benchmark(20)),
             ("adder8", adder(8, [172, 83])[0]),
             # large enough for overlapped swaps (chunk bits >= 12 outside the first pass)
             ("random22", random_circuit(np.random.default_rng(13), 22, 90)),
             ("bench23", benchmark(23)),
             # CPHASE runs on global qubits: ranks hold different diagonal op lists around the
             # overlapped swaps (the chunk choice must not depend on them)
             ("adder11", adder(11, [1234, 813])[0]),
             # small supports (non-monomials on a few qubits): rank slices outside the support
             # skip their passes, the others run support-restricted ones; pair dots of fixed
             # global qubits are skipped
             ("sparse18", sparse_circuit(np.random.default_rng(31), 18, 150, 3)),
             ("sparse22", sparse_circuit(np.random.default_rng(32), 22, 120, 4))]
    ok = True
    for name, circ in cases:
        res = run_circuit_distributed(to_product(circ), dist, device=dev)
        state = res.gathered_state(dist)
        if rank == 0:
            want = ref_engine.run_circuit(circ, ranks=world)
            same = np.array_equal(state, want.gathered_state())
            wx, wy, wz, _ = want.report
            rep = res.report
            diff = max(np.max(np.abs(np.array(rep.qx) - wx)), np.max(np.abs(np.array(rep.qy) - wy)),
                       np.max(np.abs(np.array(rep.qz) - wz)))
            led = [l.snapshot() for l in res.ledgers] == want.ledgers
            print(f"[dist {world} GPUs] {name}: state bit-exact={same} report diff={diff:.2e} "
                  f"ledgers={led} stats={res.device_stats}", flush=True)
            ok = ok and same and diff < 1e-12 and led
        res.backend.close()
    # reference choreography (no remapping): exchange-fused pair updates over NVLink
    for name, circ in [("random14_ref", random_circuit(np.random.default_rng(11), 14, 80)),
                       ("bench16_ref", benchmark(16)),
                       ("sparse14_ref", sparse_circuit(np.random.default_rng(33), 14, 80, 3))]:
        res = run_circuit_distributed(to_product(circ), dist, remap=False, device=dev)
        state = res.gathered_state(dist)
        if rank == 0:
            want = ref_engine.run_circuit(circ, ranks=world)
            same = np.array_equal(state, want.gathered_state())
            led = [l.snapshot() for l in res.ledgers] == want.ledgers
            print(f"[dist {world} GPUs] {name}: state bit-exact={same} ledgers={led} stats={res.device_stats}",
                  flush=True)
            ok = ok and same and led
        res.backend.close()
    from paper_2511_03359_b200 import PrecisionMode
    from tests.circuits import exact_class_circuit
    # FP32 storage across GPUs (remap swaps move complex64 amplitudes)
    for name, circ in [("random16_fp32", random_circuit(np.random.default_rng(21), 16, 70)),
                       ("bench18_fp32", benchmark(18)),
                       ("sparse16_fp32", sparse_circuit(np.random.default_rng(34), 16, 80, 3))]:
        res = run_circuit_distributed(to_product(circ), dist, mode=PrecisionMode.FP32, device=dev)
        state = res.gathered_state(dist)
        if rank == 0:
            want = ref_engine.run_circuit(circ, ranks=world, mode="fp32")
            same = np.array_equal(state, want.gathered_state())
            led = [l.snapshot() for l in res.ledgers] == want.ledgers
            print(f"[dist {world} GPUs] {name}: state bit-exact={same} ledgers={led} stats={res.device_stats}",
                  flush=True)
            ok = ok and same and led
        res.backend.close()
    byte_cases = [("bench14_be", benchmark(14)), ("exact12_be", exact_class_circuit(np.random.default_rng(5), 12, 40)),
                  ("random12_be", random_circuit(np.random.default_rng(6), 12, 30)),
                  ("adder6_be", adder(6, [45, 18])[0]),
                  # rank slices of >= 16 qubits: the tiled BYTE measurement (a rank slice is
                  # dense -- remap swaps move amplitudes between ranks, no support is tracked)
                  ("bench18_be", benchmark(18)), ("adder9_be", adder(9, [300, 77])[0]),
                  # tracked support across ranks (monotone): restricted passes, empty slices,
                  # pending planes cleared after remap swaps
                  ("sparse18_be", sparse_circuit(np.random.default_rng(35), 18, 80, 3)),
                  ("sparse14_be", sparse_circuit(np.random.default_rng(36), 14, 60, 2))]
    for name, circ in byte_cases:
        res = run_circuit_distributed(to_product(circ), dist, mode=PrecisionMode.BYTE, device=dev)
        planes = res.gathered_bytes(dist)
        if rank == 0:
            want = ref_engine.run_circuit(circ, ranks=world, mode="be")
            same = np.array_equal(planes[0], want.mag) and np.array_equal(planes[1], want.phase)
            cbs = res.codebook.dump() == want.codebook.dump()
            wx, wy, wz, _ = want.report
            rep = res.report
            diff = max(np.max(np.abs(np.array(rep.qx) - wx)), np.max(np.abs(np.array(rep.qy) - wy)),
                       np.max(np.abs(np.array(rep.qz) - wz)))
            led = [l.snapshot() for l in res.ledgers] == want.ledgers
            print(f"[dist {world} GPUs] {name}: bytes bit-exact={same} codebook={cbs} report diff={diff:.2e} "
                  f"ledgers={led} stats={res.device_stats}", flush=True)
            ok = ok and same and cbs and diff < 1e-12 and led
        res.backend.close()
    ok = _check_exported_slabs(dist, rank, world, dev) and ok
    flag = [ok]
    dist.broadcast_object_list(flag, src=0)
    dist.destroy_process_group()
    sys.exit(0 if flag[0] else 1)


def _check_exported_slabs(dist, rank, world, dev):
    """A slab exported over CUDA IPC must survive the slab cache's release paths while
    peers still map it (sv_slab.cu): run, free, release the cache on every rank, run the
    same shape again on the cached mappings (bit-exact), then release the mappings
    collectively and check the cache can empty."""
    import ctypes
    from paper_2511_03359_b200 import _native as nat
    from paper_2511_03359_b200.device import release_cached_memory
    from paper_2511_03359_b200.distributed import _PEER_MAPS, release_peer_maps, run_circuit_distributed
    from oracle import ref_engine
    from tests.circuits import random_circuit, to_product
    circ = random_circuit(np.random.default_rng(31), 18, 40)
    res = run_circuit_distributed(to_product(circ), dist, device=dev)
    res.backend.close()
    res.backend.dev.free()
    del res
    release_cached_memory()                 # the OOM-retry / user release path
    cached = ctypes.c_uint64(0)
    nat.load().sv_cached_bytes(ctypes.byref(cached))
    n_local = 18 - (world.bit_length() - 1)
    kept = cached.value >= (1 << n_local) * 16   # the exported 2^n_local-amplitude slab is still held
    dist.barrier()
    res = run_circuit_distributed(to_product(circ), dist, device=dev)
    reused = res.backend.maps_reused
    state = res.gathered_state(dist)
    res.backend.close()
    res.backend.dev.free()
    del res
    release_peer_maps(dist)                 # collective: unmapped everywhere, marks dropped
    release_cached_memory()
    nat.load().sv_cached_bytes(ctypes.byref(cached))
    emptied = cached.value == 0 and not _PEER_MAPS
    flags = [None] * world
    dist.all_gather_object(flags, (kept, reused, emptied))
    if rank != 0:
        return True
    want = ref_engine.run_circuit(circ, ranks=world)
    same = np.array_equal(state, want.gathered_state())
    print(f"[dist {world} GPUs] exported-slab guard: state bit-exact={same} per rank (kept, maps reused, "
          f"emptied after release)={flags}", flush=True)
    return same and all(k and e and (r == world - 1) for k, r, e in flags)


if __name__ == "__main__":
    main()
