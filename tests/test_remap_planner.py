"""CPU tests of the global<->local remapping planner (host logic only).

The planner's schedule (swaps + gates on physical qubits) is replayed on a
numpy state with the oracle's kernels; swaps are index permutations.  The
un-permuted final state must equal the oracle's straight execution bit for
bit, and the traffic must not exceed the reference's accounting.
"""
import numpy as np
import pytest

from oracle import ref_engine, ref_gates, ref_kernels, ref_optimize
from oracle.ref_builders import adder, benchmark
from paper_2511_03359_b200.remap import (Measure, PhysGate, RemapPlanner, Swap, SwapGroup, group_schedule,
                                         swap_traffic_elements)
from tests.circuits import random_circuit


def _apply(psi, gate, phys):
    if ref_gates.is_diag(gate):
        ref_kernels.diag(psi, tuple(phys), ref_gates.factor_of(gate))
    elif len(phys) == 1:
        ref_kernels.gate1(psi, phys[0], ref_gates.matrix_of(gate))
    else:
        ref_kernels.gate2(psi, phys[0], phys[1], ref_gates.matrix_of(gate))


def _swap_bits(psi, a, b):
    n = psi.size.bit_length() - 1
    idx = np.arange(psi.size)
    ba, bb = (idx >> a) & 1, (idx >> b) & 1
    src = idx ^ ((ba ^ bb) << a) ^ ((ba ^ bb) << b)
    return psi[src]


def _unpermute(psi, pos):
    """physical state -> logical state, given logical->physical map `pos`."""
    n = len(pos)
    idx = np.arange(psi.size)
    phys = np.zeros_like(idx)
    for q, p in enumerate(pos):
        phys |= ((idx >> q) & 1) << p
    return psi[phys]


def _replay(circ, n_local, remap=True, batch=True):
    planner = RemapPlanner(circ.n_qubits, n_local, remap=remap, batch=batch)
    steps = planner.plan(circ.gates)
    psi = np.zeros(1 << circ.n_qubits, dtype=np.complex128)
    psi[0] = 1.0
    for s in steps:
        if isinstance(s, Swap):
            psi = _swap_bits(psi, s.global_pos, s.local_pos)
        elif isinstance(s, SwapGroup):
            for gp, lp in s.pairs:
                psi = _swap_bits(psi, gp, lp)
        elif isinstance(s, PhysGate):
            assert remap is False or all(p < n_local for p in s.qubits) or ref_gates.is_diag(s.gate)
            _apply(psi, s.gate, s.qubits)
    return _unpermute(psi, planner.pos), steps, planner


@pytest.mark.parametrize("batch", [True, False])
@pytest.mark.parametrize("n,local,depth", [(8, 6, 40), (9, 6, 60), (10, 7, 80), (7, 4, 50)])
def test_remapped_schedule_is_bit_exact(rng, n, local, depth, batch):
    circ = random_circuit(rng, n, depth)
    got, steps, _ = _replay(circ, local, batch=batch)
    want = ref_engine.run_circuit(circ, ranks=1).gathered_state()
    assert np.array_equal(got, want)


def test_measure_steps_carry_the_permutation(rng):
    circ = random_circuit(rng, 8, 30)
    planner = RemapPlanner(8, 5)
    steps = planner.plan(circ.gates)
    m = [s for s in steps if isinstance(s, Measure)]
    assert len(m) == 1 and sorted(m[0].perm) == list(range(8))


@pytest.mark.parametrize("name", ["bench", "adder"])
def test_remap_never_moves_more_than_the_reference(name):
    if name == "bench":
        circ, local = benchmark(14), 11
    else:
        circ, local = adder(6, [45, 18])[0], 9
        circ = ref_optimize.relabel(circ, tuple(reversed(range(circ.n_qubits))))   # sources on the rank bits
    steps = RemapPlanner(circ.n_qubits, local).plan(circ.gates)
    moved = swap_traffic_elements(steps, local) * 16 * (1 << (circ.n_qubits - local))
    # the reference ledger counts L/2 per rank per global gate; physically the
    # partner's result half travels back too (engine.py:365-377): 2x the ledger
    reference_physical = 2 * ref_optimize.predicted_bytes(circ, local)
    assert moved <= reference_physical
    got, _, _ = _replay(circ, local)
    assert np.array_equal(got, ref_engine.run_circuit(circ, ranks=1).gathered_state())


def test_benchmark_n36_swap_count():
    # 3 global qubits at N=36 on 8 GPUs: the reference exchanges 5 gates x L/2
    # each way (10 half-slices physically).  Single swaps (Belady with forced
    # insertion) need 6 half-slices; batching fetches the three rank bits
    # together twice: 2 x 7/8 L = 3.5 half-slices.
    circ = benchmark(36)
    single = RemapPlanner(36, 33, batch=False).plan(circ.gates)
    swaps = [s for s in single if isinstance(s, Swap)]
    assert len(swaps) <= 6
    assert all(s.local_pos >= 5 for s in swaps)
    steps = RemapPlanner(36, 33).plan(circ.gates)
    groups = [s for s in steps if isinstance(s, SwapGroup)]
    assert groups and all(lp >= 5 for s in groups for _, lp in s.pairs)
    L = 1 << 33
    assert swap_traffic_elements(steps, 33) <= 2 * (L - L // 8)
    assert swap_traffic_elements(steps, 33) < swap_traffic_elements(single, 33)


@pytest.mark.parametrize("P,k", [(2, 1), (4, 2), (8, 3), (8, 2), (16, 3)])
def test_group_schedule_equals_sequential_swaps(rng, P, k):
    """Emulates svk_swap_group launches on P numpy slices exactly as
    CudaBackend.swap_group issues them; the result must equal k pairwise swaps."""
    n_local = 6
    L = 1 << n_local
    n = n_local + (P.bit_length() - 1)
    full = rng.standard_normal(L * P) + 1j * rng.standard_normal(L * P)
    gps = list(rng.choice(np.arange(n_local, n), size=k, replace=False))
    lps = list(rng.choice(np.arange(n_local), size=k, replace=False))
    pairs = tuple(zip(map(int, gps), map(int, lps)))
    want = full.copy()
    for gp, lp in pairs:
        want = _swap_bits(want, gp, lp)
    slices = [full[r * L:(r + 1) * L].copy() for r in range(P)]
    touched = [np.zeros(L, dtype=int) for _ in range(P)]
    for r in range(P):
        for member, vmask, own_pat, peer_pat, t0, cnt in group_schedule(r, pairs, n_local, L):
            free = [b for b in range(n_local) if not (vmask >> b) & 1]
            for t in range(t0, t0 + cnt):
                base = sum(((t >> j) & 1) << b for j, b in enumerate(free))
                x, y = base | own_pat, base | peer_pat
                slices[r][x], slices[member][y] = slices[member][y], slices[r][x]
                touched[r][x] += 1
                touched[member][y] += 1
    assert np.array_equal(np.concatenate(slices), want)
    # every moved amplitude is touched exactly once (no launch overlaps another)
    assert max(int(t.max()) for t in touched) == 1
