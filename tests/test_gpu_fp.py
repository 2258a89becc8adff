"""GPU parity tests for the FP64 / FP32 hot path (run on the B200 via gpurun).

Every comparison is against either the reference's own outputs (golden
fixtures written by tests/golden/make_golden.py from /root/reference) or the
CPU oracle (oracle/, pinned to those fixtures) on the same seeded inputs.
The bar is bit-exact amplitudes (np.array_equal) — the kernels reproduce
numpy's operand order — and exact ledgers; reports (floating-point
reductions in a different order) within 1e-12.
"""
import numpy as np
import pytest

import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import gates as g, kernels as K
from oracle import ref_engine, ref_kernels
from tests.circuits import exact_class_circuit, haar_unitary, random_circuit, to_product, unpack

pytestmark = pytest.mark.gpu
MODES = {"fp64": pb.PrecisionMode.FP64, "fp32": pb.PrecisionMode.FP32, "be": pb.PrecisionMode.BYTE}


def _rand_state(rng, n, dtype=np.complex128):
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return (psi / np.linalg.norm(psi)).astype(dtype)


def _report_tuple(rep):
    return pb.ExpectationReport(*rep[:3], norm_deviation=rep[3])


# ---- array-level operators vs the reference's outputs ------------------------------------
def test_kernels_match_reference_goldens(golden):
    k = golden("kernels.npz")
    for i in range(int(k["n_single"])):
        psi = k[f"s{i}_in"].copy()
        K.apply_single(psi, int(k[f"s{i}_q"]), k[f"s{i}_u"])
        assert np.array_equal(psi, k[f"s{i}_out"]), f"single {i}"
    for i in range(int(k["n_two"])):
        psi = k[f"t{i}_in"].copy()
        qa, qb = (int(x) for x in k[f"t{i}_q"])
        K.apply_two(psi, qa, qb, k[f"t{i}_u"])
        assert np.array_equal(psi, k[f"t{i}_out"]), f"two {i}"
    for i in range(int(k["n_diag"])):
        psi = k[f"d{i}_in"].copy()
        K.apply_diagonal(psi, tuple(int(b) for b in k[f"d{i}_bits"]), complex(k[f"d{i}_f"]))
        assert np.array_equal(psi, k[f"d{i}_out"]), f"diag {i}"
    for i in range(int(k["n_fp32"])):
        psi = k[f"f{i}_in"].copy()
        K.apply_single(psi, int(k[f"f{i}_q"]), k[f"f{i}_u"])
        assert np.array_equal(psi, k[f"f{i}_out"]), f"fp32 {i}"


def test_kernels_match_oracle_at_n20(rng):
    n = 20
    for q in (0, 1, 2, 5, 13, 19):
        psi = _rand_state(rng, n)
        u = haar_unitary(rng, 2)
        want = psi.copy()
        ref_kernels.gate1(want, q, u)
        K.apply_single(psi, q, u)
        assert np.array_equal(psi, want), q
    for qa, qb in ((0, 1), (1, 0), (0, 19), (5, 17), (18, 19), (19, 3)):
        psi = _rand_state(rng, n)
        u = haar_unitary(rng, 4)
        want = psi.copy()
        ref_kernels.gate2(want, qa, qb, u)
        K.apply_two(psi, qa, qb, u)
        assert np.array_equal(psi, want), (qa, qb)
    for bits, k in (((), 3), ((0,), 1), ((0, 7), -2), ((12, 19), 4), ((1, 2, 3), 5)):
        psi = _rand_state(rng, n)
        f = g.diagonal_factor(g.phase(0, k))
        want = psi.copy()
        ref_kernels.diag(want, bits, f)
        K.apply_diagonal(psi, bits, f)
        assert np.array_equal(psi, want), bits
    psi = _rand_state(rng, n, np.complex64)
    u = haar_unitary(rng, 2)
    want = psi.copy()
    ref_kernels.gate1(want, 4, u)
    K.apply_single(psi, 4, u)
    assert np.array_equal(psi, want)


def test_pair_and_quad_arrays(rng):
    a0, a1 = _rand_state(rng, 10), _rand_state(rng, 10)
    u = haar_unitary(rng, 2)
    got = K.apply_pair_arrays(a0, a1, u)
    want = ref_kernels.pair_arrays(a0, a1, u)
    assert all(np.array_equal(x, y) for x, y in zip(got, want))
    parts = [_rand_state(rng, 9)[:300] for _ in range(4)]
    u4 = haar_unitary(rng, 4)
    got = K.apply_quad_arrays(parts, u4)
    want = ref_kernels.quad_arrays(parts, u4)
    assert all(np.array_equal(x, y) for x, y in zip(got, want))
    psi = _rand_state(rng, 12)
    assert abs(K.norm_squared(psi) - ref_kernels.norm2(psi)) < 1e-13


def test_kernel_error_types():
    psi = np.zeros(8, dtype=np.complex128)
    with pytest.raises(IndexError):
        K.apply_single(psi, 3, g.H_MATRIX)
    with pytest.raises(ValueError):
        K.apply_two(psi, 1, 1, g.CNOT_MATRIX)
    with pytest.raises(IndexError):
        K.apply_two(psi, 0, 3, g.CNOT_MATRIX)
    with pytest.raises(IndexError):
        K.pair_indices(4, 4)
    # non-power-of-two arrays follow numpy's reshape semantics
    psi = np.arange(12, dtype=np.complex128)
    want = psi.copy()
    ref_kernels.gate1(want, 1, g.H_MATRIX)
    K.apply_single(psi, 1, g.H_MATRIX)
    assert np.array_equal(psi, want)


# ---- run_circuit vs the reference's runs ------------------------------------------------
def test_engine_runs_match_reference_goldens(golden):
    d = golden("runs.npz")
    fields = [str(f) for f in d["ledger_fields"]]
    circuits = {}
    checked = 0
    for key in (str(k) for k in d["run_keys"]):
        name, mode, P = key.split("__")
        if mode == "be":
            continue
        if name not in circuits:
            circuits[name] = to_product(unpack(d, f"{name}__circuit_"))
        for fuse in (True, False):
            res = pb.run_circuit(circuits[name], ranks=int(P), mode=MODES[mode], fuse=fuse)
            assert np.array_equal(res.gathered_state(), d[key + "__state"]), (key, fuse)
            if mode == "fp32":
                raw = np.concatenate([s.psi for s in res.states])
                assert np.array_equal(raw, d[key + "__psi32"]), key
            got = np.array([[led.snapshot()[f] for f in fields] for led in res.ledgers])
            assert np.array_equal(got, d[key + "__ledgers"]), key
            if key + "__report" in d:
                rep = res.report
                want = d[key + "__report"]
                diff = np.max(np.abs(np.array([rep.qx, rep.qy, rep.qz]) - want))
                assert diff < 1e-12, (key, diff)
                assert abs(rep.norm_deviation - float(d[key + "__normdev"])) < 1e-12
            checked += 1
    assert checked > 50


@pytest.mark.parametrize("n,depth,ranks", [(16, 80, 1), (18, 60, 4), (20, 40, 8)])
def test_engine_matches_oracle_larger(rng, n, depth, ranks):
    circ = random_circuit(rng, n, depth)
    want = ref_engine.run_circuit(circ, ranks=ranks)
    got = pb.run_circuit(to_product(circ), ranks=ranks)
    assert np.array_equal(got.gathered_state(), want.gathered_state())
    assert got.report.max_difference(_report_tuple(want.report)) < 1e-12
    for a, b in zip(got.ledgers, want.ledgers):
        assert a.snapshot() == b


def test_fp32_engine_matches_oracle(rng):
    circ = random_circuit(rng, 16, 50)
    want = ref_engine.run_circuit(circ, ranks=2, mode="fp32")
    got = pb.run_circuit(to_product(circ), ranks=2, mode=pb.PrecisionMode.FP32)
    assert np.array_equal(np.concatenate([s.psi for s in got.states]), want.psi)


def test_fusion_is_bit_identical_to_per_gate(rng):
    circ = to_product(random_circuit(rng, 17, 120))
    a = pb.run_circuit(circ, fuse=True)
    b = pb.run_circuit(circ, fuse=False)
    c = pb.run_circuit(circ, fuse=True, tile_bits=10)
    assert np.array_equal(a.gathered_state(), b.gathered_state())
    assert np.array_equal(a.gathered_state(), c.gathered_state())
    assert a.report == b.report == c.report


# ---- known answers at sizes the oracle cannot reach quickly ------------------------------
def test_benchmark_parity_kat_n26():
    n = 26
    res = pb.run_circuit(pb.build_benchmark(n), ranks=4)
    twice = {n - 5, n - 6, n - 1, 0, n - 2, 1}
    rep = res.report
    for q in range(n):
        if q in twice:
            assert abs(rep.qz[q]) < 1e-12 and abs(rep.qx[q] - 0.5) < 1e-12
        else:
            assert abs(rep.qx[q]) < 1e-12 and abs(rep.qz[q] - 0.5) < 1e-12
    assert rep.norm_deviation < 1e-12
    # ledger volume law (test_engine.py:116-126): high gates + measured high qubits
    local = 1 << 24
    high = sum(1 for gate in res.circuit.gates if gate.kind == "H" and gate.qubits[0] >= 24)
    for led in res.ledgers:
        assert led.inter_rank_bytes_sent == (high + 2) * (local // 2) * 16


def test_adder_all_ones_kat():
    for width in (6, 9):
        a = (1 << width) - 1 - (0b1010101 & ((1 << width) - 1))
        b = (1 << width) - 1 - a
        circ, regs = pb.build_adder(width, [a, b])
        rep = pb.run_circuit(circ).report
        for q in regs["R2"]:
            assert abs(rep.qz[q] - 1.0) < 1e-12
        bits = [round(v) for v in rep.qz]
        assert pb.decode_register(bits, regs["R1"]) == a


@pytest.mark.parametrize("case", ["adder9", "adder11", "random18"])
def test_combined_diagonal_runs_within_tolerance(rng, case):
    """run_circuit(exact_diagonals=False): runs of diagonal gates multiply each amplitude by
    their combined factor (sv_set_diag_combine) -- amplitudes within 1e-12 relative of the
    reference oracle (the north star's FP64 tolerance), reports within 1e-12, and the
    passes really are the combined kernels (fewer FP64 instructions than the exact ones)."""
    from oracle import ref_engine
    from oracle.ref_builders import adder
    if case.startswith("adder"):
        w = int(case[5:])
        circ = adder(w, [(1 << w) - 1 - (0x2AAA & ((1 << w) - 1)), 0x1555 & ((1 << w) - 1)])[0]
    else:
        circ = random_circuit(rng, 18, 60)
    prod = to_product(circ)
    got = pb.run_circuit(prod, exact_diagonals=False)
    want = ref_engine.run_circuit(circ)
    ref = want.gathered_state()
    dev = np.max(np.abs(got.gathered_state() - ref)) / np.max(np.abs(ref))
    assert dev < 1e-12, dev
    qx, qy, qz, _ = want.report
    assert got.report.max_difference(pb.ExpectationReport(qx, qy, qz)) < 1e-12
    assert got.device_stats["diag_combine"] is True
    exact = pb.run_circuit(prod)
    assert exact.device_stats["diag_combine"] is False
    assert np.array_equal(exact.gathered_state(), ref)


def _tiles_skipped() -> int:
    """Process-wide count of tiles the support-restricted passes left out (sv_support_info)."""
    from paper_2511_03359_b200.device import DeviceState
    dev = DeviceState(4, pb.PrecisionMode.FP64)
    try:
        return dev.support_info()["tiles_skipped_total"]
    finally:
        dev.free()


def test_support_tracking_skips_zero_tiles_bit_exact():
    """run_circuit tracks the support of its |0..0> state: the adder's state lives in the
    superposed register (the other register stays a basis state), so most tiles of most
    passes are left out -- and the state is still bit-identical to the oracle's and to a
    run with tracking off (SVB200_SUPPORT=0 semantics, via the DeviceState switch)."""
    from oracle import ref_engine
    from oracle.ref_builders import adder
    w = 9
    circ = adder(w, [0x155 & ((1 << w) - 1), 0x0AB & ((1 << w) - 1)])[0]
    skipped0 = _tiles_skipped()
    res = pb.run_circuit(to_product(circ))
    want = ref_engine.run_circuit(circ)
    assert np.array_equal(res.gathered_state(), want.gathered_state())
    sup = res.device_stats["support"]
    assert sup["tracking"] and sup["free_qubits"] < circ.n_qubits
    assert sup["tiles_skipped_total"] > skipped0   # (the generic kernel restricts too: no JIT wait)
    qx, qy, qz, _ = want.report
    assert res.report.max_difference(pb.ExpectationReport(qx, qy, qz)) < 1e-12
    # monomials on fixed qubits move the support, they do not free it
    from paper_2511_03359_b200.device import DeviceState
    dev = DeviceState(14, pb.PrecisionMode.FP64)
    dev.set_support_tracking(True)
    dev.zero(0)
    dev.apply_1q(3, pb.gates.unitary_matrix(pb.gates.x(3)))
    dev.apply_2q(3, 7, pb.gates.unitary_matrix(pb.gates.cnot(3, 7)))
    assert dev.support_info()["free_qubits"] == 0
    dev.apply_1q(5, pb.gates.H_MATRIX)
    assert dev.support_info()["free_qubits"] == 1
    out = dev.export()
    assert out[(1 << 3) | (1 << 7)] != 0 and out[(1 << 3) | (1 << 7) | (1 << 5)] != 0
    assert np.count_nonzero(out) == 2
    dev.free()


@pytest.mark.parametrize("n,depth,spread,ranks,mode", [
    (16, 120, 3, 1, "fp64"), (18, 200, 4, 4, "fp64"), (20, 160, 5, 1, "fp64"),
    (18, 150, 4, 1, "fp32"), (21, 100, 2, 8, "fp64")])
def test_support_tracking_sparse_circuits_bit_exact(n, depth, spread, ranks, mode):
    """Non-monomial gates on a few qubits, monomials (X, Y, CNOT) and diagonals anywhere: the
    tracked support moves (monomials on fixed qubits) and grows (CNOT from a free control,
    U4 across free/fixed qubits) -- state bit-identical to the oracle and to the dense run."""
    from oracle import ref_engine
    from tests.circuits import sparse_circuit
    circ = sparse_circuit(np.random.default_rng(1000 + n + depth), n, depth, spread)
    pm = {"fp64": pb.PrecisionMode.FP64, "fp32": pb.PrecisionMode.FP32}[mode]
    lib = __import__("paper_2511_03359_b200._native", fromlist=["load"]).load()
    prev = lib.sv_jit_mode(1)     # FP32 restricts only through specialised passes: compile and wait
    try:
        skipped0 = _tiles_skipped()
        res = pb.run_circuit(to_product(circ), ranks=ranks, mode=pm)
    finally:
        lib.sv_jit_mode(prev)
    want = ref_engine.run_circuit(circ, ranks=ranks, mode=mode)
    assert np.array_equal(res.gathered_state(), want.gathered_state())
    qx, qy, qz, _ = want.report
    assert res.report.max_difference(pb.ExpectationReport(qx, qy, qz)) < 1e-12
    sup = res.device_stats["support"]
    assert sup["tracking"] and sup["tiles_skipped_total"] > skipped0, sup
    dense = pb.run_circuit(to_product(circ), ranks=ranks, mode=pm, track_support=False)
    assert np.array_equal(res.gathered_state(), dense.gathered_state())
    assert res.report == dense.report or res.report.max_difference(dense.report) < 1e-12


# ---- engine contracts ---------------------------------------------------------------------
def test_scheduling_invariance(rng):
    circ = to_product(random_circuit(rng, 8, 18))
    a = pb.run_circuit(circ, ranks=8, rank_order_seed=7)
    b = pb.run_circuit(circ, ranks=8, rank_order_seed=1234)
    assert np.array_equal(a.gathered_state(), b.gathered_state())
    assert [l.snapshot() for l in a.ledgers] == [l.snapshot() for l in b.ledgers]
    assert a.report == b.report


def test_transport_failure_names_gate():
    class Failing(pb.Transport):
        def send(self, src, dst, payload, nbytes):
            raise pb.TransportError(f"link down between {src} and {dst}")

    circ = pb.Circuit(4, (g.x(0), g.h(3)))
    with pytest.raises(RuntimeError, match=r"gate 1 \(H\): link down"):
        pb.run_circuit(circ, ranks=4, transport_factory=Failing)


def test_partner_is_rank_xor_mask():
    log = []

    class Spy(pb.Transport):
        def send(self, src, dst, payload, nbytes):
            log.append((src, dst, nbytes))
            super().send(src, dst, payload, nbytes)

    pb.run_circuit(pb.Circuit(5, (g.h(4),)), ranks=8, transport_factory=Spy)
    assert sorted(log) == sorted((r, r ^ 4, 2 * 16) for r in range(8))


def test_measure_all_on_standalone_states():
    st = pb.LocalState.zero_state(3, pb.PrecisionMode.FP64, True)
    st.psi *= 2.0
    leds = [pb.TrafficLedger()]
    rep = pb.measure_all([st], pb.PartitionLayout(3, 3), pb.Transport(1, leds), leds)
    assert abs(rep.norm_deviation - 3.0) < 1e-12
    res = pb.run_circuit(pb.Circuit(6, (g.measure_all(),)), ranks=8)
    for led in res.ledgers:
        assert led.inter_rank_messages == 3 and led.inter_rank_bytes_sent == 3 * 4 * 16


def test_local_state_api():
    st = pb.LocalState.zero_state(4, pb.PrecisionMode.FP32, True)
    assert st.psi.dtype == np.complex64 and st.psi[0] == 1 and st.storage_nbytes == 16 * 8
    assert abs(st.norm_squared() - 1.0) < 1e-12
    w = st.working()
    assert w.dtype == np.complex128
    st.store(np.full(16, 0.25, dtype=np.complex128))
    assert np.allclose(st.psi, 0.25)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_gpu_torchrun_parity(world):
    """Distributed path (CUDA IPC peer kernels: remap swaps, 3-qubit group swaps, swaps
    overlapped with passes, the reference's exchange-fused pair updates, FP32 and BYTE
    planes) under torchrun vs the oracle, bit for bit.  On a box with fewer GPUs than
    ranks the ranks share the visible GPUs (SVB200_DEVICES: rank % k) -- CUDA IPC between
    processes on one device runs the same kernels over the same mappings."""
    import ctypes
    import os
    import subprocess
    import sys
    from paper_2511_03359_b200 import _native
    n = ctypes.c_int(0)
    _native.load().sv_device_count(ctypes.byref(n))
    assert n.value >= 1
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SVB200_DEVICES=str(min(n.value, world)), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", str(world), "--master-addr",
           "127.0.0.1", "--master-port", str(29530 + world), os.path.join(root, "tests", "dist_gpu_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("bit-exact=True") >= 15 and "bit-exact=False" not in r.stdout
