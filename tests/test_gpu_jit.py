"""GPU parity of the run-time specialised fused passes (sv_jit.cu).

The library compiles one kernel per pass structure in the background and runs
the generic k_fused3 until it is ready, so ordinary tests exercise whichever is
ready first.  Here the JIT is put in compile-and-wait mode (sv_jit_mode(1)) so
every FP64 fused pass runs the specialised kernel, then the generic path
(mode 0) for the same circuits; both must equal the oracle bit for bit.
Circuits cover the generated code paths: generic / real / monomial 1Q ops,
generic / monomial 2Q ops, diagonal ops with register, thread and out-of-tile
mask bits, and a pass with >= 96 diagonal ops (the diag_run descriptor loop).
"""
import numpy as np
import pytest

import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat
from paper_2511_03359_b200.device import jit_stats
from oracle import ref_engine
from oracle.ref_builders import OCircuit, adder
from oracle.ref_gates import OGate
from tests.circuits import exact_class_circuit, random_circuit, to_product

pytestmark = pytest.mark.gpu


def _diag_heavy(rng, n, count):
    """H on every qubit, then `count` CPHASE / PHASE / Z gates with a few H between."""
    gates = [OGate("H", (q,)) for q in range(n)]
    for i in range(count):
        a, b = (int(x) for x in rng.choice(n, size=2, replace=False))
        kind = ("CPHASE", "PHASE", "Z")[i % 3]
        if kind == "CPHASE":
            gates.append(OGate("CPHASE", (a, b), int(rng.integers(1, 6))))
        elif kind == "PHASE":
            gates.append(OGate("PHASE", (a,), int(rng.integers(1, 5))))
        else:
            gates.append(OGate("Z", (a,)))
        if i % 40 == 39:
            gates.append(OGate("H", (int(rng.integers(n)),)))
    gates.append(OGate("M"))
    return OCircuit(n, tuple(gates))


def _diag_run_pass(rng, n):
    """32 one-qubit gates on tile qubits, then 100 diagonal ops: the planner keeps them in
    one pass (it closes a pass at 80 ops only when >= 75 % are diagonal), whose >= 96
    diagonal ops the specialised kernel runs as the descriptor loop (diag_run)."""
    gates = [OGate(("H", "X", "Y")[i % 3], (i % 7,)) for i in range(32)]
    for i in range(100):
        a, b = (int(x) for x in rng.choice(n, size=2, replace=False))
        kind = ("CPHASE", "PHASE", "Z")[i % 3]
        if kind == "CPHASE":
            gates.append(OGate("CPHASE", (a, b), int(rng.integers(1, 6))))
        elif kind == "PHASE":
            gates.append(OGate("PHASE", (a,), int(rng.integers(1, 5))))
        else:
            gates.append(OGate("Z", (a,)))
    gates.append(OGate("M"))
    return OCircuit(n, tuple(gates))


def _cases(rng):
    return [("random18", random_circuit(np.random.default_rng(31), 18, 120)),
            ("exact16", exact_class_circuit(np.random.default_rng(32), 16, 120)),
            ("diag_heavy16", _diag_heavy(np.random.default_rng(33), 16, 260)),
            ("diag_run16", _diag_run_pass(np.random.default_rng(35), 16)),
            ("adder9", adder(9, [301, 88])[0])]


@pytest.fixture
def jit_mode():
    lib = nat.load()
    prev = lib.sv_jit_mode(-1)

    def set_mode(m):
        lib.sv_jit_mode(m)
    yield set_mode
    lib.sv_jit_mode(prev)


@pytest.fixture
def tile_cfg():
    lib = nat.load()

    def set_cfg(c):
        nat.check(lib.sv_fused_variant(c))
    yield set_cfg
    nat.check(lib.sv_fused_variant(9))


@pytest.mark.parametrize("cfg", [6, 8])
@pytest.mark.parametrize("mode", [1, 0])
def test_specialised_and_generic_passes_bit_exact(rng, jit_mode, tile_cfg, mode, cfg):
    """cfg 6: 2^11 double-buffered tiles; cfg 8: 2^12 single-buffered tiles (next tile
    requested once the last segment holds the tile in registers)."""
    jit_mode(mode)
    tile_cfg(cfg)
    before = jit_stats()
    for name, circ in _cases(rng):
        want = ref_engine.run_circuit(circ, ranks=1)
        got = pb.run_circuit(to_product(circ))
        assert np.array_equal(got.gathered_state(), want.gathered_state()), (name, mode)
        wx, wy, wz, _ = want.report
        diff = max(np.max(np.abs(np.array(got.report.qx) - wx)), np.max(np.abs(np.array(got.report.qz) - wz)))
        assert diff < 1e-12, name
    after = jit_stats()
    if mode == 1:
        assert after["jit_launches"] > before["jit_launches"] and after["failed"] == before["failed"]
    else:
        assert after["jit_launches"] == before["jit_launches"]


@pytest.mark.parametrize("cfg", [6, 8])
@pytest.mark.parametrize("mode", [1, 0])
def test_specialised_fp32_passes_bit_exact(rng, jit_mode, tile_cfg, mode, cfg):
    """FP32 storage: widened FP64 arithmetic, one rounding to float after every gate
    (kernels.py:36-40) -- the specialised kernel rounds after each op."""
    jit_mode(mode)
    tile_cfg(cfg)
    before = jit_stats()
    for name, circ in _cases(rng):
        want = ref_engine.run_circuit(circ, ranks=1, mode="fp32")
        got = pb.run_circuit(to_product(circ), mode=pb.PrecisionMode.FP32)
        assert np.array_equal(got.gathered_state(), want.gathered_state()), (name, mode)
    if mode == 1:
        assert jit_stats()["jit_launches"] > before["jit_launches"]


def test_specialised_multi_rank_emulation(rng, jit_mode):
    """ranks > 1 on one GPU: the same passes over the whole buffer, ledgers exact."""
    jit_mode(1)
    circ = random_circuit(np.random.default_rng(34), 16, 80)
    for ranks in (2, 4):
        want = ref_engine.run_circuit(circ, ranks=ranks)
        got = pb.run_circuit(to_product(circ), ranks=ranks)
        assert np.array_equal(got.gathered_state(), want.gathered_state()), ranks
        assert [led.snapshot() for led in got.ledgers] == want.ledgers


@pytest.mark.parametrize("mode", [1, 0])
def test_chunked_passes_equal_whole_passes(rng, jit_mode, mode):
    """sv_apply_fused_chunk over every chunk pattern == one sv_apply_fused (the chunked
    form runs a pass under a remap swap, tile by tile as the swap chunks land)."""
    from paper_2511_03359_b200.device import DeviceState, ops_array
    from paper_2511_03359_b200.engine import gate_to_op
    jit_mode(mode)
    n = 16
    circ = random_circuit(np.random.default_rng(41), 11, 60, measured=False)   # qubits 0..10 only
    ops = [gate_to_op(gt) for gt in to_product(circ).gates]
    psi0 = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex128)
    lib = nat.load()
    whole = DeviceState(n, pb.PrecisionMode.FP64)
    whole.import_(psi0)
    whole.apply_fused(ops)
    want = whole.export()
    chunked = DeviceState(n, pb.PrecisionMode.FP64)
    chunked.import_(psi0)
    cmask = (1 << 15) | (1 << 13)
    arr = ops_array(ops)
    for pat in (0, 1 << 13, 1 << 15, cmask):
        nat.check(lib.sv_apply_fused_chunk(chunked.handle, arr, len(ops), 12, cmask, pat))
    assert np.array_equal(chunked.export(), want)
    with pytest.raises(ValueError):      # chunk bit inside a pass tile
        nat.check(lib.sv_apply_fused_chunk(chunked.handle, arr, len(ops), 12, 1 << 3, 0))
    whole.free()
    chunked.free()
