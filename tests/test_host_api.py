"""CPU tests of the product's host logic against the reference goldens.

No GPU is touched here: planner / layout / ledger / builders / gate constants /
parser / transport, plus the C ABI library loading and exporting every
symbol include/svb200.h declares.
"""
import os
import re

import numpy as np
import pytest

import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native, gates as g
from paper_2511_03359_b200.layout import gibibytes_exchanged
from tests.circuits import random_circuit, to_product, unpack

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = {"fp64": pb.PrecisionMode.FP64, "fp32": pb.PrecisionMode.FP32, "be": pb.PrecisionMode.BYTE}


def test_library_exports_every_declared_symbol():
    lib = _native.load(require_device=False)
    header = open(os.path.join(ROOT, "include", "svb200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(sv\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.exported_symbols())
    assert lib.sv_abi_version() == 3


def test_gate_constants_bit_exact(golden):
    k = golden("kernels.npz")
    assert np.array_equal(g.H_MATRIX, k["H"])
    for e in (1, 2, 3, 4, -1, -2, -3, -4, 7, 16, 25):
        f = np.complex128(g.diagonal_factor(g.phase(0, e)))
        assert f.tobytes() == k[f"factor_{e}"].tobytes(), e
    assert g.diagonal_factor(g.z(0)) == -1.0 + 0.0j
    assert g.phase_angle(2) == np.pi / 2 and g.phase_angle(-2) == -np.pi / 2
    with pytest.raises(ValueError):
        g.phase_angle(0)


def test_gate_validation_messages():
    with pytest.raises(ValueError, match="out of range"):
        g.validate_gate(g.h(5), 4)
    with pytest.raises(ValueError, match="distinct"):
        g.validate_gate(g.cphase(2, 2, 1), 4)
    with pytest.raises(ValueError, match="not unitary"):
        g.validate_gate(g.u2(0, np.diag([1.0, 2.0])), 2)
    with pytest.raises(ValueError):
        g.validate_gate(g.Gate("M", (0,)), 2)
    for gate in (g.h(0), g.x(0), g.y(0), g.cnot(0, 1)):
        assert g.unitarity_residual(g.unitary_matrix(gate)) < 1e-15


def test_plans_match_reference(golden):
    for e in golden("planner.json")["plans"]:
        gate = g.Gate(e["kind"], tuple(e["qubits"]))
        p = pb.plan_exchange(pb.PartitionLayout(e["n"], e["local"]), gate, MODES[e["mode"]])
        assert (p.kind, list(p.masks), p.element_count, p.bytes_per_element) == \
            (e["plan_kind"], e["masks"], e["count"], e["bpe"]), e
    for e in golden("planner.json")["memory"]:
        assert pb.memory_bytes(e["n"], MODES[e["mode"]]) == e["bytes"]


def _workload(name):
    if name == "adder16":
        return pb.build_adder(16, [47302, 18233])[0]
    if name == "adder19":
        return pb.build_adder(19, [374982, 149305])[0]
    if name == "adder25":
        return pb.build_adder(25, [21346502, 12207929])[0]
    if name.startswith("bench"):
        return pb.build_benchmark(int(name[5:]))
    return None


def test_optimize_labels_matches_reference(golden):
    for e in golden("planner.json")["optimize"]:
        circ = _workload(e["name"])
        if circ is None:
            d = {k: np.array(v) for k, v in e["circuit"].items()}
            d["mats"] = np.zeros((len(d["kinds"]), 4, 4), dtype=np.complex128)
            circ = to_product(unpack(d))
        layout = pb.PartitionLayout(circ.n_qubits, e["local"])
        perm = pb.optimize_labels(circ, layout)
        assert list(perm) == e["perm"], e["name"]
        assert pb.predicted_exchange_bytes(circ, layout) == e["identity_bytes"]
        assert pb.predicted_exchange_bytes(pb.relabel(circ, perm), layout) == e["optimized_bytes"]
        assert pb.predicted_exchange_bytes(circ, layout, pb.PrecisionMode.BYTE) == e["identity_bytes_be"]


def test_builders_match_oracle_restatement():
    from oracle.ref_builders import adder, benchmark
    for n in (8, 12, 36):
        a, b = pb.build_benchmark(n), benchmark(n)
        assert [(x.kind, x.qubits) for x in a.gates] == [(x.kind, x.qubits) for x in b.gates]
        assert len(a.gates) == n + 7
    for width, vals in ((2, [1, 2]), (5, [11, 19]), (16, [47302, 18233]), (3, [1, 5, 6])):
        (a, regs), (b, _) = pb.build_adder(width, vals), adder(width, vals)
        assert [(x.kind, x.qubits, x.k) for x in a.gates] == [(x.kind, x.qubits, x.k) for x in b.gates]
    assert len(pb.build_adder(25, [21346502, 12207929])[0].gates) == 1001
    assert len(pb.build_adder(16, [47302, 18233])[0].gates) == 425
    with pytest.raises(ValueError, match="fit"):
        pb.build_adder(3, [8, 1])
    with pytest.raises(ValueError):
        pb.build_benchmark(7)


def test_parser_round_trip(rng):
    for _ in range(10):
        circ = to_product(random_circuit(rng, int(rng.integers(2, 7)), 12))
        text = pb.serialize_circuit(circ)
        again = pb.parse_circuit(text)
        assert pb.serialize_circuit(again) == text
    c = pb.parse_circuit("qubits 3\nRELABEL 2 1 0\nH 0\nM\n")
    assert c.gates[0].qubits == (2,) and c.label_permutation == (2, 1, 0)
    for bad in ["", "qubits 0", "qubits 2\nCPHASE 0 0 1", "qubits 2\nU2 0 1 2", "qubits 2\nM 0",
                "qubits 2\nRELABEL 0 0", "qubits 2\nH 9\n", "qubits 2\nFROB 1", "H 0\n"]:
        with pytest.raises(pb.ParseError):
            pb.parse_circuit(bad)


def test_ledger_and_transport_semantics():
    led = pb.TrafficLedger()
    led.count_send(3 << 30)
    led.count_receive(3 << 30)
    assert gibibytes_exchanged(led) == 6
    leds = [pb.TrafficLedger() for _ in range(2)]
    t = pb.Transport(2, leds)
    with pytest.raises(pb.TransportError):
        t.send(0, 0, None, 1)
    with pytest.raises(pb.TransportError):
        t.recv(1, 0)
    t.send(0, 1, "x", 32)
    with pytest.raises(pb.TransportError):
        t.assert_drained()
    assert t.recv(1, 0) == "x"
    t.assert_drained()
    assert leds[0].inter_rank_bytes_sent == 32 and leds[1].inter_rank_bytes_received == 32
    with pytest.raises(pb.TransportError):
        t.collective([1])


def test_run_circuit_validation_without_gpu():
    c = pb.Circuit(4, (g.h(0),))
    with pytest.raises(ValueError, match="power of two"):
        pb.run_circuit(c, ranks=3)
    with pytest.raises(ValueError):
        pb.run_circuit(c, ranks=2, local_qubits=4)
    with pytest.raises(ValueError):
        pb.run_circuit(pb.Circuit(2, (g.h(5),)))


def test_no_cpu_fallback_without_device():
    if _native.load(require_device=False).sv_device_count is None:
        pytest.skip("library not loadable")
    import ctypes
    n = ctypes.c_int(0)
    _native.load(require_device=False).sv_device_count(ctypes.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(_native.NativeUnavailable):
        pb.run_circuit(pb.build_benchmark(8))
    with pytest.raises(_native.NativeUnavailable):
        pb.kernels.apply_single(np.zeros(4, dtype=np.complex128), 0, g.H_MATRIX) \
            if hasattr(pb, "kernels") else __import__("paper_2511_03359_b200.kernels").kernels.apply_single(
                np.zeros(4, dtype=np.complex128), 0, g.H_MATRIX)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2511_03359_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), f


def _nvrtc_present():
    import ctypes.util
    return any(os.path.exists(p) for p in ("/usr/local/cuda/lib64/libnvrtc.so.12",)) or ctypes.util.find_library("nvrtc")


@pytest.mark.skipif(not _nvrtc_present(), reason="libnvrtc not in this image")
def test_specialised_pass_source_compiles_with_nvrtc(rng):
    """sv_jit.cu prints a fused pass as CUDA source with every constant folded and
    compiles it for sm_100a (CPU only: NVRTC needs no device)."""
    import ctypes
    from paper_2511_03359_b200.device import ops_array
    from paper_2511_03359_b200.engine import gate_to_op
    lib = _native.load(require_device=False)
    circ = random_circuit(rng, 14, 30, measured=False)
    ops = [gate_to_op(gt) for gt in to_product(circ).gates]
    buf = ctypes.create_string_buffer(1 << 20)
    ms = np.zeros(1)
    rc = lib.sv_jit_probe(ops_array(ops), len(ops), 14, buf, len(buf), _native.dptr(ms))
    assert rc >= 1, lib.sv_last_error()
    src = buf.value.decode()
    assert 'extern "C" __global__' in src and "sv_pass" in src
    # no op dispatch left: every op is a template call with literal arguments
    assert not re.search(r"switch|kind\[", src)


@pytest.mark.skipif(not _nvrtc_present(), reason="libnvrtc not in this image")
def test_jit_prepare_queues_one_kernel_per_pass_structure():
    from paper_2511_03359_b200.device import jit_prepare, jit_stats, jit_wait
    from paper_2511_03359_b200.engine import gate_to_op
    hs = [gate_to_op(g.h(q)) for q in range(16)]
    before = jit_stats()
    queued = jit_prepare(16, hs)
    assert queued >= 1
    assert jit_prepare(16, hs) == 0            # same structure: cached
    jit_wait()
    after = jit_stats()
    ready = (after["compiled"] - before["compiled"]) + (after["disk_hits"] - before["disk_hits"])
    assert ready == queued and after["failed"] == before["failed"]   # compiled, or from the disk cache


def test_product_pair_indices_match_reference_goldens(golden):
    """kernels.pair_indices (the product's host helper) vs the reference's outputs."""
    from paper_2511_03359_b200 import kernels
    k = golden("kernels.npz")
    keys = [key for key in k if key.startswith("pairs_")]
    assert keys
    for key in keys:
        _, n, q = key.split("_")
        assert np.array_equal(kernels.pair_indices(int(n), int(q)), k[key]), key
    with pytest.raises(IndexError):
        kernels.pair_indices(6, 6)


def test_product_codebook_resolution_and_dump_match_reference(golden):
    """Codebook.resolution / dump of the product (no device needed) on the reference's
    final propose/merge tables (codec.npz seq*) and on its saturated table."""
    c = golden("codec.npz")
    last = int(c["n_seq"]) - 1
    cb = pb.Codebook()
    cb.mags, cb.thetas = c[f"seq{last}_mags"].copy(), c[f"seq{last}_thetas"].copy()
    cb.ux, cb.uy = c[f"seq{last}_ux"].copy(), c[f"seq{last}_uy"].copy()
    cb.mag_overflow, cb.phase_overflow = (bool(x) for x in c[f"seq{last}_flags"])
    assert np.array_equal(np.array(cb.resolution()), c["resolution"])
    assert cb.dump() == str(c["seq_dump"])


_CACHE_PROBE = r"""
import ctypes, sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2511_03359_b200 import _native
from paper_2511_03359_b200.device import ops_array, jit_stats
from paper_2511_03359_b200.engine import gate_to_op
from tests.circuits import random_circuit, to_product
lib = _native.load(require_device=False)
ops = [gate_to_op(g) for g in to_product(random_circuit(np.random.default_rng(5), 14, 30, measured=False)).gates]
buf = ctypes.create_string_buffer(1 << 20)
ms = np.zeros(1)
assert lib.sv_jit_probe(ops_array(ops), len(ops), 14, buf, len(buf), _native.dptr(ms)) >= 1
st = jit_stats()
print(st["disk_hits"], st["disk_writes"], ms[0])
"""


@pytest.mark.skipif(not _nvrtc_present(), reason="libnvrtc not in this image")
def test_jit_disk_cache_serves_a_new_process(tmp_path):
    """The persistent cubin cache (sv_jit.cu, $SVB200_JIT_CACHE): the first process compiles
    and stores the pass, a second process loads it from disk instead of running NVRTC; a
    corrupted entry is ignored (source compared byte for byte) and recompiled."""
    import subprocess
    import sys
    env = dict(os.environ, SVB200_JIT_CACHE=str(tmp_path))
    run = lambda: subprocess.run([sys.executable, "-c", _CACHE_PROBE, ROOT], env=env, capture_output=True,  # noqa: E731
                                 text=True, timeout=300)
    r1 = run()
    assert r1.returncode == 0, r1.stderr
    hits, writes, _ = r1.stdout.split()
    assert (int(hits), int(writes)) == (0, 1)
    files = list(tmp_path.glob("*.svjit"))
    assert len(files) == 1
    r2 = run()
    hits, writes, ms2 = r2.stdout.split()
    assert (int(hits), int(writes)) == (1, 0) and float(ms2) < 100.0
    data = bytearray(files[0].read_bytes())
    data[20] ^= 0xFF                    # corrupt the stored source
    files[0].write_bytes(bytes(data))
    r3 = run()
    hits, writes, _ = r3.stdout.split()
    assert (int(hits), int(writes)) == (0, 1)


_VARIANT_PROBE = r"""
import ctypes, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2511_03359_b200 import _native
from paper_2511_03359_b200.device import ops_array
from paper_2511_03359_b200.engine import gate_to_op
from tests.circuits import random_circuit, to_product
lib = _native.load(require_device=False)
ops = [gate_to_op(gt) for gt in to_product(random_circuit(np.random.default_rng(5), 16, 40, measured=False)).gates]
buf = ctypes.create_string_buffer(1 << 21)
ms = np.zeros(1)
rc = lib.sv_jit_probe(ops_array(ops), len(ops), 16, buf, len(buf), _native.dptr(ms))
assert rc >= 1, lib.sv_last_error()
print(buf.value.decode())
"""


@pytest.mark.skipif(not _nvrtc_present(), reason="libnvrtc not in this image")
@pytest.mark.parametrize("env,marks", [
    ({"SVB200_PROBE_CFG": "8", "SVB200_BULK": "1"}, ["bulk_g2s(", "mbar_expect_tx(", "mbar_wait("]),
    ({"SVB200_PROBE_CFG": "11"}, ["bar_group(1 + grp, NT)", "cp_async_mbar_arrive(", "mbar_wait(cons + bi"]),
    ({"SVB200_PROBE_CFG": "10"}, ["__launch_bounds__(512, 1)"]),
])
def test_measured_off_variants_still_compile(env, marks):
    """The tile-movement variants kept as measured-and-off options (bulk TMA loads,
    the two-group ring of tile buffers, 2^13 tiles) still generate and compile for
    sm_100a with NVRTC (CPU only), so the A/B numbers in DESIGN.md stay reproducible."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _VARIANT_PROBE, root], capture_output=True, text=True,
                       env=dict(os.environ, **env), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    for m in marks:
        assert m in r.stdout, m


def _advance(ops, free, val):
    import ctypes
    from paper_2511_03359_b200.device import ops_array
    f, v = ctypes.c_uint64(free), ctypes.c_uint64(val)
    _native.check(_native.load(require_device=False).sv_support_advance(ops_array(ops), len(ops),
                                                                        ctypes.byref(f), ctypes.byref(v)))
    return f.value, v.value


def test_support_rule_host_side():
    """sv_support_advance: the support rule of the fused passes (csrc sv_capi.cu support_apply)
    -- monomials on fixed qubits move val, non-monomials and gates touching a free qubit free
    their qubits, diagonal gates keep the set."""
    from paper_2511_03359_b200.engine import gate_to_op
    op = lambda gate: gate_to_op(gate)   # noqa: E731
    assert _advance([op(g.x(3))], 0, 0) == (0, 1 << 3)
    assert _advance([op(g.x(3))], 0, 1 << 3) == (0, 0)
    assert _advance([op(g.h(5))], 0, 0) == (1 << 5, 0)
    assert _advance([op(g.cnot(1, 4))], 0, 1 << 1) == (0, (1 << 1) | (1 << 4))     # control 1: target flips
    assert _advance([op(g.cnot(1, 4))], 0, 0) == (0, 0)                           # control 0: nothing
    assert _advance([op(g.cnot(1, 4))], 1 << 1, 0) == ((1 << 1) | (1 << 4), 0)    # free control: both free
    assert _advance([op(g.z(2)), op(g.cphase(2, 6, 3)), op(g.phase(7, 2))], 0, 1 << 2) == (0, 1 << 2)
    y = gate_to_op(g.y(0))
    assert _advance([y], 0, 0) == (0, 1)                                          # Y: monomial with phase
    # the same rule as the handle-side tracking of a run: a sparse circuit's free set
    from tests.circuits import sparse_circuit
    circ = to_product(sparse_circuit(np.random.default_rng(3), 20, 120, 3, measured=False))
    free, val = _advance([gate_to_op(x) for x in circ.gates], 0, 0)
    assert bin(free).count("1") < 20 and val & free == 0


def test_distributed_support_bookkeeping():
    """CudaBackend's support bookkeeping (no device): remap swaps exchange the bits of the
    physical positions, a rank whose slice lies outside the support skips its passes."""
    from paper_2511_03359_b200.distributed import CudaBackend
    be = CudaBackend.__new__(CudaBackend)
    be.n, be.n_local, be.track = 6, 4, True
    be.sup_free, be.sup_val = 0b000011, 0b100100     # global bit 5 fixed at 1, bit 4 fixed at 0
    for rank, empty in ((0, True), (1, True), (2, False), (3, True)):
        be.rank = rank
        assert be._slice_empty() is empty
    be._swap_bits(((5, 0),))                          # position 5 <-> position 0
    assert (be.sup_free, be.sup_val) == (0b100010, 0b000101)
    be.rank = 0
    assert not be._slice_empty()                      # bit 5 now free, bit 4 fixed at 0
    be.rank = 1
    assert be._slice_empty()
    assert be._pair_is_zero(4) and not be._pair_is_zero(5)
    # local bits a restricted remap swap fixes: the support's fixed local bits minus the victims
    assert be._fixed_local(((4, 2),)) == 0b1111 & ~0b0010 & ~0b0100
    be.track = False
    assert be._fixed_local(((4, 2),)) == 0 and not be._pair_is_zero(4)
