"""Seeded workload circuits shared by the golden generator and the tests.

Restates the reference test fixtures (pkg/tests/conftest.py:8-70): a QR-based
Haar unitary, a random circuit over the full gate set and the byte-exact
"exact class" circuit.  Circuits are built from ``oracle.ref_gates.OGate`` so
the same object can be fed to the reference (via ``to_reference``), to the
oracle and — via ``to_product`` — to the B200 package.
"""
from __future__ import annotations

import numpy as np

from oracle.ref_builders import OCircuit
from oracle.ref_gates import OGate

SEED = 20240817                                        # conftest.py:85-87


def haar_unitary(rng: np.random.Generator, dim: int) -> np.ndarray:
    """conftest.py:8-11."""
    a = rng.normal(size=(dim, dim)) + 1j * rng.normal(size=(dim, dim))
    q, r = np.linalg.qr(a)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def random_circuit(rng, n_qubits: int, depth: int, measured: bool = True) -> OCircuit:
    """conftest.py:14-44 — same draw sequence as the reference fixture."""
    kinds = ["H", "X", "Y", "Z", "PHASE", "CPHASE", "CNOT", "U2", "U4"]
    out = []
    for _ in range(depth):
        kind = kinds[rng.integers(len(kinds))]
        q1 = int(rng.integers(n_qubits))
        q2 = int((q1 + 1 + rng.integers(n_qubits - 1)) % n_qubits)
        k = int(rng.integers(1, 5))
        if kind in ("H", "X", "Y", "Z"):
            out.append(OGate(kind, (q1,)))
        elif kind == "PHASE":
            out.append(OGate("PHASE", (q1,), k if rng.integers(2) else -k))
        elif kind == "CPHASE":
            out.append(OGate("CPHASE", (q1, q2), k))
        elif kind == "CNOT":
            out.append(OGate("CNOT", (q1, q2)))
        elif kind == "U2":
            out.append(OGate("U2", (q1,), 0, haar_unitary(rng, 2)))
        else:
            out.append(OGate("U4", (q1, q2), 0, haar_unitary(rng, 4)))
    if measured:
        out.append(OGate("M"))
    return OCircuit(n_qubits, tuple(out))


def exact_class_circuit(rng, n_qubits: int, depth: int, measured: bool = True) -> OCircuit:
    """conftest.py:47-70 — H, X, CNOT, Z, pi phases only."""
    kinds = ["H", "X", "CNOT", "Z", "PHASE", "CPHASE"]
    out = []
    for _ in range(depth):
        kind = kinds[rng.integers(len(kinds))]
        q1 = int(rng.integers(n_qubits))
        q2 = int((q1 + 1 + rng.integers(n_qubits - 1)) % n_qubits)
        if kind in ("H", "X", "Z"):
            out.append(OGate(kind, (q1,)))
        elif kind == "CNOT":
            out.append(OGate("CNOT", (q1, q2)))
        elif kind == "PHASE":
            out.append(OGate("PHASE", (q1,), 1))
        else:
            out.append(OGate("CPHASE", (q1, q2), 1))
    if measured:
        out.append(OGate("M"))
    return OCircuit(n_qubits, tuple(out))


def sparse_circuit(rng, n_qubits: int, depth: int, n_spread: int = 4, measured: bool = True) -> OCircuit:
    """Random circuit whose non-monomial gates (H, U2, U4) touch only ``n_spread`` random
    qubits; X / Y / CNOT (monomials: they move a basis state) and Z / PHASE / CPHASE
    (diagonal) act anywhere.  From |0..0> the state keeps a small support -- the case support
    tracking (csrc/sv_capi.cu Support, byte_state.py sup_free) restricts passes to."""
    spread = [int(q) for q in rng.choice(n_qubits, size=n_spread, replace=False)]
    kinds = ["H", "U2", "U4", "X", "Y", "CNOT", "Z", "PHASE", "CPHASE"]
    out = []
    for _ in range(depth):
        kind = kinds[rng.integers(len(kinds))]
        q1 = int(rng.integers(n_qubits))
        q2 = int((q1 + 1 + rng.integers(n_qubits - 1)) % n_qubits)
        k = int(rng.integers(1, 5))
        if kind in ("H", "U2"):
            q = spread[rng.integers(n_spread)]
            out.append(OGate("H", (q,)) if kind == "H" else OGate("U2", (q,), 0, haar_unitary(rng, 2)))
        elif kind == "U4":
            a, b = (int(x) for x in rng.choice(spread, size=2, replace=False))
            out.append(OGate("U4", (a, b), 0, haar_unitary(rng, 4)))
        elif kind in ("X", "Y", "Z"):
            out.append(OGate(kind, (q1,)))
        elif kind == "PHASE":
            out.append(OGate("PHASE", (q1,), k if rng.integers(2) else -k))
        elif kind == "CPHASE":
            out.append(OGate("CPHASE", (q1, q2), k))
        else:
            out.append(OGate("CNOT", (q1, q2)))
    if measured:
        out.append(OGate("M"))
    return OCircuit(n_qubits, tuple(out))


# --- (de)serialisation so circuits travel inside golden .npz files ---------

def pack(circuit) -> dict:
    gates = circuit.gates
    G = len(gates)
    kinds = np.array([g.kind for g in gates], dtype="U8")
    qubits = np.full((G, 2), -1, dtype=np.int64)
    ks = np.zeros(G, dtype=np.int64)
    mats = np.zeros((G, 4, 4), dtype=np.complex128)
    for i, g in enumerate(gates):
        qubits[i, :len(g.qubits)] = g.qubits
        ks[i] = g.k
        if g.matrix is not None:
            m = np.asarray(g.matrix)
            mats[i, :m.shape[0], :m.shape[1]] = m
    return dict(n_qubits=np.int64(circuit.n_qubits), kinds=kinds, qubits=qubits, ks=ks,
                mats=mats, label=np.array(circuit.label_permutation, dtype=np.int64))


def unpack(d, prefix: str = "") -> OCircuit:
    kinds = d[prefix + "kinds"]
    qubits = d[prefix + "qubits"]
    ks = d[prefix + "ks"]
    mats = d[prefix + "mats"]
    out = []
    for i, kind in enumerate(kinds):
        kind = str(kind)
        qs = tuple(int(q) for q in qubits[i] if q >= 0)
        mat = None
        if kind == "U2":
            mat = mats[i, :2, :2].copy()
        elif kind == "U4":
            mat = mats[i].copy()
        out.append(OGate(kind, qs, int(ks[i]), mat))
    return OCircuit(int(d[prefix + "n_qubits"]), tuple(out),
                    tuple(int(p) for p in d[prefix + "label"]))


def to_reference(circuit, ref):
    """Build the reference package's Circuit from an OCircuit."""
    gates = tuple(ref.gates.Gate(g.kind, tuple(g.qubits), g.k,
                                 None if g.matrix is None else np.asarray(g.matrix, dtype=np.complex128))
                  for g in circuit.gates)
    return ref.Circuit(circuit.n_qubits, gates, tuple(circuit.label_permutation))


def to_product(circuit):
    """Build the B200 package's Circuit from an OCircuit."""
    from paper_2511_03359_b200 import Circuit, gates as pg
    gates = tuple(pg.Gate(g.kind, tuple(g.qubits), g.k,
                          None if g.matrix is None else np.asarray(g.matrix, dtype=np.complex128))
                  for g in circuit.gates)
    return Circuit(circuit.n_qubits, gates, tuple(circuit.label_permutation))


def ladder_cases():
    """SURVEY 8(c) parity ladder (tests/golden/ladder.json): (name, circuit, mode, ranks).
    C1 is build_benchmark(20) FP64 at P=1 (builders.py:14-25)."""
    from oracle.ref_builders import adder, benchmark
    return [
        ("C1_bench20", benchmark(20), "fp64", (1,)),
        ("bench22", benchmark(22), "fp64", (1, 8)),
        ("bench24", benchmark(24), "fp64", (1, 8)),
        ("adder11", adder(11, [1234, 813])[0], "fp64", (1, 8)),
        ("bench22_fp32", benchmark(22), "fp32", (1,)),
        ("bench20_be", benchmark(20), "be", (8,)),
        ("bench22_be", benchmark(22), "be", (8,)),
        ("adder10_be", adder(10, [700, 323])[0], "be", (8,)),
    ]
