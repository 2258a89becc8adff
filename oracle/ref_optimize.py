"""Oracle restatement of the static relabel optimizer (svsim/optimize.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from . import ref_gates, ref_layout
from .ref_builders import OCircuit


def relabel(circuit, perm):
    """optimize.py:19-27 — gate qubit q -> perm[q]; label record composes."""
    if sorted(perm) != list(range(circuit.n_qubits)):
        raise ValueError("relabeling must be a bijection on the qubit indices")
    gates = tuple(ref_gates.OGate(g.kind, tuple(perm[q] for q in g.qubits), g.k, g.matrix)
                  for g in circuit.gates)
    label = tuple(perm[p] for p in circuit.label_permutation)
    return OCircuit(circuit.n_qubits, gates, label)


def predicted_bytes(circuit, local: int, mode: str = "fp64") -> int:
    """optimize.py:30-41 — gate-exchange bytes summed over all ranks."""
    P = 1 << (circuit.n_qubits - local)
    tot = 0
    for g in circuit.gates:
        _, _, count, bpe = ref_layout.plan(circuit.n_qubits, local, g, mode)
        tot += count * bpe * P
    return tot


def optimize_labels(circuit, local: int):
    """optimize.py:44-72 — heaviest exchange-inducing qubits to the lowest labels."""
    n = circuit.n_qubits
    L = 1 << local
    w = [0] * n
    for g in circuit.gates:
        if g.kind == "M" or ref_gates.is_diag(g):
            continue
        vol = L // 2 if len(g.qubits) == 1 else 3 * L // 4
        for q in g.qubits:
            w[q] += vol
    ranked = sorted(range(n), key=lambda q: (-w[q], q))
    perm = [0] * n
    for new, q in enumerate(ranked):
        perm[q] = new
    perm = tuple(perm)
    if predicted_bytes(relabel(circuit, perm), local) < predicted_bytes(circuit, local):
        return perm
    return tuple(range(n))
