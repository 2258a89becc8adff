"""Oracle restatement of the reference gate constants (svsim/gates.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Gates are duck-typed: anything with ``kind``, ``qubits``, ``k`` and ``matrix``
attributes works (the reference's ``svsim.gates.Gate``, the product's
``paper_2511_03359_b200.gates.Gate`` or the ``OGate`` tuple below).
"""
from __future__ import annotations

import math
from collections import namedtuple

import numpy as np

# gates.py:18 — sqrt(1/2) as computed by math.sqrt
_S = math.sqrt(0.5)

# gates.py:20-29 — the constant matrices, complex128
MATRICES = {
    "H": np.array([[_S, _S], [_S, -_S]], dtype=np.complex128),
    "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    # basis index = bit(qa) + 2*bit(qb) with (qa, qb) = (control, target)
    "CNOT": np.array([[1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0], [0, 1, 0, 0]],
                     dtype=np.complex128),
}

DIAGONAL = frozenset(("Z", "PHASE", "CPHASE"))          # gates.py:31
TWO_QUBIT = frozenset(("CNOT", "CPHASE", "U4"))          # gates.py:33

OGate = namedtuple("OGate", "kind qubits k matrix", defaults=((), 0, None))


def angle_of(k: int) -> float:
    """gates.py:85-89 — sign(k) * 2*pi / 2**|k|."""
    if k == 0:
        raise ValueError("phase exponent must be nonzero")
    return math.copysign(2.0 * math.pi / (1 << abs(k)), k)


def factor_of(gate) -> complex:
    """gates.py:96-102 — the diagonal multiplier, computed with numpy's exp."""
    if gate.kind == "Z":
        return complex(-1.0, 0.0)
    if gate.kind in ("PHASE", "CPHASE"):
        return complex(np.exp(1j * angle_of(gate.k)))
    raise ValueError(gate.kind)


def matrix_of(gate) -> np.ndarray:
    """gates.py:105-121 — the dense unitary of a non-diagonal gate."""
    if gate.kind in MATRICES:
        return MATRICES[gate.kind]
    if gate.kind in ("U2", "U4"):
        return np.asarray(gate.matrix, dtype=np.complex128)
    raise ValueError(gate.kind)


def is_diag(gate) -> bool:
    return gate.kind in DIAGONAL
