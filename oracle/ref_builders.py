"""Oracle restatement of the workload builders (svsim/builders.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from dataclasses import dataclass

from .ref_gates import OGate


@dataclass(frozen=True)
class OCircuit:
    n_qubits: int
    gates: tuple
    label_permutation: tuple = ()

    def __post_init__(self):
        if not self.label_permutation:
            object.__setattr__(self, "label_permutation", tuple(range(self.n_qubits)))


def benchmark(n: int) -> OCircuit:
    """builders.py:14-25 — H on n-1..0, then n-5, n-6, n-1, 0, n-2, 1, then M."""
    if n < 8:
        raise ValueError("benchmark circuit needs at least 8 qubits")
    seq = list(range(n - 1, -1, -1)) + [n - 5, n - 6, n - 1, 0, n - 2, 1]
    return OCircuit(n, tuple(OGate("H", (q,)) for q in seq) + (OGate("M"),))


def adder(width: int, addends):
    """builders.py:28-115 — Draper QFT adder; returns (circuit, {name: range})."""
    if width < 1:
        raise ValueError("register width must be positive")
    if len(addends) not in (2, 3):
        raise ValueError("adder takes two or three addends")
    for a in addends:
        if not 0 <= a < (1 << width):
            raise ValueError(f"addend {a} does not fit in {width} bits")
    R = len(addends)
    res = (R - 1) * width
    out = []
    for i, a in enumerate(addends):                      # builders.py:28-34 (MSB first)
        out += [OGate("X", (i * width + t,)) for t in range(width)
                if (a >> (width - 1 - t)) & 1]
    for u in range(width):                               # builders.py:37-55
        out += [OGate("CPHASE", (res + u, res + t), u - t + 1) for t in range(u - 1, -1, -1)]
        out.append(OGate("H", (res + u,)))
    for i in range(R - 1):                               # builders.py:67-80
        src = i * width
        for ta in range(width):
            out += [OGate("CPHASE", (src + ta, res + t), ta - t + 1) for t in range(ta, -1, -1)]
    for u in range(width - 1, -1, -1):                   # builders.py:58-64
        out.append(OGate("H", (res + u,)))
        out += [OGate("CPHASE", (res + u, res + t), -(u - t + 1)) for t in range(u)]
    out.append(OGate("M"))
    regs = {name: range(i * width, (i + 1) * width)
            for i, name in enumerate(["R1", "R2", "R3"][:R])}
    return OCircuit(R * width, tuple(out)), regs
