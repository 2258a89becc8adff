"""Oracle restatement of the strided gate kernels (svsim/kernels.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The arithmetic contract being restated:
  * every update is computed in complex128 whatever the storage dtype, and the
    store back into complex64 rounds once (kernels.py:1-5);
  * 2x2 / 4x4 rows are ``m[r,0]*a0 + m[r,1]*a1 (+ m[r,2]*a2) (+ m[r,3]*a3)``,
    matrix entry first, summed left to right (kernels.py:39-40, 60-64);
  * diagonal updates multiply the array first: ``a * factor`` (kernels.py:75, 81).
numpy evaluates each complex product as (fma(ar,br,-(ai*bi)), fma(ar,bi,ai*br))
with ``a`` the first operand; restating the same expressions reproduces it.
"""
from __future__ import annotations

import numpy as np

C128 = np.complex128


def low_members(n_local: int, q: int) -> np.ndarray:
    """kernels.py:21-27 — ascending indices whose bit q is clear."""
    if q < 0 or q >= n_local:
        raise IndexError(f"qubit {q} outside local range {n_local}")
    t = np.arange(1 << (n_local - 1), dtype=np.int64)
    below = t & ((1 << q) - 1)
    return ((t >> q) << (q + 1)) | below


def _rows2(m, a0, a1):
    return m[0, 0] * a0 + m[0, 1] * a1, m[1, 0] * a0 + m[1, 1] * a1


def _rows4(m, a):
    return [m[r, 0] * a[0] + m[r, 1] * a[1] + m[r, 2] * a[2] + m[r, 3] * a[3]
            for r in range(4)]


def gate1(psi: np.ndarray, q: int, m: np.ndarray) -> None:
    """kernels.py:30-40 — in-place 2x2 on all pairs (i, i + 2**q)."""
    stride = 1 << q
    if stride >= psi.size:
        raise IndexError(f"qubit {q} outside local array of {psi.size} amplitudes")
    blocks = psi.reshape(-1, 2, stride)
    lo = blocks[:, 0, :].astype(C128)
    hi = blocks[:, 1, :].astype(C128)
    blocks[:, 0, :], blocks[:, 1, :] = _rows2(m, lo, hi)


def _quad_views(psi: np.ndarray, qa: int, qb: int):
    """The four strided component views in basis order bit(qa) + 2*bit(qb)."""
    low, high = min(qa, qb), max(qa, qb)
    v = psi.reshape(-1, 2, 1 << (high - low - 1), 2, 1 << low)
    out = []
    for basis in range(4):
        ba, bb = basis & 1, basis >> 1
        b_high, b_low = (ba, bb) if qa == high else (bb, ba)
        out.append(v[:, b_high, :, b_low, :])
    return out


def gate2(psi: np.ndarray, qa: int, qb: int, m: np.ndarray) -> None:
    """kernels.py:43-64 — in-place 4x4 on the quadruples of (qa, qb)."""
    if qa == qb:
        raise ValueError("two-qubit gate requires distinct qubits")
    if (1 << qa) >= psi.size or (1 << qb) >= psi.size:
        raise IndexError(f"qubits ({qa}, {qb}) outside local array of {psi.size} amplitudes")
    views = _quad_views(psi, qa, qb)
    comps = [v.astype(C128) for v in views]
    for view, row in zip(views, _rows4(m, comps)):
        view[...] = row


def active_mask(size: int, bits) -> np.ndarray:
    idx = np.arange(size, dtype=np.int64)
    sel = np.ones(size, dtype=bool)
    for b in bits:
        sel &= ((idx >> b) & 1) == 1
    return sel


def diag(psi: np.ndarray, bits, factor: complex) -> None:
    """kernels.py:67-81 — multiply (array first) where all local ``bits`` are 1."""
    if not bits:
        psi *= C128(factor)
        return
    sel = active_mask(psi.size, bits)
    psi[sel] = psi[sel].astype(C128) * factor


def pair_arrays(a0, a1, m):
    """kernels.py:84-88."""
    return _rows2(m, a0.astype(C128), a1.astype(C128))


def quad_arrays(parts, m):
    """kernels.py:91-98."""
    return _rows4(m, [p.astype(C128) for p in parts])


def norm2(psi: np.ndarray) -> float:
    """kernels.py:101-103."""
    w = psi.astype(C128, copy=False)
    return float(np.real(np.vdot(w, w)))
