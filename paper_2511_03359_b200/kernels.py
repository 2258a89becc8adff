"""Array-level gate operators (``svsim.kernels`` surface) executed on the B200.

Mirrors /root/reference/pkg/src/svsim/kernels.py: ``pair_indices`` (21-27),
``apply_single`` (30-40), ``apply_two`` (43-64), ``apply_diagonal`` (67-81),
``apply_pair_arrays`` (84-88), ``apply_quad_arrays`` (91-98) and
``norm_squared`` (101-103), with the same signatures, in-place semantics and
exception types.  The caller's host array is copied to HBM, updated by a
libsvb200 kernel and copied back — the host <-> device copies are part of the
call, exactly what a user of the reference API pays.  Arithmetic is FP64
with numpy's operand order, so results are bit-identical to the reference;
complex64 arrays are computed in FP64 and rounded once on store.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat

_MODE_OF = {np.dtype(np.complex128): nat.SV_FP64, np.dtype(np.complex64): nat.SV_FP32}


def pair_indices(n_local: int, q: int) -> np.ndarray:
    """Ascending indices with bit q clear (host integer helper, as in the reference)."""
    if not 0 <= q < n_local:
        raise IndexError(f"qubit {q} outside local range {n_local}")
    t = np.arange(1 << (n_local - 1), dtype=np.int64)
    return ((t >> q) << (q + 1)) | (t & ((1 << q) - 1))


class _Staged:
    """Host arrays staged in one device allocation for the duration of a call."""

    def __init__(self, arrays, mode: int):
        self.arrays = arrays
        self.mode = mode
        self.stream = nat.Stream(0)
        self.itemsize = 16 if mode == nat.SV_FP64 else 8
        self.offsets, off = [], 0
        for a in arrays:
            self.offsets.append(off)
            off += (a.size * self.itemsize + 255) // 256 * 256
        self.buf = nat.DeviceBuffer(max(off, 256))
        for a, o in zip(arrays, self.offsets):
            if a.size:
                self._h2d(a, o)

    def _h2d(self, a, o):
        a = np.ascontiguousarray(a)
        nat.check(nat.load().sv_copy_h2d(self.buf.offset(o), a.ctypes.data_as(ctypes.c_void_p),
                                         a.nbytes, self.stream.ptr))

    def ptr(self, i):
        return self.buf.offset(self.offsets[i])

    def fetch(self, i, out: np.ndarray):
        if out.size == 0:
            return out
        tmp = out if out.flags.c_contiguous else np.empty_like(out, order="C")
        nat.check(nat.load().sv_copy_d2h(tmp.ctypes.data_as(ctypes.c_void_p), self.ptr(i), tmp.nbytes,
                                         self.stream.ptr))
        if tmp is not out:
            out[...] = tmp
        return out

    def close(self):
        self.stream.synchronize()
        self.buf.free()
        self.stream.close()


def _write_back(st: "_Staged", i: int, psi: np.ndarray) -> None:
    out = np.empty(psi.size, dtype=psi.dtype)
    st.fetch(i, out)
    psi[...] = out.reshape(psi.shape)


def _mode_of(psi: np.ndarray) -> int:
    try:
        return _MODE_OF[psi.dtype]
    except KeyError:
        raise TypeError(f"amplitude arrays must be complex128 or complex64, got {psi.dtype}") from None


def apply_single(psi: np.ndarray, q: int, matrix: np.ndarray) -> None:
    """In-place 2x2 update of all (i, i + 2**q) pairs."""
    n = psi.size
    if q < 0 or (1 << q) >= n:
        raise IndexError(f"qubit {q} outside local array of {n} amplitudes")
    mode = _mode_of(psi)
    st = _Staged([psi.ravel()], mode)
    try:
        m = nat.mat_buffer(matrix)
        nat.check(nat.load().svk_apply_1q(st.ptr(0), n, mode, q, nat.dptr(m), st.stream.ptr))
        _write_back(st, 0, psi)
    finally:
        st.close()


def apply_two(psi: np.ndarray, qa: int, qb: int, matrix: np.ndarray) -> None:
    """In-place 4x4 update; matrix basis index bit(qa) + 2*bit(qb)."""
    n = psi.size
    if qa == qb:
        raise ValueError("two-qubit gate requires distinct qubits")
    if (1 << qa) >= n or (1 << qb) >= n:
        raise IndexError(f"qubits ({qa}, {qb}) outside local array of {n} amplitudes")
    mode = _mode_of(psi)
    st = _Staged([psi.ravel()], mode)
    try:
        m = nat.mat_buffer(matrix)
        nat.check(nat.load().svk_apply_2q(st.ptr(0), n, mode, qa, qb, nat.dptr(m), st.stream.ptr))
        _write_back(st, 0, psi)
    finally:
        st.close()


def apply_diagonal(psi: np.ndarray, local_bits: tuple, factor: complex) -> None:
    """Multiply by ``factor`` where every listed local bit reads 1 (all if none)."""
    mode = _mode_of(psi)
    mask = 0
    for b in local_bits:
        mask |= 1 << int(b)
    st = _Staged([psi.ravel()], mode)
    try:
        f = np.array([complex(factor).real, complex(factor).imag])
        nat.check(nat.load().svk_apply_diag(st.ptr(0), psi.size, mode, mask, nat.dptr(f), st.stream.ptr))
        _write_back(st, 0, psi)
    finally:
        st.close()


def apply_pair_arrays(a0: np.ndarray, a1: np.ndarray, matrix: np.ndarray):
    """2x2 across two aligned buffers; returns new complex128 buffers."""
    b0 = np.asarray(a0).astype(np.complex128)
    b1 = np.asarray(a1).astype(np.complex128)
    if b0.shape != b1.shape:
        raise ValueError("pair buffers must have the same shape")
    st = _Staged([b0.ravel(), b1.ravel()], nat.SV_FP64)
    try:
        m = nat.mat_buffer(matrix)
        nat.check(nat.load().svk_pair_update(st.ptr(0), st.ptr(1), b0.size, nat.SV_FP64, nat.dptr(m),
                                             st.stream.ptr))
        st.fetch(0, b0.reshape(-1))
        st.fetch(1, b1.reshape(-1))
    finally:
        st.close()
    return b0, b1


def apply_quad_arrays(components: list, matrix: np.ndarray) -> list:
    """4x4 across four aligned buffers (basis order 0..3); returns new buffers."""
    parts = [np.asarray(c).astype(np.complex128) for c in components]
    if len(parts) != 4 or len({p.shape for p in parts}) != 1:
        raise ValueError("quad update takes four buffers of one shape")
    st = _Staged([p.ravel() for p in parts], nat.SV_FP64)
    try:
        m = nat.mat_buffer(matrix)
        ptrs = (ctypes.c_void_p * 4)(*[st.ptr(i) for i in range(4)])
        nat.check(nat.load().svk_quad_update(ptrs, parts[0].size, nat.SV_FP64, nat.dptr(m), st.stream.ptr))
        for i, p in enumerate(parts):
            st.fetch(i, p.reshape(-1))
    finally:
        st.close()
    return parts


def norm_squared(psi: np.ndarray) -> float:
    """Sum of |a|^2 (a device reduction over a zero-padded power-of-two buffer)."""
    a = np.asarray(psi).ravel()
    if a.dtype not in _MODE_OF:
        a = a.astype(np.complex128)
    mode = _mode_of(a)
    size = 1 << max(0, (a.size - 1).bit_length())
    padded = np.zeros(size, dtype=a.dtype)
    padded[:a.size] = a
    st = _Staged([padded], mode)
    try:
        k = size.bit_length() - 1
        norm = np.zeros(1)
        ones = np.zeros(max(k, 1))
        cross = np.zeros(2 * max(k, 1))
        nat.check(nat.load().svk_measure(st.ptr(0), size, mode, nat.dptr(norm), nat.dptr(ones),
                                         nat.dptr(cross), st.stream.ptr))
    finally:
        st.close()
    return float(norm[0])
