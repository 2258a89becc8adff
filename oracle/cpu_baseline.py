"""CPU baseline timing of the reference algorithm — TEST/BENCH INFRASTRUCTURE ONLY.

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm.
The per-element arithmetic is exactly ref_kernels' restatement of
svsim/kernels.py (numpy complex128, matrix entry first).  The reference
executes one numpy ufunc loop per gate on one core; here the independent
pair blocks of the same reshape view are split over a thread pool (numpy
releases the GIL inside ufunc loops), so the baseline uses every host core
it is given — a stronger baseline than the reference's own single thread.
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import ref_gates

C128 = np.complex128


def _split(view, axis_candidates, parts):
    """Slices of `view` cut along the first axis long enough to give `parts` pieces."""
    for ax in axis_candidates:
        n = view.shape[ax]
        if n >= parts:
            edges = np.linspace(0, n, parts + 1).astype(int)
            out = []
            for a, b in zip(edges[:-1], edges[1:]):
                sl = [slice(None)] * view.ndim
                sl[ax] = slice(a, b)
                out.append(tuple(sl))
            return out
    return [tuple([slice(None)] * view.ndim)]


class ThreadedKernels:
    def __init__(self, threads: int | None = None):
        self.threads = threads or os.cpu_count() or 1
        self.pool = ThreadPoolExecutor(self.threads)

    def close(self):
        self.pool.shutdown()

    def gate1(self, psi, q, m):
        v = psi.reshape(-1, 2, 1 << q)

        def work(sl):
            blk = v[sl]
            a0 = blk[:, 0, :].astype(C128)
            a1 = blk[:, 1, :].astype(C128)
            blk[:, 0, :] = m[0, 0] * a0 + m[0, 1] * a1
            blk[:, 1, :] = m[1, 0] * a0 + m[1, 1] * a1
        list(self.pool.map(work, _split(v, (0, 2), self.threads)))

    def gate2(self, psi, qa, qb, m):
        lo, hi = min(qa, qb), max(qa, qb)
        v = psi.reshape(-1, 2, 1 << (hi - lo - 1), 2, 1 << lo)

        def comp(blk, basis):
            ba, bb = basis & 1, basis >> 1
            bh, bl = (ba, bb) if qa == hi else (bb, ba)
            return blk[:, bh, :, bl, :]

        def work(sl):
            blk = v[sl]
            a = [comp(blk, i).astype(C128) for i in range(4)]
            for r in range(4):
                comp(blk, r)[...] = m[r, 0] * a[0] + m[r, 1] * a[1] + m[r, 2] * a[2] + m[r, 3] * a[3]
        list(self.pool.map(work, _split(v, (0, 2, 4), self.threads)))

    def diag(self, psi, bits, f):
        n = psi.size
        edges = np.linspace(0, n, self.threads + 1).astype(np.int64)

        def work(ab):
            a, b = ab
            idx = np.arange(a, b, dtype=np.int64)
            sel = np.ones(b - a, dtype=bool)
            for bit in bits:
                sel &= ((idx >> bit) & 1) == 1
            seg = psi[a:b]
            seg[sel] = seg[sel].astype(C128) * f
        list(self.pool.map(work, zip(edges[:-1], edges[1:])))

    def apply(self, psi, gate):
        if ref_gates.is_diag(gate):
            self.diag(psi, tuple(gate.qubits), ref_gates.factor_of(gate))
        elif len(gate.qubits) == 1:
            self.gate1(psi, gate.qubits[0], ref_gates.matrix_of(gate))
        else:
            self.gate2(psi, gate.qubits[0], gate.qubits[1], ref_gates.matrix_of(gate))


def gate_bytes(gate, n: int, bpe: int = 16) -> int:
    """Algorithmic HBM bytes of one gate on 2**n amplitudes (read + write of the
    touched elements)."""
    if gate.kind == "M":
        return 0
    if ref_gates.is_diag(gate):
        return 2 * bpe * ((1 << n) >> len(gate.qubits))
    return 2 * bpe * (1 << n)


def time_layers(layers, n: int, threads: int | None = None, rng_seed: int = 1):
    """Run gate layers on a 2**n FP64 state; returns per-layer (seconds, bytes, gates)."""
    rng = np.random.default_rng(rng_seed)
    psi = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(C128)
    psi /= np.linalg.norm(psi)
    tk = ThreadedKernels(threads)
    out = []
    try:
        for layer in layers:
            t0 = time.perf_counter()
            for gate in layer:
                tk.apply(psi, gate)
            dt = time.perf_counter() - t0
            out.append((dt, sum(gate_bytes(gt, n) for gt in layer), len(layer)))
    finally:
        tk.close()
    return out, tk.threads
