"""Oracle restatement of the per-gate bulk-synchronous engine and measurement.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates svsim/engine.py (run_circuit 82-105, _execute 149-164, local paths
166-215, BYTE barrier 217-225, exchange rounds 246-377) and svsim/measure.py
(measure_all 59-109) on ONE global array instead of a list of rank slices.
That is exact for the amplitudes: every exchange round in the reference
evaluates the same per-element expression (apply_pair_arrays /
apply_quad_arrays, kernels.py:84-98) as the local kernels, so only the
*grouping* differs — and the grouping is kept where it is observable:

  * BYTE proposals are formed per rank from exactly the values that rank
    computed in the reference's choreography (engine.py:186-215, 246-363),
    because the chain de-duplication in ``propose`` is partition-sensitive;
  * measurement sums are formed per rank slice and combined in rank order
    (measure.py:73-106), which fixes the floating-point summation order;
  * ledgers are charged message by message as the reference's transport
    would (transport.py:30-35).
"""
from __future__ import annotations

import numpy as np

from . import ref_codec, ref_gates, ref_kernels, ref_layout

C128 = np.complex128


class RefRun:
    """What run_circuit returns, as plain arrays (engine.py:40-79)."""

    def __init__(self, n, local, mode):
        self.n_qubits, self.local_qubits, self.mode = n, local, mode
        self.ranks = 1 << (n - local)
        self.ledgers = [ref_layout.new_ledger() for _ in range(self.ranks)]
        self.report = None
        self.codebook = ref_codec.RefCodebook() if mode == "be" else None
        size = 1 << n
        if mode == "be":
            self.mag = np.zeros(size, dtype=np.uint8)
            self.phase = np.zeros(size, dtype=np.uint8)
            self.mag[0] = 1                              # state.py:53-55
        else:
            self.psi = np.zeros(size, dtype=C128 if mode == "fp64" else np.complex64)
            self.psi[0] = 1.0

    def rank_slice(self, r):
        L = 1 << self.local_qubits
        return slice(r * L, (r + 1) * L)

    def working(self):
        if self.mode == "be":
            return self.codebook.decode(self.mag, self.phase)
        return self.psi.astype(C128)

    def gathered_state(self):
        return self.working()

    def rank_states(self):
        """Per-rank storage arrays as LocalState would hold them."""
        out = []
        for r in range(self.ranks):
            sl = self.rank_slice(r)
            if self.mode == "be":
                out.append((self.mag[sl].copy(), self.phase[sl].copy()))
            else:
                out.append(self.psi[sl].copy())
        return out


def _active_ranks(run, gate):
    """engine.py:182-184 — ranks whose global bits of the gate all read 1."""
    loc = run.local_qubits
    return [r for r in range(run.ranks)
            if all((r >> (q - loc)) & 1 for q in gate.qubits if q >= loc)]


def _diag_positions(run, gate):
    """Global positions a diagonal gate modifies, grouped by rank."""
    loc, L = run.local_qubits, 1 << run.local_qubits
    bits = tuple(q for q in gate.qubits if q < loc)
    out = {}
    for r in _active_ranks(run, gate):
        local = np.flatnonzero(ref_kernels.active_mask(L, bits)) if bits else np.arange(L)
        out[r] = local + r * L
    return out


def _producer_positions(run, gate, kind, masks):
    """Global positions whose new values each rank computes (engine.py:246-363)."""
    loc, L, P = run.local_qubits, 1 << run.local_qubits, run.ranks
    half = L // 2
    out = {}
    if kind == "none":
        for r in range(P):
            out[r] = np.arange(r * L, (r + 1) * L)
    elif kind == "pairwise" and len(gate.qubits) == 1:
        m = masks[0]
        for r in range(P):
            offs = np.arange(0, half) if (r & m) == 0 else np.arange(half, L)
            out[r] = np.concatenate([offs + r * L, offs + (r ^ m) * L])
    elif kind == "pairwise":
        m = masks[0]
        (ql,) = [q for q in gate.qubits if q < loc]
        bases = ref_kernels.low_members(loc, ql)
        quarter = len(bases) // 2
        for r in range(P):
            mine = bases[:quarter] if (r & m) == 0 else bases[quarter:]
            offs = np.concatenate([mine, mine + (1 << ql)])
            out[r] = np.concatenate([offs + r * L, offs + (r ^ m) * L])
    else:
        ma, mb = masks
        q4 = L // 4
        for r in range(P):
            pos = (1 if r & ma else 0) + (2 if r & mb else 0)
            base = r & ~(ma | mb)
            members = [base | (ma if p & 1 else 0) | (mb if p & 2 else 0) for p in range(4)]
            offs = np.arange(pos * q4, (pos + 1) * q4)
            out[r] = np.concatenate([offs + mem * L for mem in members])
    return out


def _charge_gate(run, gate, kind, masks, bpe):
    L, P = 1 << run.local_qubits, run.ranks
    if kind == "pairwise":
        for r in range(P):
            ref_layout.charge(run.ledgers, r, r ^ masks[0], (L // 2) * bpe)
    elif kind == "quad":
        ma, mb = masks
        for r in range(P):
            base = r & ~(ma | mb)
            for p in range(4):
                mem = base | (ma if p & 1 else 0) | (mb if p & 2 else 0)
                if mem != r:
                    ref_layout.charge(run.ledgers, r, mem, (L // 4) * bpe)


def _apply_unitary(arr, gate):
    m = ref_gates.matrix_of(gate)
    if len(gate.qubits) == 1:
        ref_kernels.gate1(arr, gate.qubits[0], m)
    else:
        ref_kernels.gate2(arr, gate.qubits[0], gate.qubits[1], m)


def _gate_fp(run, gate, kind, masks):
    if ref_gates.is_diag(gate):
        loc = run.local_qubits
        bits = tuple(q for q in gate.qubits if q < loc)
        f = ref_gates.factor_of(gate)
        for r in _active_ranks(run, gate):
            ref_kernels.diag(run.psi[run.rank_slice(r)], bits, f)
    else:
        _apply_unitary(run.psi, gate)


def _gate_byte(run, gate, kind, masks):
    cb = run.codebook
    work = run.working()
    if ref_gates.is_diag(gate):
        groups = _diag_positions(run, gate)
        f = ref_gates.factor_of(gate)
        produced = {r: work[pos] * f for r, pos in groups.items()}
    else:
        _apply_unitary(work, gate)
        groups = _producer_positions(run, gate, kind, masks)
        produced = {r: work[pos] for r, pos in groups.items()}
    empty = np.zeros(0, dtype=C128)
    cb.merge([cb.propose(produced.get(r, empty)) for r in range(run.ranks)])
    for r, pos in groups.items():
        mi, pi = cb.encode(produced[r])
        run.mag[pos] = mi
        run.phase[pos] = pi


def measure(run):
    """measure.py:59-109 — (qx, qy, qz, norm_deviation) with rank-ordered sums."""
    n, loc, P = run.n_qubits, run.local_qubits, run.ranks
    L = 1 << loc
    half = L // 2
    bpe = ref_layout.BYTES_PER_ELEMENT[run.mode]
    full = run.working()
    works = [full[run.rank_slice(r)] for r in range(P)]
    norms = [float(np.real(np.vdot(w, w))) for w in works]
    total = sum(norms)
    qx, qy, qz = [], [], []
    for q in range(n):
        ones, cross = [0.0] * P, [0j] * P
        if q < loc:
            for r in range(P):
                v = works[r].reshape(-1, 2, 1 << q)
                ones[r] = float(np.sum(np.abs(v[:, 1, :]) ** 2))
                cross[r] = complex(np.sum(v[:, 0, :].conj() * v[:, 1, :]))
        else:
            m = 1 << (q - loc)
            for r in range(P):
                ref_layout.charge(run.ledgers, r, r ^ m, half * bpe)
            for r in range(P):
                low = (r & m) == 0
                sl = slice(0, half) if low else slice(half, L)
                own, other = works[r][sl], works[r ^ m][sl]
                a0, a1 = (own, other) if low else (other, own)
                cross[r] = complex(np.sum(a0.conj() * a1))
                if (r >> (q - loc)) & 1:
                    ones[r] = norms[r]
        s, z = sum(cross), sum(ones)
        qx.append((1.0 - 2.0 * s.real) / 2.0)
        qy.append((1.0 - 2.0 * s.imag) / 2.0)
        qz.append(z)
    return tuple(qx), tuple(qy), tuple(qz), abs(total - 1.0)


def run_circuit(circuit, ranks=1, local_qubits=None, mode="fp64") -> RefRun:
    """engine.py:82-105 with the dispatch of engine.py:149-164."""
    if ranks < 1 or ranks & (ranks - 1):
        raise ValueError("rank count must be a power of two")
    n = circuit.n_qubits
    if local_qubits is None:
        local_qubits = n - (ranks.bit_length() - 1)
    ref_layout.check_layout(n, local_qubits)
    if (1 << (n - local_qubits)) != ranks:
        raise ValueError("rank count does not cover the qubits")
    run = RefRun(n, local_qubits, mode)
    for gate in circuit.gates:
        kind, masks, _, bpe = ref_layout.plan(n, local_qubits, gate, mode)
        if gate.kind == "M":
            run.report = measure(run)
        else:
            _charge_gate(run, gate, kind, masks, bpe)
            if mode == "be":
                _gate_byte(run, gate, kind, masks)
            else:
                _gate_fp(run, gate, kind, masks)
        for led in run.ledgers:
            led["gate_operations"] += 1
    return run


def relabel_report(report, perm):
    """measure.py:36-42 — present a (qx, qy, qz, dev) report in program labels."""
    qx, qy, qz, dev = report
    return (tuple(qx[p] for p in perm), tuple(qy[p] for p in perm),
            tuple(qz[p] for p in perm), dev)
