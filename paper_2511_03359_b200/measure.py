"""All-qubit three-axis report (``svsim.measure`` surface) computed on the B200.

Mirrors /root/reference/pkg/src/svsim/measure.py: ``ExpectationReport``
(25-48; Q = (1 - <sigma>) / 2 per axis, Qz = P(bit = 1)) and ``measure_all``
(59-109).  The reference makes one full pass over the state per qubit and an
L/2 exchange per global qubit; here one tiled device pass produces the norm
and every Qz, and ceil((N - 12) / 7) further passes produce the cross sums
for all remaining qubits (sv_measure.cu).  The ledger is still charged one
half-slice message per global qubit per rank, as the reference does
(measure.py:83-91), so traffic accounting stays identical.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .layout import PartitionLayout
from .transport import ExchangeToken


@dataclass(frozen=True)
class ExpectationReport:
    qx: tuple
    qy: tuple
    qz: tuple
    norm_deviation: float = 0.0

    @property
    def n_qubits(self) -> int:
        return len(self.qz)

    def relabelled(self, permutation: tuple) -> "ExpectationReport":
        """Program labels: label q lives at storage index permutation[q]."""
        pick = lambda seq: tuple(seq[p] for p in permutation)  # noqa: E731
        return ExpectationReport(pick(self.qx), pick(self.qy), pick(self.qz), self.norm_deviation)

    def max_difference(self, other: "ExpectationReport") -> float:
        return max(max(abs(a - b) for a, b in zip(mine, theirs))
                   for mine, theirs in ((self.qx, other.qx), (self.qy, other.qy), (self.qz, other.qz)))


def report_from_sums(norm: float, ones, cross) -> ExpectationReport:
    qx = tuple(float((1.0 - 2.0 * c.real) / 2.0) for c in cross)
    qy = tuple(float((1.0 - 2.0 * c.imag) / 2.0) for c in cross)
    qz = tuple(float(v) for v in ones)
    return ExpectationReport(qx, qy, qz, norm_deviation=abs(norm - 1.0))


def charge_measurement(layout: PartitionLayout, transport, bytes_per_element: int, order,
                       ordinal: int = -1) -> None:
    """The reference's measurement messages: one L/2 half per global qubit per rank."""
    half = layout.local_size // 2
    for q in range(layout.local_qubits, layout.total_qubits):
        mask = 1 << (q - layout.local_qubits)
        for rank in order:
            lo = (rank & mask) == 0
            token = ExchangeToken(ordinal, rank, rank ^ mask, half if lo else 0, half)
            transport.send(rank, rank ^ mask, token, half * bytes_per_element)
        for rank in order:
            transport.recv(rank, rank ^ mask)


def _whole_buffer(states):
    """The DeviceState holding all rank slices contiguously in rank order, if any."""
    dev = getattr(states[0], "_dev", None)
    if dev is None:
        return None
    size = states[0].size
    for r, s in enumerate(states):
        if getattr(s, "_dev", None) is not dev or s._offset != r * size:
            return None
    return dev if dev.size == size * len(states) else None


def device_sums(states, codebook=None):
    """(norm, ones[N], cross[N]) of the gathered state, computed on the device."""
    dev = _whole_buffer(states)
    if dev is None:
        from .device import DeviceState
        from .state import PrecisionMode
        n_total = states[0].n_local + (len(states).bit_length() - 1)
        mode = PrecisionMode.FP64 if states[0].mode is PrecisionMode.BYTE else states[0].mode
        dev = DeviceState(n_total, mode, device=getattr(getattr(states[0], "_dev", None), "device", 0))
        for r, s in enumerate(states):
            vals = s.working(codebook) if s.mode is PrecisionMode.BYTE else s.psi
            dev.import_(vals, r * s.size)
    return dev.measure_sums(codebook) if hasattr(dev, "measure_sums") else dev.measure()


def measure_all(states, layout: PartitionLayout, transport, ledgers, codebook=None,
                rank_order=None) -> ExpectationReport:
    order = list(rank_order) if rank_order is not None else list(range(layout.rank_count))
    transport.collective([None] * layout.rank_count)          # norm gather (measure.py:74)
    charge_measurement(layout, transport, states[0].mode.bytes_per_element, order)
    norm, ones, cross = device_sums(states, codebook)
    for _ in range(layout.total_qubits):                      # cross / ones gathers (102-103)
        transport.collective([None] * layout.rank_count)
        transport.collective([None] * layout.rank_count)
    return report_from_sums(norm, ones, np.asarray(cross))
