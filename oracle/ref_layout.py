"""Oracle restatement of partitioning, exchange plans and ledgers (svsim/layout.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from . import ref_gates

BYTES_PER_ELEMENT = {"fp64": 16, "fp32": 8, "be": 2}     # state.py:24-27
_MEM_SHIFT = {"fp64": 4, "fp32": 3, "be": 1}              # layout.py:50-55


def memory_bytes(n_qubits: int, mode: str) -> int:
    if n_qubits < 1:
        raise ValueError("need at least one qubit")
    return 1 << (n_qubits + _MEM_SHIFT[mode])


def check_layout(total: int, local: int) -> None:
    """layout.py:31-36."""
    if total < 1:
        raise ValueError("need at least one qubit")
    if not 1 <= local <= total:
        raise ValueError(f"local qubits {local} not in [1, {total}]")


def plan(total: int, local: int, gate, mode: str):
    """layout.py:78-96 — (kind, masks, element_count, bytes_per_element)."""
    bpe = BYTES_PER_ELEMENT[mode]
    if gate.kind == "M" or ref_gates.is_diag(gate):
        return ("none", (), 0, bpe)
    high = [q for q in gate.qubits if q >= local]
    if not high:
        return ("none", (), 0, bpe)
    size = 1 << local
    if len(high) == 1:
        if len(gate.qubits) == 2 and size < 4:
            raise ValueError("two-qubit exchange needs at least 4 local amplitudes")
        return ("pairwise", (1 << (high[0] - local),), size // 2, bpe)
    if size < 4:
        raise ValueError("two-qubit exchange needs at least 4 local amplitudes")
    return ("quad", tuple(1 << (q - local) for q in high), 3 * size // 4, bpe)


def new_ledger() -> dict:
    """layout.py:99-121 — counters as a plain dict (snapshot() layout)."""
    return dict(inter_rank_bytes_sent=0, inter_rank_bytes_received=0,
                inter_rank_messages=0, tier_bytes_moved=0, tier_transfer_count=0,
                gate_operations=0)


def charge(ledgers, src: int, dst: int, nbytes: int) -> None:
    """transport.py:30-35 — one counted message src -> dst."""
    ledgers[src]["inter_rank_bytes_sent"] += nbytes
    ledgers[src]["inter_rank_messages"] += 1
    ledgers[dst]["inter_rank_bytes_received"] += nbytes
