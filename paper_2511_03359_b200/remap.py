"""Global<->local qubit-remapping planner (the paper's traffic optimizer, B200 form).

The reference moves data for every gate that touches a rank bit: a pairwise
exchange of L/2 elements per rank whose result half comes back through
shared memory (engine.py:246-377), i.e. physically L/2 in each direction
per gate, every time the qubit is used.  It only has a *static* relabeling
optimizer (optimize.py:44-72).

On the B200 build a gate on a global qubit g is made local by swapping g
with a local qubit l: one NVLink pass that moves L/2 elements per direction
per rank pair (svk_swap_peer), after which every later gate on that logical
qubit is free until it is evicted again.  The planner tracks the logical ->
physical qubit permutation and picks the victim l with Belady's rule (the
local qubit whose next non-diagonal use is farthest away), preferring
physical positions >= MIN_VICTIM so fused tile passes keep their contiguous
low qubits.  Diagonal gates never move data (layout.py:81-82): their global
bits only select which ranks are active.

Results are bit-identical to the unpermuted execution (swaps are pure moves;
each gate runs the same arithmetic on the same amplitudes); reports and
exported states are mapped back to logical order.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import gates as g

MIN_VICTIM = 5


@dataclass(frozen=True)
class Swap:
    global_pos: int     # physical rank-bit position (>= n_local)
    local_pos: int      # physical local position (< n_local)


@dataclass(frozen=True)
class PhysGate:
    ordinal: int
    gate: object        # the logical gate
    qubits: tuple       # physical positions of gate.qubits
    perm: tuple = ()    # logical -> physical permutation in force


@dataclass(frozen=True)
class Measure:
    ordinal: int
    perm: tuple         # logical qubit -> physical position at that point


class RemapPlanner:
    def __init__(self, n_qubits: int, n_local: int, remap: bool = True, min_victim: int = MIN_VICTIM):
        self.n = n_qubits
        self.n_local = n_local
        self.remap = remap
        self.min_victim = min(min_victim, max(n_local - 1, 0))
        self.pos = list(range(n_qubits))      # logical -> physical
        self.at = list(range(n_qubits))       # physical -> logical

    def _next_uses(self, gates):
        """next_use[i][q]: index of the next non-diagonal gate after i using logical q."""
        inf = len(gates) + 1
        nxt = [inf] * self.n
        table = [None] * len(gates)
        for i in range(len(gates) - 1, -1, -1):
            table[i] = list(nxt)
            gate = gates[i]
            if gate.kind != "M" and not g.is_diagonal(gate):
                for q in gate.qubits:
                    nxt[q] = i
        return table

    def _swap(self, gp: int, lp: int) -> Swap:
        a, b = self.at[gp], self.at[lp]
        self.at[gp], self.at[lp] = b, a
        self.pos[a], self.pos[b] = lp, gp
        return Swap(gp, lp)

    def plan(self, gates) -> list:
        gates = list(gates)
        steps = []
        nxt = self._next_uses(gates) if self.remap else None
        for i, gate in enumerate(gates):
            if gate.kind == "M":
                steps.append(Measure(i, tuple(self.pos)))
                continue
            needs = [] if g.is_diagonal(gate) else [q for q in gate.qubits if self.pos[q] >= self.n_local]
            if needs and self.remap:
                busy = {self.pos[q] for q in gate.qubits}
                for q in needs:
                    cands = [lp for lp in range(self.n_local) if lp not in busy]
                    high = [lp for lp in cands if lp >= self.min_victim]
                    # Belady (evict the local qubit needed latest) over the high physical
                    # positions, so tile passes keep their contiguous low qubits
                    lp = max(high or cands, key=lambda p: (nxt[i][self.at[p]], p))
                    steps.append(self._swap(self.pos[q], lp))
                    busy.add(lp)
            steps.append(PhysGate(i, gate, tuple(self.pos[q] for q in gate.qubits), tuple(self.pos)))
        return steps


def swap_traffic_elements(steps, n_local: int) -> int:
    """Elements each rank sends over the link for the planned swaps (L/2 per swap)."""
    return sum(1 for s in steps if isinstance(s, Swap)) * ((1 << n_local) // 2)
