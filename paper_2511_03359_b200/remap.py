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

Several global qubits needed close together are fetched in ONE batched swap
(SwapGroup, svk_swap_group): k global qubits exchanged with k victims is an
all-to-all inside each 2^k-rank group that moves (1 - 2^-k) L elements per
direction per rank, against k L/2 for k single swaps.  A global qubit joins
the batch when its next use comes before the next use of the victim it would
evict (and within `window` gates).

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
class SwapGroup:
    pairs: tuple        # ((global_pos, local_pos), ...), k >= 2, simultaneous


def deposit(code: int, positions) -> int:
    """Bits of `code` (bit j) placed at positions[j]."""
    out = 0
    for j, p in enumerate(positions):
        out |= ((code >> j) & 1) << p
    return out


def group_schedule(rank: int, pairs, n_local: int, n_local_elems: int):
    """This rank's share of a batched swap: [(member_rank, vmask, own_pat, peer_pat,
    t_begin, t_count)].  Rank r with group code c trades its amplitudes whose victim
    bits read m with member m's amplitudes whose victim bits read c; the pair splits
    the remaining-bit range in half (the lower code takes the first half)."""
    bits = [gp - n_local for gp, _ in pairs]
    lps = [lp for _, lp in pairs]
    k = len(pairs)
    vmask = deposit((1 << k) - 1, lps)
    c = sum(((rank >> b) & 1) << j for j, b in enumerate(bits))
    rest = n_local_elems >> k
    half = rest // 2
    base = rank & ~sum(1 << b for b in bits)
    out = []
    for m in range(1 << k):
        if m == c:
            continue
        member = base | sum(((m >> j) & 1) << b for j, b in enumerate(bits))
        t0 = 0 if c < m else half
        out.append((member, vmask, deposit(m, lps), deposit(c, lps), t0, half))
    return out


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
    def __init__(self, n_qubits: int, n_local: int, remap: bool = True, min_victim: int = MIN_VICTIM,
                 batch: bool = True, window: int = 64):
        self.batch = batch and n_local >= 2
        self.window = window
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
                chosen = []

                def victim():
                    cands = [lp for lp in range(self.n_local) if lp not in busy]
                    high = [lp for lp in cands if lp >= self.min_victim]
                    # Belady (evict the local qubit needed latest) over the high physical
                    # positions, so tile passes keep their contiguous low qubits
                    return max(high or cands, key=lambda p: (nxt[i][self.at[p]], p)) if cands else None

                for q in needs:
                    lp = victim()
                    chosen.append((self.pos[q], lp))
                    busy.add(lp)
                if self.batch:
                    soon = sorted((nxt[i][q], q) for q in range(self.n)
                                  if self.pos[q] >= self.n_local and q not in gate.qubits)
                    for when, q in soon:
                        if when > i + self.window:
                            break
                        lp = victim()
                        if lp is None or nxt[i][self.at[lp]] <= when:
                            break
                        chosen.append((self.pos[q], lp))
                        busy.add(lp)
                if len(chosen) == 1:
                    steps.append(self._swap(*chosen[0]))
                else:
                    for gp, lp in chosen:
                        self._swap(gp, lp)
                    steps.append(SwapGroup(tuple(chosen)))
            steps.append(PhysGate(i, gate, tuple(self.pos[q] for q in gate.qubits), tuple(self.pos)))
        return steps


def swap_traffic_elements(steps, n_local: int) -> int:
    """Elements each rank sends over the link for the planned swaps (L/2 per
    single swap, (1 - 2^-k) L per batched swap of k qubits)."""
    L = 1 << n_local
    total = 0
    for s in steps:
        if isinstance(s, Swap):
            total += L // 2
        elif isinstance(s, SwapGroup):
            k = len(s.pairs)
            total += L - (L >> k)
    return total
