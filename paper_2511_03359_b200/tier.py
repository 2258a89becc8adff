"""Two-tier state memory: HBM (fast) plus pinned host memory (slow) per rank.

The reference (``svsim/tier.py``) models the paper's strategy 5 -- explicit
copies between the fast and slow memory of a GH200 steered by a look-ahead
over the gate sequence -- as a staging plan plus counters.
This module keeps that API and its numbers (``TierConfig`` tier.py:37-50,
``StagingGroup``/``StagingPlan`` 53-83, ``plan_passes`` 98-143,
``recommended_fast_bytes`` 146-153, ``TierAccount`` 156-208,
``naive_staging_bytes`` 211-224): the plan and the ledger counters are
golden-checked against the reference (tests/golden/tier.json).

On the B200 the plan is also EXECUTED when asked (``run_circuit(...,
tier_config=cfg, tier_execute=True)``, or automatically when the state does
not fit in HBM): the rank slice is cut into chunks of ``chunk_bytes``; the
chunks ``TierAccount.fast_resident`` marks stay in HBM, the others live in
pinned host memory and are staged through ``STAGING_SLOTS`` HBM slots by the
copy engines, overlapped with the fused passes (csrc/sv_tier.cu).  Arithmetic
is the same kernels' on the same amplitudes, so tiered results equal
untiered results bit for bit, as in the reference.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import gates as g
from .layout import TrafficLedger
from .state import PrecisionMode

STAGING_SLOTS = 4            # fast-tier chunk slots kept free for staging (tier.py:30)
SLOW_FAST_RATIO = (4, 11)    # paper: best LPDDR5:HBM3 data ratio 4/11 (tier.py:33)


@dataclass(frozen=True)
class TierConfig:
    """Fast-tier capacity and chunk size in bytes per rank; look-ahead window in gates."""
    fast_capacity_bytes: int
    chunk_bytes: int
    lookahead_window: int = 64

    def __post_init__(self):
        c = self.chunk_bytes
        if c < 1 or (c & (c - 1)) != 0:
            raise ValueError("chunk size must be a power of two")
        if self.fast_capacity_bytes < 2 * c:
            raise ValueError("fast tier must hold at least two chunks")
        if self.lookahead_window < 1:
            raise ValueError("look-ahead window must be positive")


@dataclass(frozen=True)
class StagingGroup:
    """Gates executed under one staging decision: kind "run" (chunk-local), "mid"
    (chunk pairs / quads, `chunk_groups`), "exchange" (inter-rank) or "measure"."""
    kind: str
    gate_indices: tuple
    chunk_groups: tuple = ()


@dataclass(frozen=True)
class StagingPlan:
    groups: tuple
    chunk_qubits: int
    n_chunks: int

    def passes(self):
        """(chunks, gate indices) in execution order."""
        every = tuple(range(self.n_chunks))
        seq = []
        for grp in self.groups:
            if grp.kind == "run":
                seq += [(j, grp.gate_indices) for j in every]
            elif grp.kind == "mid":
                seq += [(members, grp.gate_indices) for members in grp.chunk_groups]
            else:
                seq.append((every, grp.gate_indices))
        return seq


def _kind(gate, chunk_qubits: int, n_local: int) -> str:
    if gate.kind == "M":
        return "measure"
    if g.is_diagonal(gate):
        return "run"            # element-wise: any chunk on its own
    if max(gate.qubits) >= n_local:
        return "exchange"
    return "run" if max(gate.qubits) < chunk_qubits else "mid"


def _chunk_groups(high_masks, n_chunks: int) -> tuple:
    """Every chunk j with none of the mask bits set, followed by its partners (the
    subsets of the masks added in order): (j, j|m0) or (j, j|m0, j|m1, j|m0|m1)."""
    any_mask = 0
    for m in high_masks:
        any_mask |= m
    out = []
    for j in range(n_chunks):
        if j & any_mask:
            continue
        members = [j]
        for m in high_masks:
            members = members + [x | m for x in members]
        out.append(tuple(members))
    return tuple(out)


def plan_passes(gate_list, config, n_local: int, mode: PrecisionMode) -> StagingPlan:
    """Look-ahead staging plan of `gate_list` for one rank's 2^n_local slice."""
    bpe = mode.bytes_per_element
    state_bytes = bpe << n_local
    chunk_bytes = min(config.chunk_bytes, state_bytes)
    if chunk_bytes < bpe or state_bytes % chunk_bytes:
        raise ValueError("chunk size must hold at least one element and divide the state")
    c = (chunk_bytes // bpe).bit_length() - 1
    n_chunks = state_bytes // chunk_bytes
    kinds = [_kind(gt, c, n_local) for gt in gate_list]
    groups = []
    i, n = 0, len(gate_list)
    while i < n:
        k = kinds[i]
        if k == "run":
            end = i
            while end < n and kinds[end] == "run" and end - i < config.lookahead_window:
                end += 1
            groups.append(StagingGroup("run", tuple(range(i, end))))
            i = end
            continue
        if k == "mid":
            masks = [1 << (q - c) for q in gate_list[i].qubits if q >= c]
            if (chunk_bytes << len(masks)) > config.fast_capacity_bytes:
                raise ValueError(f"gate needs {1 << len(masks)} co-resident chunks; shrink the chunk size")
            groups.append(StagingGroup("mid", (i,), _chunk_groups(masks, n_chunks)))
        else:
            groups.append(StagingGroup(k, (i,)))
        i += 1
    return StagingPlan(tuple(groups), c, n_chunks)


def recommended_fast_bytes(state_bytes: int, chunk_bytes: int) -> int:
    """Fast-tier data target for an oversubscribed state: slow:fast near 4:11,
    rounded down to whole chunks."""
    slow, fast = SLOW_FAST_RATIO
    return (state_bytes * fast // (slow + fast)) // chunk_bytes * chunk_bytes


class TierAccount:
    """Chunk residency of one rank and the staging charged to its ledger."""

    def __init__(self, state_bytes: int, config, ledger: TrafficLedger):
        self.config = config
        self.ledger = ledger
        self.chunk_bytes = min(config.chunk_bytes, state_bytes)
        self.n_chunks = state_bytes // self.chunk_bytes
        if state_bytes <= config.fast_capacity_bytes:
            n_fast = self.n_chunks
        else:
            budget = max(config.fast_capacity_bytes // self.chunk_bytes - STAGING_SLOTS, 0)
            target = recommended_fast_bytes(state_bytes, self.chunk_bytes) // self.chunk_bytes
            n_fast = min(budget, target, self.n_chunks)
        # spread the fast chunks evenly: chunk j is fast when floor((j+1)F/C) steps up at j
        C = self.n_chunks
        self.fast_resident = [((j + 1) * n_fast) // C != (j * n_fast) // C for j in range(C)]
        self.static_fast_bytes = n_fast * self.chunk_bytes
        self.high_water_bytes = self.static_fast_bytes

    @property
    def slow_chunks(self) -> list:
        return [j for j, fast in enumerate(self.fast_resident) if not fast]

    @property
    def slow_bytes(self) -> int:
        return self.chunk_bytes * len(self.slow_chunks)

    def _stage(self, chunks: int) -> None:
        level = self.static_fast_bytes + chunks * self.chunk_bytes
        if level > self.config.fast_capacity_bytes:
            raise ValueError("staging would overflow the fast tier")
        if level > self.high_water_bytes:
            self.high_water_bytes = level

    def account(self, group: StagingGroup) -> None:
        cb = self.chunk_bytes
        if group.kind == "mid":
            for members in group.chunk_groups:
                k = sum(1 for j in members if not self.fast_resident[j])
                if k:
                    self._stage(k)
                    self.ledger.count_tier(2 * cb * k, 2 * k)
            return
        # run / exchange: each slow chunk in and back out once; measure: in only
        write_back = group.kind in ("run", "exchange")
        if not write_back and group.kind != "measure":
            return
        for _ in self.slow_chunks:
            self._stage(1)
            self.ledger.count_tier(2 * cb if write_back else cb, 2 if write_back else 1)


def naive_staging_bytes(gate_list, config, n_local: int, mode: PrecisionMode) -> int:
    """Cost of staging the slow part in and out around every gate (M: in only)."""
    acct = TierAccount(mode.bytes_per_element << n_local, config, TrafficLedger())
    slow = acct.slow_bytes
    return sum(slow if gt.kind == "M" else 2 * slow for gt in gate_list)


def tier_layout_flags(accounts) -> list:
    """Per-chunk fast flags of the whole (all-ranks) buffer: rank r's slice is chunks
    [r*C, (r+1)*C) and follows its own TierAccount's placement."""
    flags = []
    for acct in accounts:
        flags += [1 if f else 0 for f in acct.fast_resident]
    return flags


class TieredDeviceState:
    """A state split between HBM and pinned host memory (csrc/sv_tier.cu), driven by a
    StagingPlan: the physical form of the reference's tier model.  Same surface as
    device.DeviceState where the engine and LocalState mirrors use it."""

    def __init__(self, n_qubits: int, mode, chunk_qubits: int, fast_flags, device: int = 0,
                 slots: int = STAGING_SLOTS):
        import ctypes

        import numpy as np

        from . import _native as nat
        lib = nat.load()
        self.n_qubits = int(n_qubits)
        self.mode_code = nat.mode_code(mode)
        self.chunk_qubits = int(chunk_qubits)
        self.device = device
        flags = np.ascontiguousarray(np.asarray(fast_flags, dtype=np.uint8))
        if flags.size != 1 << (self.n_qubits - self.chunk_qubits):
            raise ValueError("one fast flag per chunk expected")
        h = ctypes.c_void_p()
        nat.check(lib.svt_create(device, self.n_qubits, self.mode_code, self.chunk_qubits,
                                 flags.ctypes.data_as(ctypes.c_void_p), slots, ctypes.byref(h)))
        self.handle = h
        self.version = 0
        self.launches = 0

    @property
    def size(self) -> int:
        return 1 << self.n_qubits

    @property
    def dtype(self):
        import numpy as np
        return np.complex64 if self.mode_code == 1 else np.complex128

    def _touch(self, launches: int = 1):
        self.version += 1
        self.launches += launches

    def zero(self, unit_index: int | None = 0, lazy: bool = False) -> None:
        from . import _native as nat
        nat.check(nat.load().svt_zero_state(self.handle, -1 if unit_index is None else unit_index))
        self._touch(0)

    def apply_run(self, ops, tile_bits: int = 12) -> None:
        from . import _native as nat
        from .device import ops_array
        if ops:
            nat.check(nat.load().svt_apply_run(self.handle, ops_array(ops), len(ops), tile_bits))
            self._touch(len(ops))

    def apply_pairing(self, op) -> None:
        import ctypes

        from . import _native as nat
        nat.check(nat.load().svt_apply_pairing(self.handle, ctypes.byref(op)))
        self._touch()

    def measure(self):
        import numpy as np

        from . import _native as nat
        n = self.n_qubits
        norm, ones, cross = np.zeros(1), np.zeros(n), np.zeros(2 * n)
        nat.check(nat.load().svt_measure(self.handle, nat.dptr(norm), nat.dptr(ones), nat.dptr(cross)))
        self.launches += 1
        return float(norm[0]), ones.copy(), cross[0::2] + 1j * cross[1::2]

    def export(self, first: int = 0, count: int | None = None):
        import ctypes

        import numpy as np

        from . import _native as nat
        count = self.size - first if count is None else count
        out = np.empty(count, dtype=self.dtype)
        nat.check(nat.load().svt_export(self.handle, out.ctypes.data_as(ctypes.c_void_p), first, count))
        return out

    def import_(self, values, first: int = 0) -> None:
        import ctypes

        import numpy as np

        from . import _native as nat
        arr = np.ascontiguousarray(np.asarray(values), dtype=self.dtype)
        nat.check(nat.load().svt_import(self.handle, arr.ctypes.data_as(ctypes.c_void_p), first, arr.size))
        self._touch(0)

    def export_storage(self, first: int, count: int):
        return self.export(first, count)

    def import_storage(self, values, first: int = 0) -> None:
        self.import_(values, first)

    def synchronize(self) -> None:
        from . import _native as nat
        nat.check(nat.load().svt_synchronize(self.handle))

    def stats(self) -> dict:
        import ctypes

        from . import _native as nat
        v = (ctypes.c_uint64 * 8)()
        nat.check(nat.load().svt_stats(self.handle, v))
        keys = ("h2d_bytes", "d2h_bytes", "h2d_copies", "d2h_copies", "zero_copy_bytes", "slot_memsets",
                "passes", "hbm_fast_bytes")
        return dict(zip(keys, (int(x) for x in v)))

    def free(self) -> None:
        if getattr(self, "handle", None):
            from . import _native as nat
            nat.load(require_device=False).svt_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
