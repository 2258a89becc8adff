"""Circuit execution on the B200 (``svsim.engine`` surface).

Mirrors /root/reference/pkg/src/svsim/engine.py: ``RunResult`` (40-79) and
``run_circuit`` (82-105) with the same keyword arguments, validation and
error wrapping (``RuntimeError("gate {ordinal} ({kind}): ...")`` for a
transport failure, 161-162).

Execution model (single process, one GPU):
  * all 2**(N-N') rank slices live in ONE HBM buffer in rank order, so rank r
    owns elements [r*L, (r+1)*L) exactly as in the reference layout
    (layout.py:26-47).  A gate on a global qubit is then an ordinary strided
    update over the whole buffer — the reference's pairwise / quad exchange
    rounds (engine.py:246-363) compute the same per-element expressions, so
    the amplitudes are bit-identical and nothing needs to cross a link;
  * the control plane still walks the reference choreography message by
    message through the transport, so ledgers, partners, failure injection
    and rank-order shuffling behave exactly as in the reference;
  * consecutive gates are queued and flushed as fused tile passes
    (svk_apply_fused): every gate keeps its own rounding, so fusion changes
    the number of HBM passes, never the results.
Multi-GPU execution (one process per GPU, NVLink exchanges) is in
distributed.py.
"""
from __future__ import annotations

import random
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import gates as g
from .circuit import Circuit, validate_circuit
from .device import gate_op
from .layout import PartitionLayout, TrafficLedger, plan_exchange
from .measure import ExpectationReport, charge_measurement, report_from_sums
from .state import LocalState, PrecisionMode
from .transport import ExchangeToken, Transport, TransportError

FUSE_QUEUE_LIMIT = 1024
# SVB200_SUPPORT=0: run_circuit processes every tile of every pass (no support tracking)
import os as _os
_SUPPORT_TRACKING = _os.environ.get("SVB200_SUPPORT", "1") != "0"


@dataclass
class RunResult:
    circuit: Circuit
    layout: PartitionLayout
    mode: PrecisionMode
    states: list
    ledgers: list
    report: ExpectationReport | None
    codebook: object
    tier_accounts: list | None
    wall_time_seconds: float
    device_stats: dict = field(default_factory=dict)

    @property
    def gate_operations(self) -> int:
        return self.ledgers[0].gate_operations

    @property
    def total_bytes_sent(self) -> int:
        return sum(led.inter_rank_bytes_sent for led in self.ledgers)

    @property
    def total_messages(self) -> int:
        return sum(led.inter_rank_messages for led in self.ledgers)

    @property
    def total_tier_bytes(self) -> int:
        return sum(led.tier_bytes_moved for led in self.ledgers)

    @property
    def total_tier_transfers(self) -> int:
        return sum(led.tier_transfer_count for led in self.ledgers)

    def gathered_state(self) -> np.ndarray:
        """Global state vector (complex128) assembled from the rank slices."""
        dev = self.states[0].device_state
        if self.mode is PrecisionMode.BYTE:
            return dev.decode()
        return dev.export().astype(np.complex128)

    def report_in_program_labels(self) -> ExpectationReport | None:
        if self.report is None:
            return None
        return self.report.relabelled(self.circuit.label_permutation)


def gate_to_op(gate: g.Gate):
    """One gate as an sv_op over the global index (all ranks in one buffer)."""
    if g.is_diagonal(gate):
        mask = 0
        for q in gate.qubits:
            mask |= 1 << q
        f = g.diagonal_factor(gate)
        return gate_op(nat.SV_OP_DIAG, mask=mask, data=(f.real, f.imag))
    m = nat.mat_buffer(g.unitary_matrix(gate))
    if len(gate.qubits) == 1:
        return gate_op(nat.SV_OP_1Q, qa=gate.qubits[0], data=m)
    return gate_op(nat.SV_OP_2Q, qa=gate.qubits[0], qb=gate.qubits[1], data=m)


def tier_ledger_plan(circuit: Circuit, layout: PartitionLayout, mode: PrecisionMode, tier_config, ledgers):
    """The reference's staging plan of the whole circuit and one TierAccount per rank,
    charging `ledgers` (engine.py:127-133)."""
    from .tier import TierAccount, plan_passes
    plan = plan_passes(circuit.gates, tier_config, layout.local_qubits, mode)
    state_bytes = layout.local_size * mode.bytes_per_element
    return plan, [TierAccount(state_bytes, tier_config, led) for led in ledgers]


def _fits_in_hbm(n_bytes: int, device: int) -> bool:
    import ctypes
    free, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
    nat.check(nat.load().sv_mem_info(device, ctypes.byref(free), ctypes.byref(total)))
    return n_bytes + (1 << 30) <= free.value + nat_cached_bytes()


def nat_cached_bytes() -> int:
    import ctypes
    v = ctypes.c_uint64(0)
    nat.check(nat.load(require_device=False).sv_cached_bytes(ctypes.byref(v)))
    return int(v.value)


def run_circuit(circuit: Circuit, *, ranks: int = 1, local_qubits: int | None = None,
                mode: PrecisionMode = PrecisionMode.FP64, tier_config=None,
                rank_order_seed: int | None = None, transport_factory=Transport,
                device: int = 0, fuse: bool = True, tile_bits: int = 12,
                tier_execute: bool | None = None, exact_diagonals: bool = True,
                track_support: bool = True) -> RunResult:
    """svsim.run_circuit (engine.py:82-105) on one B200.

    tier_config (svsim TierConfig or tier.TierConfig): the reference's staging plan and
    TierAccount counters are charged exactly as svsim does.  tier_execute: also EXECUTE
    the plan with the slow chunks in pinned host memory (csrc/sv_tier.cu); None = only
    when the FP64/FP32 state does not fit in HBM.  Results are identical either way.

    exact_diagonals=False (FP64, fused, resident): runs of consecutive diagonal gates in a
    fused pass multiply each amplitude by their combined factor -- amplitudes within 1e-12
    relative of the reference (the north star's FP64 tolerance) instead of bit-identical;
    the QFT adder's CPHASE runs then cost one multiply per register mask, not per gate.

    track_support (FP64/FP32, one GPU, default on): the state starts as |0..0>; the device
    records which index bits may differ from it (freed by non-monomial gates, moved by
    monomials, untouched by diagonal gates) and fused passes and the measurement read
    only the tiles that can hold nonzero amplitudes.  The skipped amplitudes are zeros
    that stay zero, so results are identical; False processes every tile."""
    validate_circuit(circuit)
    if ranks < 1 or ranks & (ranks - 1):
        raise ValueError("rank count must be a power of two")
    if local_qubits is None:
        local_qubits = circuit.n_qubits - (ranks.bit_length() - 1)
    layout = PartitionLayout(circuit.n_qubits, local_qubits)
    if layout.rank_count != ranks:
        raise ValueError(f"{ranks} ranks with {local_qubits} local qubits does not cover "
                         f"{circuit.n_qubits} qubits")
    start = time.perf_counter()
    tier = None
    if tier_config is not None:
        tier = _TierRun(circuit, layout, mode, tier_config, tier_execute, device)
    launches0 = nat.launch_count()
    combine = (not exact_diagonals and fuse and mode is PrecisionMode.FP64
               and not (tier is not None and tier.execute))
    eng = _Engine(circuit, layout, mode, rank_order_seed, transport_factory, device, fuse, tile_bits, tier,
                  combine_diag=combine, support_tracking=track_support and _SUPPORT_TRACKING)
    eng.run()
    eng.launches = nat.launch_count() - launches0
    return RunResult(circuit, layout, mode, eng.states, eng.ledgers, eng.report, eng.codebook,
                     tier.accounts if tier else None, time.perf_counter() - start, eng.stats())


class _TierRun:
    """tier_config of one run: the plan (accounts bound to the engine's ledgers later)
    and whether the plan is executed physically."""

    def __init__(self, circuit, layout, mode, cfg, execute, device):
        from .tier import plan_passes
        self.cfg = cfg
        self.plan = plan_passes(circuit.gates, cfg, layout.local_qubits, mode)   # validates first
        self.accounts = None
        if execute is None:
            execute = mode is not PrecisionMode.BYTE and not _fits_in_hbm(
                (1 << circuit.n_qubits) * mode.bytes_per_element, device)
        if execute and mode is PrecisionMode.BYTE:
            raise NotImplementedError("physical tier execution holds FP64 / FP32 storage; BYTE states "
                                      "(2 B/amplitude) stay resident and are charged the plan's counters")
        if execute and self.plan.chunk_qubits < 5:
            raise ValueError("physical tier execution needs chunks of at least 32 amplitudes")
        self.execute = bool(execute)

    def bind(self, layout, mode, ledgers):
        from .tier import TierAccount
        state_bytes = layout.local_size * mode.bytes_per_element
        self.accounts = [TierAccount(state_bytes, self.cfg, led) for led in ledgers]


class _Engine:
    def __init__(self, circuit, layout, mode, rank_order_seed, transport_factory, device, fuse,
                 tile_bits, tier=None, combine_diag=False, support_tracking=True):
        self.circuit = circuit
        self.combine_diag = combine_diag
        self.tier = tier
        self.layout = layout
        self.mode = mode
        self.fuse = fuse
        self.tile_bits = tile_bits
        n = layout.rank_count
        self.ledgers = [TrafficLedger() for _ in range(n)]
        self.transport = transport_factory(n, self.ledgers)
        self.order = list(range(n))
        if rank_order_seed is not None:
            random.Random(rank_order_seed).shuffle(self.order)
        self.report = None
        self.codebook = None
        if tier is not None:
            tier.bind(layout, mode, self.ledgers)
        if mode is PrecisionMode.BYTE:
            from .byte_state import ByteEngineState
            self.dev = ByteEngineState(circuit.n_qubits, layout, device=device)
            self.codebook = self.dev.codebook
        elif tier is not None and tier.execute:
            from .tier import TieredDeviceState, tier_layout_flags
            t0 = time.perf_counter()
            self.dev = TieredDeviceState(circuit.n_qubits, mode, tier.plan.chunk_qubits,
                                         tier_layout_flags(tier.accounts), device=device)
            tier.setup_seconds = time.perf_counter() - t0
        else:
            from .device import DeviceState
            self.dev = DeviceState(circuit.n_qubits, mode, device=device)
            if combine_diag:
                self.dev.set_diag_combine(True)
            # the state starts as |0..0>: fused passes skip the tiles that can only hold zeros
            self.dev.set_support_tracking(support_tracking)
        if mode is PrecisionMode.BYTE:
            self.dev.zero(0)
        else:   # the first fused pass generates |0..0> instead of reading a written state
            self.dev.zero(0, lazy=fuse)
        L = layout.local_size
        self.states = [LocalState(layout.local_qubits, mode, _device_state=self.dev, _offset=r * L)
                       for r in range(n)]
        self.pending = []
        self.gates_applied = 0

    # -- device queue ----------------------------------------------------------------
    def _enqueue(self, gate):
        if self.mode is PrecisionMode.BYTE:
            self.dev.apply_gate(gate, self.layout)
            self.gates_applied += 1
            return
        self.pending.append(gate_to_op(gate))
        self.gates_applied += 1
        if not self.fuse or len(self.pending) >= FUSE_QUEUE_LIMIT:
            self._flush()

    def _flush(self):
        if not self.pending:
            return
        if self.fuse:
            self.dev.apply_fused(self.pending, self.tile_bits)
        else:
            for op in self.pending:
                self._apply_single_op(op)
        self.pending = []

    def _apply_single_op(self, op):
        m = np.array(op.m[:32])
        if op.kind == nat.SV_OP_1Q:
            nat.check(nat.load().sv_apply_1q(self.dev.handle, op.qa, nat.dptr(m)))
        elif op.kind == nat.SV_OP_2Q:
            nat.check(nat.load().sv_apply_2q(self.dev.handle, op.qa, op.qb, nat.dptr(m)))
        else:
            nat.check(nat.load().sv_apply_diag(self.dev.handle, op.diag_mask, nat.dptr(m)))
        self.dev._touch()

    # -- control plane -----------------------------------------------------------------
    def _exchange_messages(self, plan, ordinal):
        """The reference's send phase then receive phase (engine.py:246-363)."""
        L = self.layout.local_size
        if plan.kind == "pairwise":
            mask = plan.masks[0]
            for rank in self.order:
                tok = ExchangeToken(ordinal, rank, rank ^ mask, 0, plan.element_count)
                self.transport.send(rank, rank ^ mask, tok, plan.bytes_per_rank)
            for rank in self.order:
                self.transport.recv(rank, rank ^ mask)
            return
        ma, mb = plan.masks
        quarter = L // 4

        def member(rank, pos):
            return (rank & ~(ma | mb)) | (ma if pos & 1 else 0) | (mb if pos & 2 else 0)

        for rank in self.order:
            for pos in range(4):
                dst = member(rank, pos)
                if dst != rank:
                    tok = ExchangeToken(ordinal, rank, dst, pos * quarter, quarter)
                    self.transport.send(rank, dst, tok, quarter * plan.bytes_per_element)
        for rank in self.order:
            for pos in range(4):
                src = member(rank, pos)
                if src != rank:
                    self.transport.recv(rank, src)

    def _measure(self, ordinal):
        self._flush()
        P = self.layout.rank_count
        self.transport.collective([None] * P)
        charge_measurement(self.layout, self.transport, self.mode.bytes_per_element, self.order, ordinal)
        if self.mode is PrecisionMode.BYTE:
            norm, ones, cross = self.dev.measure_sums()
        else:
            norm, ones, cross = self.dev.measure()
        for _ in range(self.layout.total_qubits):
            self.transport.collective([None] * P)
            self.transport.collective([None] * P)
        self.report = report_from_sums(norm, ones, cross)

    def _run_tiered(self):
        """Group by group as the reference (engine.py:137-145): every rank's TierAccount is
        charged, then the group's gates run -- physically staged when the plan executes."""
        physical = self.tier.execute
        gates = self.circuit.gates
        for grp in self.tier.plan.groups:
            for acct in self.tier.accounts:
                acct.account(grp)
            ops = []
            for ordinal in grp.gate_indices:
                gate = gates[ordinal]
                plan = plan_exchange(self.layout, gate, self.mode)
                try:
                    if gate.kind == "M":
                        if physical and ops:
                            self.dev.apply_run(ops, self.tile_bits)
                            ops = []
                        self._measure(ordinal)
                    else:
                        if plan.kind != "none":
                            self._exchange_messages(plan, ordinal)
                        if not physical:
                            self._enqueue(gate)
                        elif grp.kind == "run":
                            ops.append(gate_to_op(gate))
                        else:
                            self.dev.apply_pairing(gate_to_op(gate))
                        if physical:
                            self.gates_applied += 1
                except TransportError as exc:
                    raise RuntimeError(f"gate {ordinal} ({gate.kind}): {exc}") from exc
                for led in self.ledgers:
                    led.gate_operations += 1
            if physical and ops:
                self.dev.apply_run(ops, self.tile_bits)
        self._flush()
        self.dev.synchronize()
        self.transport.assert_drained()

    def run(self):
        t0 = time.perf_counter()
        try:
            self._run()
        finally:
            self.run_seconds = time.perf_counter() - t0

    def _run(self):
        if self.tier is not None:
            if self.fuse and not self.tier.execute and self.mode in (PrecisionMode.FP64, PrecisionMode.FP32):
                from .device import jit_prepare
                jit_prepare(self.circuit.n_qubits, [gate_to_op(g) for g in self.circuit.gates if g.kind != "M"],
                            self.tile_bits, self.dev.mode_code)
            self._run_tiered()
            return
        if self.fuse and self.mode in (PrecisionMode.FP64, PrecisionMode.FP32):
            # queue the specialised pass kernels of the whole circuit (compiled in the
            # background; passes whose kernel is not ready yet run the generic one)
            from .device import jit_prepare
            jit_prepare(self.circuit.n_qubits, [gate_to_op(g) for g in self.circuit.gates if g.kind != "M"],
                        self.tile_bits, self.dev.mode_code, combine_diag=self.combine_diag)
        for ordinal, gate in enumerate(self.circuit.gates):
            plan = plan_exchange(self.layout, gate, self.mode)
            try:
                if gate.kind == "M":
                    self._measure(ordinal)
                else:
                    if plan.kind != "none":
                        self._exchange_messages(plan, ordinal)
                    self._enqueue(gate)
            except TransportError as exc:
                raise RuntimeError(f"gate {ordinal} ({gate.kind}): {exc}") from exc
            for led in self.ledgers:
                led.gate_operations += 1
        self._flush()
        self.dev.synchronize()
        self.transport.assert_drained()

    def stats(self) -> dict:
        out = {"device": self.dev.device, "kernel_launches": getattr(self, "launches", self.dev.launches),
               "diag_combine": self.combine_diag,
               "support": self.dev.support_info() if hasattr(self.dev, "support_info") else None,
               "gates_applied": self.gates_applied, "fused": self.fuse and self.mode is not PrecisionMode.BYTE,
               "physical_link_bytes": 0}
        if self.mode is PrecisionMode.BYTE:
            out.update(byte_passes=self.dev.passes, byte_reencodes=self.dev.reencodes,
                       byte_host_fixes=self.dev.host_fixes)
        if self.tier is not None:
            out["tier"] = {"executed": self.tier.execute, "groups": len(self.tier.plan.groups),
                           "chunk_qubits": self.tier.plan.chunk_qubits}
            if self.tier.execute:
                out["tier"].update(self.dev.stats())
                out["tier"]["setup_seconds"] = round(getattr(self.tier, "setup_seconds", 0.0), 3)
                out["tier"]["run_seconds"] = round(getattr(self, "run_seconds", 0.0), 3)
        return out
