"""Multi-GPU execution: one process per GPU, NVLink 5 / NVSwitch exchanges.

Launch with torchrun (``python -m torch.distributed.run --nproc-per-node P``)
and call ``run_circuit_distributed`` on every rank.  Rank r owns the 2**N'
amplitudes whose top log2(P) index bits equal r (svsim/layout.py:26-47),
in its own GPU's HBM.

Control plane: ``torch.distributed`` (gloo, CPU) for rendezvous, the CUDA IPC
handle exchange, barriers and the few scalars of a measurement.  Data plane:
libsvb200 kernels on IPC-mapped peer memory —
  * gates whose qubits are local: fused tile passes (same kernels as 1 GPU);
  * a non-diagonal gate on a global qubit: the remap planner (remap.py)
    swaps it with a local qubit first (svk_swap_peer: every amplitude that has
    to move crosses NVLink once, L/2 per direction per rank pair);
  * diagonal gates: no data movement, global bits select the active ranks
    (layout.py:81-82);
  * measure-all: local tiled passes for local qubits, svk_pair_dot over
    NVLink for the cross terms of global qubits (measure.py:83-101), then
    one all-reduce of 3N + 1 scalars.
The reference's ledgers are still charged exactly as svsim would
(layout.plan_exchange per gate, one L/2 message per global qubit at
measurement); the bytes that physically crossed NVLink are reported next to
them.
"""
from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import gates as g
from .circuit import Circuit, validate_circuit
from .device import gate_op, ops_array
from .layout import PartitionLayout, TrafficLedger, plan_exchange
from .measure import ExpectationReport, report_from_sums
from .byte_state import IN_PLACE as BYTE_IN_PLACE, MAX_TAGGED_RANKS
from .remap import Measure, PhysGate, RemapPlanner, Swap, SwapGroup, deposit, group_schedule
from .state import PrecisionMode


def phys_op(gate, phys: tuple, n_local: int, rank: int):
    """sv_op for a gate on physical positions; None if this rank is inactive (diagonal)."""
    if g.is_diagonal(gate):
        mask = 0
        for p in phys:
            if p >= n_local:
                if not (rank >> (p - n_local)) & 1:
                    return None
            else:
                mask |= 1 << p
        f = g.diagonal_factor(gate)
        return gate_op(nat.SV_OP_DIAG, mask=mask, data=(f.real, f.imag))
    m = nat.mat_buffer(g.unitary_matrix(gate))
    if len(phys) == 1:
        return gate_op(nat.SV_OP_1Q, qa=phys[0], data=m)
    return gate_op(nat.SV_OP_2Q, qa=phys[0], qb=phys[1], data=m)


def all_gather_candidates(dist, mine):
    """The per-gate codebook barrier's exchange: every rank's [(magnitudes, phase values)]
    per reference rank, gathered in rank order -- the result of dist.all_gather_object,
    built from two tensor all-gathers (lengths, then one padded float64 buffer per rank)
    instead of pickling on the per-gate path.  Non-gloo groups use all_gather_object."""
    world = dist.get_world_size()
    if dist.get_backend() != "gloo":
        every = [None] * world
        dist.all_gather_object(every, mine)
        return every
    import torch
    R = len(mine)
    parts = [np.asarray([len(m) for m, _ in mine] + [len(p) for _, p in mine], dtype=np.float64)]
    for m, p in mine:
        parts.append(np.ascontiguousarray(m, dtype=np.float64).ravel())
        parts.append(np.ascontiguousarray(p, dtype=np.complex128).ravel().view(np.float64))
    buf = np.concatenate(parts)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([buf.size], dtype=torch.int64))
    L = max(int(t.item()) for t in sizes)
    mine_t = torch.zeros(L, dtype=torch.float64)
    mine_t[:buf.size] = torch.from_numpy(buf)
    outs = [torch.empty(L, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(outs, mine_t)
    every = []
    for t in outs:
        a = t.numpy()
        lm, lp = a[:R].astype(np.int64), a[R:2 * R].astype(np.int64)
        off, lst = 2 * R, []
        for r in range(R):
            m = a[off:off + lm[r]].copy()
            off += int(lm[r])
            ph = a[off:off + 2 * lp[r]].copy().view(np.complex128)
            off += 2 * int(lp[r])
            lst.append((m, ph))
        every.append(lst)
    return every


# SVB200_SUPPORT=0: distributed FP runs process every tile of every pass (no support tracking)
_DIST_SUPPORT = os.environ.get("SVB200_SUPPORT", "1") != "0"


# IPC mappings of the peers' FP slices, kept across runs of the same shape:
# (device, rank, world) -> {"shape": (n_local, mode), "maps": {peer: (handle bytes, ptr)}}.
# A run of the same shape gets the same slab back from the slab cache (sv_slab.cu), hence
# the same handle, and reuses the mapping instead of mapping 2^n_local amplitudes again.
# Every slab this process exported stays allocated (the slab cache never hands an exported
# slab back to the driver, not even on an out-of-memory retry) until every rank has closed
# its mappings: _unmap_everywhere closes them all, holds a barrier and only then releases
# the export marks (sv_ipc_unexport_all).
_PEER_MAPS: dict = {}


def _close_peer_maps(key) -> None:
    ent = _PEER_MAPS.pop(key, None)
    if ent:
        for _, p in ent["maps"].values():
            nat.load().sv_ipc_close(key[0], p)


def _unmap_everywhere(dist) -> None:
    """Collective: close every cached mapping of this process, wait for every rank to do
    the same, then drop the export marks (the slabs may go back to the driver)."""
    for key in list(_PEER_MAPS):
        _close_peer_maps(key)
    dist.barrier()
    nat.check(nat.load().sv_ipc_unexport_all(None))


def release_peer_maps(dist=None) -> None:
    """Close every cached peer mapping of this process.  With `dist` (collective, every
    rank calls it) the export marks are dropped afterwards, so the slab cache may return
    the slabs to the driver; without it the slabs stay pinned in the cache."""
    if dist is None:
        for key in list(_PEER_MAPS):
            _close_peer_maps(key)
        return
    _unmap_everywhere(dist)


def _prepare_peer_maps(dist, device: int, shape) -> dict:
    """Before a rank allocates its slice: keep the cached mappings when the shape matches
    on EVERY rank, else close them all everywhere.  The decision is collective (one
    all-gather of the stale flags): a rank whose cache differs (an earlier constructor
    raised, a partial release, another group of the same size) forces every rank through
    the same close + barrier path instead of leaving one rank in a barrier while the
    others enter the handle all-gather."""
    key = (device, dist.get_rank(), dist.get_world_size())
    stale = any(k != key or e["shape"] != shape for k, e in _PEER_MAPS.items()) or key not in _PEER_MAPS
    flags = [None] * dist.get_world_size()
    dist.all_gather_object(flags, (bool(stale), shape))
    if any(f[0] for f in flags) or any(f[1] != shape for f in flags):
        _unmap_everywhere(dist)
    return _PEER_MAPS.setdefault(key, {"shape": shape, "maps": {}})["maps"]


# inter-process events of the overlapped swaps, created and exchanged once per process
# (events live as long as the process; peers' handles stay valid)
_OVERLAP_EVENTS: dict = {}  # (device, rank, world, chunks) -> (stream, own events, peer events)


class _SupportBook:
    """The global state's support {i : (i & ~sup_free) == sup_val} in physical positions,
    identical on every rank (the same ops move it everywhere); a remap swap exchanges the
    bits of its two positions."""

    def _swap_bits(self, pairs) -> None:
        for a, b in pairs:
            for name in ("sup_free", "sup_val"):
                x = getattr(self, name)
                if ((x >> a) ^ (x >> b)) & 1:
                    x ^= (1 << a) | (1 << b)
                setattr(self, name, x)

    def _slice_empty(self) -> bool:
        """True when a fixed global bit of the support differs from this rank's bit."""
        gmask = ((1 << self.n) - 1) & ~((1 << self.n_local) - 1)
        return bool((self.sup_val ^ (self.rank << self.n_local)) & gmask & ~self.sup_free)

    def _pair_is_zero(self, global_pos: int) -> bool:
        """A fixed global qubit: one amplitude of every pair is zero, the cross sum is 0."""
        return self.track and not (self.sup_free >> global_pos) & 1


class CudaBackend(_SupportBook):
    """This rank's slice in HBM plus IPC-mapped slices of every other rank."""

    def __init__(self, dist, n_local: int, mode: PrecisionMode, device: int, tile_bits: int = 12):
        from .device import DeviceState
        nat.check(nat.load().sv_set_device(device))
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.n_local = n_local
        self.mode = mode
        self.tile_bits = tile_bits
        cached = _prepare_peer_maps(dist, device, (n_local, nat.mode_code(mode)))
        self.dev = DeviceState(n_local, mode, device=device)
        self.dev.zero(0 if self.rank == 0 else None)
        self.bpe = mode.bytes_per_element
        handle = (ctypes.c_char * 64)()
        nat.check(nat.load().sv_ipc_handle(self.dev.handle, handle))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle))
        self.peers = {}
        self.maps_reused = 0
        for r, hb in enumerate(handles):
            if r == self.rank:
                continue
            if r in cached and cached[r][0] == hb:     # same slab as last run: mapping still valid
                self.peers[r] = cached[r][1]
                self.maps_reused += 1
                continue
            if r in cached:
                nat.load().sv_ipc_close(device, cached.pop(r)[1])
            p = ctypes.c_void_p()
            buf = (ctypes.c_char * 64).from_buffer_copy(hb)
            nat.check(nat.load().sv_ipc_open(device, buf, ctypes.byref(p)))
            self.peers[r] = p
            cached[r] = (hb, p)
        self.link_bytes = 0
        self.swap_timing = False
        self.swap_events = []
        self._overlap = None          # chunk events / swap stream, created on first overlapped swap
        self.overlapped = 0
        # support of the global state in physical positions (csrc sv_capi.cu Support): the run
        # starts from |0..0>, every rank moves it through the same non-diagonal ops, so every
        # rank holds the same set.  A rank slice outside it holds zeros (passes, measurement
        # and pair dots skipped); inside it, the handle gets the slice's restriction before
        # each local pass, since remap swaps move bits between local and global positions.
        self.n = n_local + (self.world.bit_length() - 1)
        self.track = _DIST_SUPPORT
        self.sup_free, self.sup_val = 0, 0
        self.skipped_passes = 0
        dist.barrier()

    # -- support tracking ------------------------------------------------------------------
    def _advance(self, ops) -> None:
        if not self.track or not ops:
            return
        f, v = ctypes.c_uint64(self.sup_free), ctypes.c_uint64(self.sup_val)
        nat.check(nat.load(require_device=False).sv_support_advance(ops_array(ops), len(ops), ctypes.byref(f),
                                                                    ctypes.byref(v)))
        self.sup_free, self.sup_val = f.value, v.value

    def _restrict(self) -> bool:
        """Hand this slice's support to the handle; False when the slice can only hold zeros."""
        if not self.track:
            return True
        if self._slice_empty():
            return False
        lm = (1 << self.n_local) - 1
        nat.check(nat.load().sv_set_support(self.dev.handle, self.sup_free & lm, self.sup_val & lm))
        return True

    def _fixed_local(self, pairs) -> int:
        """Local bits the support fixes, outside the swap victims (0: dense swap)."""
        if not self.track:
            return 0
        victims = sum(1 << l for _, l in pairs)
        return ~self.sup_free & ((1 << self.n_local) - 1) & ~victims

    def _swap_restricted(self, pairs) -> bool:
        """A remap swap of a state whose support fixes local bits outside the victims: on
        every rank only the amplitudes whose fixed bits read val can be nonzero, so the swap
        is the chunk form of the group swap over them alone (svk_swap_group_chunk with the
        fixed bits as the chunk).  False when nothing is fixed (the dense kernels run)."""
        cmask = self._fixed_local(pairs)
        if not cmask:
            return False
        L = self.dev.size
        cpat = self.sup_val & cmask
        T = L >> (len(pairs) + bin(cmask).count("1"))     # remaining-bit indices per member pair
        lo = T - T // 2
        sched = group_schedule(self.rank, pairs, self.n_local, L)
        self._sync_all()
        lib = nat.load()
        for member, vmask, own_pat, peer_pat, t0, cnt in sched:
            tb, tc = (0, lo) if t0 == 0 else (lo, T - lo)
            if tc:
                nat.check(lib.svk_swap_group_chunk(self.dev.ptr, self.peers[member], L, self.dev.mode_code, vmask,
                                                   own_pat, peer_pat, cmask, cpat, tb, tc, self.dev.stream))
            self.link_bytes += 2 * tc * self.bpe
        self._sync_all()
        self.dev._touch()
        self._swap_bits(pairs)
        return True

    def apply_local(self, ops):
        if self._restrict():
            self.dev.apply_fused(ops, self.tile_bits)
        else:
            self.skipped_passes += 1
        self._advance(ops)

    # -- remap swap overlapped with the following pass ------------------------------------
    OVERLAP_CHUNK_BITS = int(__import__("os").environ.get("SVB200_OVERLAP_CHUNK_BITS", "4"))   # 16 chunks
    OVERLAP_SWAP_BLOCKS = int(__import__("os").environ.get("SVB200_OVERLAP_BLOCKS", "128"))   # swap grid (4 GPUs: 128 best of 64-1184)
    # measure-all: pair-dot grid (0: one full wave) and the measurement CTA slots left free
    # for it.  Co-resident pair dots + local passes were measured SLOWER than letting the
    # full-grid kernels run back to back (N=33, 2 GPUs: 196 ms vs 206-420 ms for grids of
    # 32-148 / reserves 16-74, profiles/r01_dist_measure_overlap_2gpu.log): the peer's
    # NVLink reads of this HBM starve under the passes' HBM load.  Defaults keep the full grids.
    PAIR_DOT_BLOCKS = int(__import__("os").environ.get("SVB200_PAIR_DOT_BLOCKS", "0"))
    MEASURE_RESERVE = int(__import__("os").environ.get("SVB200_MEASURE_RESERVE", "0"))

    def _overlap_setup(self):
        """Second stream for the swap chunks and one inter-process event per chunk, the
        handles exchanged once per process (cached across runs); peers' events opened for
        cross-GPU ordering."""
        lib = nat.load()
        # events belong to the calling thread's current device (pair_dots calls this from
        # a worker thread): make it this rank's device first
        nat.check(lib.sv_set_device(self.dev.device))
        C = 1 << self.OVERLAP_CHUNK_BITS
        key = (self.dev.device, self.rank, self.world, C)
        if key in _OVERLAP_EVENTS:
            self._overlap = _OVERLAP_EVENTS[key]
            return
        stream = nat.Stream(self.dev.device)
        own, handles = [], bytearray()
        for _ in range(2 * C):       # [0, C): swap chunk done; [C, 2C): pass-before chunk done
            ev = ctypes.c_void_p()
            h = (ctypes.c_char * 64)()
            nat.check(lib.sv_event_create_ipc(ctypes.byref(ev), h))
            own.append(ev)
            handles += bytes(h)
        every = [None] * self.world
        self.dist.all_gather_object(every, bytes(handles))
        peers = {}
        for r, hb in enumerate(every):
            if r == self.rank:
                continue
            evs = []
            for i in range(2 * C):
                ev = ctypes.c_void_p()
                buf = (ctypes.c_char * 64).from_buffer_copy(hb[64 * i:64 * (i + 1)])
                nat.check(lib.sv_event_open_ipc(buf, ctypes.byref(ev)))
                evs.append(ev)
            peers[r] = evs
        self._overlap = (stream, own, peers)
        _OVERLAP_EVENTS[key] = self._overlap

    def _chunk_bits(self, pairs, ops):
        """Chunk positions for an overlapped swap: the highest local positions >= 12 that no
        non-diagonal op of the overlapped pass touches and that are not swap victims (the
        same on every rank: only diagonal ops differ between ranks)."""
        victims = {lp for _, lp in pairs}
        used = set()
        for op in ops:
            if op.kind == nat.SV_OP_1Q:
                used.add(op.qa)
            elif op.kind == nat.SV_OP_2Q:
                used.update((op.qa, op.qb))
        bits = [q for q in range(self.n_local - 1, 11, -1) if q not in used and q not in victims]
        return bits[:self.OVERLAP_CHUNK_BITS] if len(bits) >= self.OVERLAP_CHUNK_BITS else []

    @staticmethod
    def _need(op) -> int:
        if op.kind == nat.SV_OP_1Q:
            return 1 << op.qa
        if op.kind == nat.SV_OP_2Q:
            return (1 << op.qa) | (1 << op.qb)
        return 0             # diagonal ops never need a tile position

    @classmethod
    def _first_pass(cls, ops, K: int = 11):
        """Longest prefix of ops whose NON-DIAGONAL qubits fit one 2^K tile with the five
        lowest qubits (it may still be several passes when it holds more than 128 ops).  Only
        diagonal ops differ between ranks (phys_op), so the qubit set -- and the chunk bits
        derived from it -- is the same on every rank."""
        need = 0x1F
        for i, op in enumerate(ops):
            m = cls._need(op)
            if bin(need | m).count("1") > K:
                return ops[:i], ops[i:]
            need |= m
        return ops, []

    @classmethod
    def _last_pass(cls, ops, K: int = 11):
        """(head, last): the longest suffix of ops whose non-diagonal qubits fit one tile."""
        need = 0x1F
        for i in range(len(ops) - 1, -1, -1):
            m = cls._need(ops[i])
            if bin(need | m).count("1") > K:
                return ops[:i + 1], ops[i + 1:]
            need |= m
        return [], ops

    def swap_then_apply(self, pairs, ops, before=()) -> None:
        """A remap swap (one or k global qubits) with the ops before and after it, the
        transfer overlapping both neighbouring passes: the last pass before the swap, the swap
        (second stream) and the first pass after it run chunk by chunk over 16 chunks (fixed
        values of four high local bits outside both passes' tiles and the victims); each swap
        chunk waits for that chunk of the pass before on this rank and every partner, each
        chunk of the pass after waits for that swap chunk everywhere (inter-process events).
        The control flow (barriers, events) is identical on every rank: the chunk bits come
        from non-diagonal ops only, and empty op ranges still record their events.  Same
        amplitudes, same arithmetic as apply_local + swap + apply_local."""
        before = list(before)
        first, rest = self._first_pass(ops)
        head, last = self._last_pass(before)
        # (a support fixing local bits: the restricted swap moves little, no overlap needed)
        dense = self.mode is PrecisionMode.FP64 and not self._fixed_local(pairs)
        bits = self._chunk_bits(pairs, list(first) + list(last)) if dense else []
        if not bits:
            if before:
                self.apply_local(before)
            if len(pairs) == 1:
                self.swap(*pairs[0])
            else:
                self.swap_group(pairs)
            if ops:
                self.apply_local(ops)
            return
        if self._overlap is None:
            self._overlap = ()
            self._overlap_setup()
        stream, own_ev, peer_ev = self._overlap
        self.overlapped += 1
        lib = nat.load()
        L = self.dev.size
        k = len(pairs)
        sched = group_schedule(self.rank, pairs, self.n_local, L)
        cmask = sum(1 << b for b in bits)
        half = (L >> (k + len(bits))) // 2
        C = 1 << len(bits)
        members = [m for m, *_ in sched]
        if head:
            self.apply_local(head)
        if self.swap_timing:
            e0 = nat.Event()
            e0.record(self.dev.stream)
        arr_l = ops_array(last)
        for i in range(C):           # stage 1: the pass before, chunk by chunk
            if last:
                nat.check(lib.sv_apply_fused_chunk(self.dev.handle, arr_l, len(last), self.tile_bits, cmask,
                                                   deposit(i, bits)))
            nat.check(lib.sv_event_record(own_ev[C + i], self.dev.stream))
        self._advance(last)          # (chunked passes run dense: sv_apply_fused_chunk ends tracking)
        self.dist.barrier()          # every rank's stage-1 events are recorded
        prev_blocks = lib.sv_swap_blocks(self.OVERLAP_SWAP_BLOCKS)
        for i in range(C):           # stage 2: the swap, chunk by chunk on the second stream
            cpat = deposit(i, bits)
            nat.check(lib.sv_stream_wait_event(stream.ptr, own_ev[C + i]))
            for m in members:
                nat.check(lib.sv_stream_wait_event(stream.ptr, peer_ev[m][C + i]))
            for member, vmask, own_pat, peer_pat, t0, cnt in sched:
                nat.check(lib.svk_swap_group_chunk(self.dev.ptr, self.peers[member], L, self.dev.mode_code, vmask,
                                                   own_pat, peer_pat, cmask, cpat, 0 if t0 == 0 else half, half,
                                                   stream.ptr))
                self.link_bytes += 2 * half * self.bpe
            nat.check(lib.sv_event_record(own_ev[i], stream.ptr))
        lib.sv_swap_blocks(prev_blocks)
        self._swap_bits(pairs)
        self.dist.barrier()          # every rank's stage-2 events are recorded
        arr = ops_array(first)
        for i in range(C):           # stage 3: the pass after, chunk by chunk
            nat.check(lib.sv_stream_wait_event(self.dev.stream, own_ev[i]))
            for m in members:
                nat.check(lib.sv_stream_wait_event(self.dev.stream, peer_ev[m][i]))
            if first:
                nat.check(lib.sv_apply_fused_chunk(self.dev.handle, arr, len(first), self.tile_bits, cmask,
                                                   deposit(i, bits)))
        self._advance(first)
        if self.swap_timing:
            e1 = nat.Event()
            e1.record(self.dev.stream)
            self.swap_events.append((e0, e1))
        self.dev._touch()
        if rest:
            self.apply_local(rest)

    def _sync_all(self):
        self.dev.synchronize()
        self.dist.barrier()

    def swap(self, global_pos: int, local_pos: int):
        if self._swap_restricted(((global_pos, local_pos),)):
            return
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        side = (self.rank >> bit) & 1
        self._sync_all()
        if self.swap_timing:
            e0, e1 = nat.Event(), nat.Event()
            e0.record(self.dev.stream)
        nat.check(nat.load().svk_swap_peer(self.dev.ptr, self.peers[partner], self.dev.size, self.dev.mode_code,
                                           local_pos, side, self.dev.stream))
        if self.swap_timing:
            e1.record(self.dev.stream)
            self.swap_events.append((e0, e1))
        self._sync_all()
        self.dev._touch()
        self._swap_bits(((global_pos, local_pos),))
        self.link_bytes += 2 * (self.dev.size // 4) * self.bpe      # this rank's reads + writes over NVLink

    def swap_group(self, pairs) -> None:
        """Batched swap of k global qubits (remap.SwapGroup): one svk_swap_group launch
        per other member of this rank's 2^k group, all ranks concurrently (every
        launch touches a disjoint set of amplitudes)."""
        if self._swap_restricted(pairs):
            return
        sched = group_schedule(self.rank, pairs, self.n_local, self.dev.size)
        self._sync_all()
        if self.swap_timing:
            e0, e1 = nat.Event(), nat.Event()
            e0.record(self.dev.stream)
        lib = nat.load()
        for member, vmask, own_pat, peer_pat, t0, cnt in sched:
            nat.check(lib.svk_swap_group(self.dev.ptr, self.peers[member], self.dev.size, self.dev.mode_code, vmask,
                                         own_pat, peer_pat, t0, cnt, self.dev.stream))
            self.link_bytes += 2 * cnt * self.bpe
        if self.swap_timing:
            e1.record(self.dev.stream)
            self.swap_events.append((e0, e1))
        self._sync_all()
        self.dev._touch()
        self._swap_bits(pairs)

    def pair_gate(self, global_pos: int, matrix) -> None:
        """The reference's pairwise round for a single-qubit gate on a global qubit
        (engine.py:246-269), fused with the exchange: the low rank updates offsets
        [0, L/2) of both slices, the high rank [L/2, L), reading and writing the
        partner's HBM directly (svk_pair_update with a peer pointer)."""
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        low = ((self.rank >> bit) & 1) == 0
        half = self.dev.size // 2
        esz = np.dtype(self.dev.dtype).itemsize
        off = 0 if low else half
        own = ctypes.c_void_p(self.dev.ptr.value + off * esz)
        peer = ctypes.c_void_p(self.peers[partner].value + off * esz)
        a0, a1 = (own, peer) if low else (peer, own)
        m = nat.mat_buffer(matrix)
        self._sync_all()
        nat.check(nat.load().svk_pair_update(a0, a1, half, self.dev.mode_code, nat.dptr(m), self.dev.stream))
        self._sync_all()
        self.dev._touch()
        self.link_bytes += 2 * half * self.bpe
        self._advance([gate_op(nat.SV_OP_1Q, qa=global_pos, data=m)])

    def measure_local(self):
        if not self._restrict():      # zeros: sums of zeros
            n = self.n_local
            return 0.0, np.zeros(n), np.zeros(n, dtype=np.complex128)
        return self.dev.measure()

    def _pair_dot_restricted(self, global_pos: int, stream, max_blocks: int):
        """The cross sum of a free global qubit when the support fixes local bits: only the
        amplitudes whose fixed bits read val enter (svk_pair_dot_chunk over the whole slices,
        the rest indices split between the two ranks); None when nothing is fixed."""
        cmask = self._fixed_local(())
        if not cmask:
            return None
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        low = ((self.rank >> bit) & 1) == 0
        a0, a1 = (self.dev.ptr, self.peers[partner]) if low else (self.peers[partner], self.dev.ptr)
        L = self.dev.size
        T = L >> bin(cmask).count("1")
        lo = T - T // 2
        tb, tc = (0, lo) if low else (lo, T - lo)
        res = np.zeros(2)
        nat.check(nat.load().svk_pair_dot_chunk(a0, a1, L, self.dev.mode_code, cmask, self.sup_val & cmask, tb, tc,
                                                max_blocks, nat.dptr(res), stream))
        self.link_bytes += tc * self.bpe
        return complex(res[0], res[1])

    def pair_dot(self, global_pos: int) -> complex:
        """This rank's share of sum conj(a0) a1 for a global qubit (measure.py:92-99)."""
        if self._pair_is_zero(global_pos):
            return 0j
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        low = ((self.rank >> bit) & 1) == 0
        half = self.dev.size // 2
        esz = np.dtype(self.dev.dtype).itemsize
        self._sync_all()
        r = self._pair_dot_restricted(global_pos, self.dev.stream, 0)
        if r is not None:
            return r
        out = np.zeros(2)
        if low:
            a0, a1 = self.dev.ptr, self.peers[partner]
            off = 0
        else:
            a0, a1 = self.peers[partner], self.dev.ptr
            off = half
        p0 = ctypes.c_void_p(a0.value + off * esz)
        p1 = ctypes.c_void_p(a1.value + off * esz)
        nat.check(nat.load().svk_pair_dot(p0, p1, half, self.dev.mode_code, 0, nat.dptr(out), self.dev.stream))
        self.link_bytes += half * self.bpe
        return complex(out[0], out[1])

    def pair_dots(self, positions):
        """pair_dot of several global qubits on the second stream with no host barrier in
        between (the caller synchronised all ranks): runs on a worker thread while the local
        measurement passes stream HBM on the main stream -- NVLink-bound next to HBM-bound."""
        if self._overlap is None:
            self._overlap = ()
            self._overlap_setup()
        stream = self._overlap[0]
        lib = nat.load()
        nat.check(lib.sv_set_device(self.dev.device))
        half = self.dev.size // 2
        esz = np.dtype(self.dev.dtype).itemsize
        out = {}
        for global_pos in positions:
            if self._pair_is_zero(global_pos):
                out[global_pos] = 0j
                continue
            r = self._pair_dot_restricted(global_pos, stream.ptr, self.PAIR_DOT_BLOCKS)
            if r is not None:
                out[global_pos] = r
                continue
            bit = global_pos - self.n_local
            partner = self.rank ^ (1 << bit)
            low = ((self.rank >> bit) & 1) == 0
            a0, a1 = (self.dev.ptr, self.peers[partner]) if low else (self.peers[partner], self.dev.ptr)
            off = 0 if low else half
            res = np.zeros(2)
            nat.check(lib.svk_pair_dot(ctypes.c_void_p(a0.value + off * esz),
                                       ctypes.c_void_p(a1.value + off * esz), half, self.dev.mode_code,
                                       self.PAIR_DOT_BLOCKS, nat.dptr(res), stream.ptr))
            self.link_bytes += half * self.bpe
            out[global_pos] = complex(res[0], res[1])
        return out

    def export(self) -> np.ndarray:
        return self.dev.export()

    def close(self):
        """End of the run: every rank is done with the peers' slices.  The mappings stay
        cached for the next run of this shape (release_peer_maps closes them)."""
        self.dev.synchronize()
        self.dist.barrier()
        self.peers = {}


class CudaByteBackend(_SupportBook):
    """BYTE slice (two uint8 planes, double-buffered) + IPC-mapped peer planes.

    Every gate runs the reference's per-gate codebook barrier across ranks: each rank
    encodes its work items speculatively (or scans first after a table grew), tags every
    produced value with its REFERENCE producer rank (computed from the logical index,
    so remapping does not change who proposes what), the raw candidates of all ranks
    are all-gathered, and every rank merges the same proposals in rank order
    (codec.py:154-191) -> identical tables everywhere."""

    def __init__(self, dist, n_local: int, layout, device: int):
        from .byte_state import ByteDeviceState
        from .codec import Codebook
        nat.check(nat.load().sv_set_device(device))
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.n_local = n_local
        self.layout = layout
        self.mode = PrecisionMode.BYTE
        _prepare_peer_maps(dist, device, ("byte", n_local))   # drop the FP mappings first
        self.st = ByteDeviceState(n_local, Codebook(), device)
        self.st.zero(0 if self.rank == 0 else None)
        self.dev = self.st
        handles = (ctypes.c_char * 256)()
        nat.check(nat.load().svb_ipc_handles(self.st.handle, handles))
        every = [None] * self.world
        dist.all_gather_object(every, bytes(handles))
        self.peers = {}
        for r, hb in enumerate(every):
            if r == self.rank:
                continue
            planes = [[None, None], [None, None]]
            for b in range(2):
                for pl in range(2):
                    ptr = ctypes.c_void_p()
                    buf = (ctypes.c_char * 64).from_buffer_copy(hb[64 * (2 * b + pl):64 * (2 * b + pl + 1)])
                    nat.check(nat.load().sv_ipc_open(device, buf, ctypes.byref(ptr)))
                    planes[b][pl] = ptr
            self.peers[r] = planes
        self.link_bytes = 0
        self.passes = 0
        self.scan_first = False
        self.host_fixes = 0
        # support tracking (_SupportBook), monotone as in ByteEngineState: every non-diagonal
        # gate frees its qubits, so both plane buffers hold zeros outside the support -- after
        # a remap swap moved the current planes, the pending ones are cleared to keep that
        self.n = n_local + (self.world.bit_length() - 1)
        self.track = _DIST_SUPPORT
        self.sup_free, self.sup_val = 0, 0
        dist.barrier()

    def _tracked(self) -> bool:
        """Tracking, and the support still fixes some bit (else every pass is dense)."""
        return self.track and self.sup_free != (1 << self.n) - 1

    def _after_swap(self, pairs) -> None:
        if not self.track:
            return
        tracked = self._tracked()
        self._swap_bits(pairs)
        if tracked:
            nat.check(nat.load().svb_clear_pending(self.st.handle))

    def _sync_all(self):
        self.st.synchronize()
        self.dist.barrier()

    def _peer_cur(self, r):
        c = nat.load().svb_cur(self.st.handle)
        return self.peers[r][c]

    def swap(self, global_pos: int, local_pos: int):
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        side = (self.rank >> bit) & 1
        pm, pp = self._peer_cur(partner)
        self._sync_all()
        nat.check(nat.load().svb_swap_peer(self.st.handle, pm, pp, local_pos, side))
        self._sync_all()
        self.st.version += 1
        self._after_swap(((global_pos, local_pos),))
        self.link_bytes += 2 * (self.st.size // 4) * 2

    def swap_group(self, pairs) -> None:
        sched = group_schedule(self.rank, pairs, self.n_local, self.st.size)
        self._sync_all()
        lib = nat.load()
        for member, vmask, own_pat, peer_pat, t0, cnt in sched:
            pm, pp = self._peer_cur(member)
            nat.check(lib.svb_swap_group(self.st.handle, pm, pp, vmask, own_pat, peer_pat, t0, cnt))
            self.link_bytes += 2 * cnt * 2
        self._sync_all()
        self.st.version += 1
        self._after_swap(pairs)

    def _desc(self, gate, phys, pos):
        from .byte_state import SvbGateDesc, _exchange_fields, set_logical_bits
        d = SvbGateDesc()
        n_local = self.n_local
        if g.is_diagonal(gate):
            d.kind = nat.SV_OP_DIAG
            mask = 0
            active = True
            for p in phys:
                if p >= n_local:
                    active = active and bool((self.rank >> (p - n_local)) & 1)
                else:
                    mask |= 1 << p
            d.diag_mask = mask if active else (1 << n_local)     # inactive rank: copy everything
            f = g.diagonal_factor(gate)
            d.m[0], d.m[1] = f.real, f.imag
        else:
            m = nat.mat_buffer(g.unitary_matrix(gate))
            for i, v in enumerate(m):
                d.m[i] = v
            d.kind = nat.SV_OP_1Q if len(phys) == 1 else nat.SV_OP_2Q
            d.qa = phys[0]
            d.qb = phys[1] if len(phys) == 2 else 0
        plan = plan_exchange(self.layout, gate, PrecisionMode.BYTE)
        _exchange_fields(d, gate, self.layout, plan)
        set_logical_bits(d, self.layout, pos, self.rank << n_local)
        d.mag_cut = d.ph_cut = 1e308
        if self._tracked():   # the passes visit only the slice's support items (an empty slice: one)
            lm = (1 << n_local) - 1
            if self._slice_empty():
                d.sup_fixed, d.sup_val = lm, 0
            else:
                d.sup_fixed = ~self.sup_free & lm
                d.sup_val = self.sup_val & d.sup_fixed
        return d

    def _pass(self, d, producer, collect, scan, in_place=False):
        d.producer = producer
        d.collect = 1 if collect else 0
        d.scan_only = 1 if scan else 0
        self.st.reset()
        self.st.gate_pass(d, in_place)
        self.passes += 1
        mags, ph, flags = self.st.read_candidates() if collect else (None, None, 0)
        if flags & 1:
            raise RuntimeError("codebook candidate buffer overflow (multi-GPU BYTE)")
        unsure = self.st.read_unsure()
        return mags, ph, unsure

    def apply_gate(self, gate, phys, pos):
        cb = self.st.codebook
        self.st.sync_tables()
        sat_mag, sat_ph = cb.tables_saturated
        d = self._desc(gate, phys, pos)
        d.want_mag = 0 if sat_mag else 1
        d.want_ph = 0 if sat_ph else 1
        # as ByteEngineState.apply_gate: a diagonal gate's final write pass runs in place
        # (the same decision on every rank: it depends on the gate and the shared codebook)
        in_place = BYTE_IN_PLACE and d.kind == nat.SV_OP_DIAG
        final_in_place = False
        if sat_mag and sat_ph:
            _, _, (ui, uv) = self._pass(d, -1, False, False, in_place)
            final_in_place = in_place
        else:
            scan = self.scan_first or in_place   # diagonal: scan, then write in place
            mine = []
            unsure = []
            ranks = self.layout.rank_count
            tagged = None
            if 1 < ranks <= MAX_TAGGED_RANKS:
                d.scan_only = 1 if scan else 0
                tagged = self.st.collect_tagged(d, ranks)      # one pass, candidates tagged by rank
                self.passes += 1
            if tagged is not None:
                mine, u = tagged
                unsure.append(u)
            else:
                for r in range(ranks):
                    mags, ph, u = self._pass(d, r, True, scan)
                    mine.append((mags, ph))
                    unsure.append(u)
            every = all_gather_candidates(self.dist, mine)
            proposals = []
            for r in range(self.layout.rank_count):
                mags = np.concatenate([every[k][r][0] for k in range(self.world)])
                ph = np.concatenate([every[k][r][1] for k in range(self.world)])
                proposals.append(cb.finalize_proposal(mags, ph))
            version = cb.version
            cb.merge(proposals)
            grew = cb.version != version
            self.scan_first = grew
            if scan or grew:
                self.st.sync_tables()
                _, _, (ui, uv) = self._pass(d, -1, False, False, in_place)
                final_in_place = in_place
            else:
                ui = np.concatenate([u[0] for u in unsure])
                uv = np.concatenate([u[1] for u in unsure])
        self.host_fixes += self.st.finish_gate(ui, uv, final_in_place)
        if self.track and not g.is_diagonal(gate):
            for p in phys:
                self.sup_free |= 1 << p

    def measure_local(self):
        if self._tracked():
            if self._slice_empty():
                n = self.n_local
                return 0.0, np.zeros(n), np.zeros(n, dtype=np.complex128)
            lm = (1 << self.n_local) - 1
            self.st.sup_free, self.st.sup_val = self.sup_free & lm, self.sup_val & lm   # svb_measure_support
        try:
            return self.st.measure_sums()
        finally:
            self.st.sup_free = (1 << self.n_local) - 1

    def pair_dot(self, global_pos: int) -> complex:
        if self._pair_is_zero(global_pos):
            return 0j
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        low = ((self.rank >> bit) & 1) == 0
        half = self.st.size // 2
        om, op = ctypes.c_void_p(), ctypes.c_void_p()
        nat.check(nat.load().svb_planes(self.st.handle, ctypes.byref(om), ctypes.byref(op)))
        pm, pp = self._peer_cur(partner)
        self._sync_all()
        off = 0 if low else half
        sh = lambda p: ctypes.c_void_p(p.value + off)  # noqa: E731
        a, b = ((om, op), (pm, pp)) if low else ((pm, pp), (om, op))
        out = np.zeros(2)
        nat.check(nat.load().svb_pair_dot(self.st.handle, sh(a[0]), sh(a[1]), sh(b[0]), sh(b[1]), half,
                                          nat.dptr(out)))
        self.link_bytes += half * 2
        return complex(out[0], out[1])

    def export(self) -> np.ndarray:
        return self.st.decode()

    def close(self):
        """End of the run: unmap the peers' planes on every rank, then (after a barrier)
        drop the export marks so the slab cache may free them again."""
        self.st.synchronize()
        self.dist.barrier()
        for planes in self.peers.values():
            for b in range(2):
                for pl in range(2):
                    nat.load().sv_ipc_close(self.st.device, planes[b][pl])
        self.peers = {}
        _unmap_everywhere(self.dist)


@dataclass
class DistRunResult:
    circuit: Circuit
    layout: PartitionLayout
    mode: PrecisionMode
    rank: int
    ledgers: list
    report: ExpectationReport | None
    perm: tuple                       # logical qubit -> physical position at the end
    wall_time_seconds: float
    device_stats: dict = field(default_factory=dict)
    backend: object = None

    def local_slice(self) -> np.ndarray:
        """This rank's slice in PHYSICAL order (after remapping)."""
        return self.backend.export()

    def gathered_bytes(self, dist):
        """BYTE mode: logical-order (mag_idx, phase_idx) planes on rank 0 (collective)."""
        st = self.backend.st
        mine = st.export_storage(0, st.size)
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, mine)
        if self.rank != 0:
            return None
        src = self._logical_source(sum(p[0].size for p in parts))
        mi = np.concatenate([p[0] for p in parts])[src]
        pi = np.concatenate([p[1] for p in parts])[src]
        return mi, pi

    def _logical_source(self, size):
        idx = np.arange(size)
        src = np.zeros_like(idx)
        for q, p in enumerate(self.perm):
            src |= ((idx >> q) & 1) << p
        return src

    def gathered_state(self, dist) -> np.ndarray | None:
        """Logical-order global state on rank 0 (collective; small N only)."""
        mine = self.local_slice().astype(np.complex128)
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, mine)
        if self.rank != 0:
            return None
        phys = np.concatenate(parts)
        idx = np.arange(phys.size)
        src = np.zeros_like(idx)
        for q, p in enumerate(self.perm):
            src |= ((idx >> q) & 1) << p
        return phys[src]


def _charge_reference(layout, ledgers, gate, mode):
    """The reference ledger entries of one gate (transport.py:30-35 via engine.py)."""
    plan = plan_exchange(layout, gate, mode)
    L = layout.local_size
    P = layout.rank_count
    if plan.kind == "pairwise":
        for r in range(P):
            ledgers[r].count_send(plan.bytes_per_rank)
            ledgers[r ^ plan.masks[0]].count_receive(plan.bytes_per_rank)
    elif plan.kind == "quad":
        ma, mb = plan.masks
        for r in range(P):
            base = r & ~(ma | mb)
            for pos in range(4):
                dst = base | (ma if pos & 1 else 0) | (mb if pos & 2 else 0)
                if dst != r:
                    ledgers[r].count_send((L // 4) * plan.bytes_per_element)
                    ledgers[dst].count_receive((L // 4) * plan.bytes_per_element)


def run_circuit_distributed(circuit: Circuit, dist, *, mode: PrecisionMode = PrecisionMode.FP64,
                            remap: bool = True, device: int | None = None, backend_factory=None,
                            tile_bits: int = 12, fuse_limit: int = 1024, overlap: bool = True) -> DistRunResult:
    """Run `circuit` with one rank per process of the torch.distributed group `dist`."""
    validate_circuit(circuit)
    P = dist.get_world_size()
    rank = dist.get_rank()
    if P & (P - 1):
        raise ValueError("rank count must be a power of two")
    n = circuit.n_qubits
    n_local = n - (P.bit_length() - 1)
    layout = PartitionLayout(n, n_local)
    if not remap and mode is PrecisionMode.BYTE:
        raise NotImplementedError("BYTE runs use the remap planner (remap=True)")
    start = time.perf_counter()
    dev_id = rank if device is None else device
    if backend_factory is not None:
        be = backend_factory(dist, n_local, mode)
    elif mode is PrecisionMode.BYTE:
        be = CudaByteBackend(dist, n_local, layout, dev_id)
        if os.environ.get("SVB200_TIME_BYTE_PASSES"):   # probes: CUDA events around every pass
            be.st.time_passes, be.st.pass_events = True, []
    else:
        be = CudaBackend(dist, n_local, mode, dev_id, tile_bits)
    byte = mode is PrecisionMode.BYTE and backend_factory is None
    ledgers = [TrafficLedger() for _ in range(P)]
    planner = RemapPlanner(n, n_local, remap=remap)
    steps = planner.plan(circuit.gates)
    pending = []
    report = None
    swaps = groups = 0
    pending_swap = None          # FP backends: a swap waits for the ops after it (overlapped)
    pending_before = []          # ... and keeps the ops before it (the last pass overlaps too)
    overlap = overlap and not byte and hasattr(be, "swap_then_apply")

    def flush():
        nonlocal pending, pending_swap, pending_before
        if pending_swap is not None:
            be.swap_then_apply(pending_swap, pending, before=pending_before)
            pending_swap, pending_before = None, []
        elif pending:
            be.apply_local(pending)
        pending = []

    for step in steps:
        if isinstance(step, (Swap, SwapGroup)):
            pairs = ((step.global_pos, step.local_pos),) if isinstance(step, Swap) else step.pairs
            if overlap:
                if pending_swap is not None:     # two swaps back to back: run the first
                    flush()
                pending_before, pending = pending, []
                pending_swap = pairs
            else:
                flush()
                if isinstance(step, Swap):
                    be.swap(step.global_pos, step.local_pos)
                else:
                    be.swap_group(step.pairs)
            swaps += 1
            groups += isinstance(step, SwapGroup)
        elif isinstance(step, PhysGate):
            _charge_reference(layout, ledgers, step.gate, mode)
            if byte:
                be.apply_gate(step.gate, step.qubits, tuple(planner_pos_at(steps, step)))
            elif not remap and not g.is_diagonal(step.gate) and any(p >= n_local for p in step.qubits):
                flush()
                _reference_exchange(be, step, n_local, rank)
            else:
                op = phys_op(step.gate, step.qubits, n_local, rank)
                if op is not None:
                    pending.append(op)
                    if len(pending) >= fuse_limit:
                        flush()
            for led in ledgers:
                led.gate_operations += 1
        elif isinstance(step, Measure):
            flush()
            report = _measure(be, layout, ledgers, step.perm, rank, mode, dist)
            for led in ledgers:
                led.gate_operations += 1
    flush()
    stats = {"swaps": swaps, "swap_groups": groups, "physical_link_bytes": be.link_bytes,
             "planner": "remap" if remap else "reference",
             "overlapped_swaps": getattr(be, "overlapped", 0)}
    if byte:
        stats.update(byte_passes=be.passes, byte_host_fixes=be.host_fixes)
    elif hasattr(be, "skipped_passes"):
        stats.update(support_free_qubits=bin(be.sup_free).count("1") if be.track else None,
                     passes_skipped_empty_slice=be.skipped_passes)
    res = DistRunResult(circuit, layout, mode, rank, ledgers, report, tuple(planner.pos),
                        time.perf_counter() - start, stats, be)
    if byte:
        res.codebook = be.st.codebook
    return res


def _reference_exchange(be, step, n_local, rank):
    """remap=False: the reference's exchange per global gate.  Single-qubit gates use
    the exchange-fused pair update; two-qubit gates borrow local qubits for the
    duration of the gate (swap in, apply, swap back)."""
    gate, phys = step.gate, step.qubits
    if len(phys) == 1:
        be.pair_gate(phys[0], g.unitary_matrix(gate))
        return
    busy = set(phys)
    temps, moved = [], list(phys)
    for i, p in enumerate(phys):
        if p >= n_local:
            lp = next(q for q in range(n_local - 1, -1, -1) if q not in busy)
            busy.add(lp)
            be.swap(p, lp)
            temps.append((p, lp))
            moved[i] = lp
    op = phys_op(gate, tuple(moved), n_local, rank)
    if op is not None:
        be.apply_local([op])
    for p, lp in reversed(temps):
        be.swap(p, lp)


def planner_pos_at(steps, step):
    """Logical -> physical permutation in force when `step` runs."""
    return step.perm


def _measure(be, layout, ledgers, perm, rank, mode, dist):
    import torch
    n, n_local = layout.total_qubits, layout.local_qubits
    half_bytes = (layout.local_size // 2) * mode.bytes_per_element
    for q in range(n_local, n):        # reference accounting: one L/2 message per global qubit
        m = 1 << (q - n_local)
        for r in range(layout.rank_count):
            ledgers[r].count_send(half_bytes)
            ledgers[r ^ m].count_receive(half_bytes)
    remote = {}
    if hasattr(be, "pair_dots") and n > n_local:
        # global-qubit cross sums (NVLink) concurrently with the local passes (HBM)
        import threading
        be._sync_all()
        box = {}

        def work():
            try:
                box["v"] = be.pair_dots(range(n_local, n))
            except BaseException as exc:   # re-raised on the calling thread
                box["e"] = exc
        th = threading.Thread(target=work)
        reserve = getattr(be, "MEASURE_RESERVE", 0)
        prev = nat.load().sv_measure_reserve(reserve) if reserve else None
        try:
            th.start()
            norm, ones_l, cross_l = be.measure_local()
        finally:
            th.join()
            if prev is not None:
                nat.load().sv_measure_reserve(prev)
        if "e" in box:
            raise box["e"]
        remote = box["v"]
    else:
        norm, ones_l, cross_l = be.measure_local()
    ones_p = np.zeros(n)
    cross_p = np.zeros(n, dtype=np.complex128)
    ones_p[:n_local] = ones_l
    cross_p[:n_local] = cross_l
    for p in range(n_local, n):
        cross_p[p] = remote[p] if p in remote else be.pair_dot(p)
        ones_p[p] = norm if (rank >> (p - n_local)) & 1 else 0.0
    vec = torch.tensor(np.concatenate([[norm], ones_p, cross_p.real, cross_p.imag]), dtype=torch.float64)
    dist.all_reduce(vec)
    v = vec.numpy()
    norm_t, ones_t = float(v[0]), v[1:1 + n]
    cross_t = v[1 + n:1 + 2 * n] + 1j * v[1 + 2 * n:1 + 3 * n]
    ones = [ones_t[perm[q]] for q in range(n)]
    cross = [cross_t[perm[q]] for q in range(n)]
    return report_from_sums(norm_t, ones, cross)
