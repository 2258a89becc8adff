"""HBM-resident BYTE (two-plane uint8) state and the per-gate codebook barrier.

``ByteDeviceState`` wraps an ``sv_bhandle`` (include/svb200.h): current and
pending (magnitude, phase) index planes, the device codebook tables and the
candidate buffers.  ``ByteEngineState`` adds the reference's per-gate
protocol (engine.py:186-225, 365-377):

  1. one device pass per reference rank (its "produced" values, as the
     reference's exchange choreography assigns them) decodes, applies the
     gate, encodes against the current tables into the pending planes and
     reduces that rank's not-yet-representable values to candidates;
  2. the host turns every rank's candidates into its proposal and merges
     them (codec.py:137-191) — identical tables on every rank by construction;
  3. if a table grew, one more pass re-encodes from the untouched current
     planes with the new tables;
  4. atan2-ambiguous amplitudes are re-encoded with numpy and patched in;
  5. pending planes become current.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as nat
from . import gates as g
from .codec import CAPACITY, Codebook

_BIG = 1e308
# SVB200_BYTE_PHASE_SKIP=0: always read and write the phase plane
PHASE_PLANE_SKIP = os.environ.get("SVB200_BYTE_PHASE_SKIP", "1") != "0"
_CAP = 1 << 22                # = CAP_UNSURE of sv_byte_api.cu (uncertain-phase list)
_CCAP = 1 << 20               # = CAP_MAG / CAP_PH (candidate buffers)
MAX_TAGGED_RANKS = 8          # candidate set regions per CTA (sv_byte.cu CtaSets)
# diagonal write passes with fixed tables run in place (SVB200_BYTE_IN_PLACE=0: off)
IN_PLACE = os.environ.get("SVB200_BYTE_IN_PLACE", "1") != "0"


class SvbGateDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("qa", ctypes.c_int32), ("qb", ctypes.c_int32),
                ("n_local", ctypes.c_int32), ("diag_mask", ctypes.c_uint64), ("m", ctypes.c_double * 32),
                ("xkind", ctypes.c_int32), ("qlow_top", ctypes.c_int32),
                ("xmask_a", ctypes.c_uint64), ("xmask_b", ctypes.c_uint64),
                ("producer", ctypes.c_int32), ("collect", ctypes.c_int32),
                ("want_mag", ctypes.c_int32), ("want_ph", ctypes.c_int32),
                ("mag_cut", ctypes.c_double), ("ph_cut", ctypes.c_double),
                ("scan_only", ctypes.c_int32), ("rank_bits", ctypes.c_int32),
                ("phys_base", ctypes.c_uint64), ("lbit", ctypes.c_int8 * 16),
                ("ph_zero_in", ctypes.c_int32), ("ph_zero_out", ctypes.c_int32),
                ("sup_fixed", ctypes.c_uint64), ("sup_val", ctypes.c_uint64)]


class ByteDeviceState:
    """2**n amplitudes as (magnitude index, phase index) byte planes in HBM."""

    mode_code = nat.SV_BYTE

    track_support = False      # only the engine's whole-register state maintains a support

    def __init__(self, n_qubits: int, codebook: Codebook | None = None, device: int = 0):
        lib = nat.load()
        self.n_qubits = int(n_qubits)
        self.device = device
        h = ctypes.c_void_p()
        nat.check(lib.svb_create(device, self.n_qubits, ctypes.byref(h)))
        self.handle = h
        s = ctypes.c_void_p()
        nat.check(lib.svb_info(h, None, None, ctypes.byref(s)))
        self.stream = s
        self.codebook = codebook if codebook is not None else Codebook()
        self._tables_version = None
        self.version = 0
        self.launches = 0
        # every phase index of both plane buffers is 0 (the phase table has held one entry
        # whenever a pass wrote them): passes then neither read nor write the phase plane
        self.ph_zero = False

    @property
    def size(self) -> int:
        return 1 << self.n_qubits

    def sync_tables(self) -> None:
        cb = self.codebook
        key = (cb.version, len(cb.mags), len(cb.thetas))
        if key == self._tables_version:
            return
        mags = np.ascontiguousarray(cb.mags, dtype=np.float64)
        th = np.ascontiguousarray(cb.thetas, dtype=np.float64)
        ux = np.ascontiguousarray(cb.ux, dtype=np.float64)
        uy = np.ascontiguousarray(cb.uy, dtype=np.float64)
        nat.check(nat.load().svb_set_tables(self.handle, nat.dptr(mags), len(mags), nat.dptr(th), nat.dptr(ux),
                                            nat.dptr(uy), len(th)))
        self._tables_version = key

    def zero(self, unit_index: int | None = 0) -> None:
        nat.check(nat.load().svb_zero_state(self.handle, -1 if unit_index is None else unit_index))
        self.version += 1
        self.ph_zero = PHASE_PLANE_SKIP and len(self.codebook.thetas) == 1
        # support of a basis state: every other bit fixed (all zeros, or a state whose passes do
        # not maintain it -- the distributed slices, whose remap swaps move data between ranks --
        # is dense)
        tracked = unit_index is not None and self.track_support
        self.sup_free = 0 if tracked else (1 << self.n_qubits) - 1
        self.sup_val = unit_index or 0

    def export_storage(self, first: int, count: int):
        mi = np.empty(count, dtype=np.uint8)
        pi = np.empty(count, dtype=np.uint8)
        nat.check(nat.load().svb_export(self.handle, mi.ctypes.data_as(ctypes.c_void_p),
                                        pi.ctypes.data_as(ctypes.c_void_p), first, count))
        return mi, pi

    def import_storage(self, parts, first: int = 0) -> None:
        mi = np.ascontiguousarray(parts[0], dtype=np.uint8)
        pi = np.ascontiguousarray(parts[1], dtype=np.uint8)
        nat.check(nat.load().svb_import(self.handle, mi.ctypes.data_as(ctypes.c_void_p),
                                        pi.ctypes.data_as(ctypes.c_void_p), first, mi.size))
        self.version += 1
        self.ph_zero = False
        self.sup_free = (1 << self.n_qubits) - 1   # arbitrary bytes: dense

    def decode(self, first: int = 0, count: int | None = None) -> np.ndarray:
        self.sync_tables()
        count = self.size - first if count is None else count
        out = np.empty(count, dtype=np.complex128)
        nat.check(nat.load().svb_decode(self.handle, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        first, count))
        self.launches += 1
        return out

    def decode_all(self, codebook=None) -> np.ndarray:
        return self.decode()

    def measure_sums(self, codebook=None):
        self.sync_tables()
        n = self.n_qubits
        norm = np.zeros(1)
        ones = np.zeros(max(n, 1))
        cross = np.zeros(2 * max(n, 1))
        full = (1 << self.n_qubits) - 1
        free = getattr(self, "sup_free", full)
        if free != full:   # tracked support: only its tiles are read
            fixed = full & ~free
            nat.check(nat.load().svb_measure_support(self.handle, fixed, getattr(self, "sup_val", 0) & fixed,
                                                     nat.dptr(norm), nat.dptr(ones), nat.dptr(cross)))
        else:
            nat.check(nat.load().svb_measure(self.handle, nat.dptr(norm), nat.dptr(ones), nat.dptr(cross)))
        self.launches += 2
        return float(norm[0]), ones[:n].copy(), cross[0:2 * n:2] + 1j * cross[1:2 * n:2]

    def measure_range(self, first: int, count: int):
        vals = self.decode(first, count)
        from .kernels import norm_squared
        return norm_squared(vals), None, None

    def synchronize(self) -> None:
        nat.check(nat.load().sv_stream_synchronize(self.stream))

    # -- candidate plumbing -----------------------------------------------------------
    def _host_buffers(self):
        """Candidate / uncertain-list landing buffers, allocated once per state (136 MB of
        host memory; a fresh np.empty of them per gate was an mmap + munmap per call)."""
        b = getattr(self, "_hbuf", None)
        if b is None:
            b = self._hbuf = (np.empty(_CCAP, dtype=np.float64), np.empty((_CCAP, 4), dtype=np.float64),
                              np.empty(_CAP, dtype=np.uint64), np.empty(2 * _CAP, dtype=np.float64))
        return b

    def read_candidates(self):
        lib = nat.load()
        mags, ph = self._host_buffers()[:2]
        nm, npp = ctypes.c_uint64(0), ctypes.c_uint64(0)
        flags = ctypes.c_int(0)
        nat.check(lib.svb_candidates(self.handle, nat.dptr(mags), _CCAP, ctypes.byref(nm),
                                     ph.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _CCAP, ctypes.byref(npp),
                                     ctypes.byref(flags)))
        ph = ph[:npp.value]
        return mags[:nm.value].copy(), (ph[:, 0] + 1j * ph[:, 1]), flags.value

    def read_candidate_tags(self, n_mag: int, n_ph: int):
        """Producer rank of each candidate of the last tagged pass (producer == -2)."""
        mt = np.empty(max(n_mag, 1), dtype=np.int32)
        pt = np.empty(max(n_ph, 1), dtype=np.int32)
        nat.check(nat.load().svb_candidate_tags(self.handle, mt.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                                mt.size, pt.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                                pt.size))
        return mt[:n_mag], pt[:n_ph]

    def collect_tagged(self, d: "SvbGateDesc", ranks: int):
        """One pass over every work item with candidates tagged by reference producer rank;
        returns per-rank [(mags, phase values)] and the uncertain amplitudes, or None when
        the candidate buffer overflowed (the caller then runs one pass per rank)."""
        d.producer = -2
        d.collect = 1
        self.reset()
        self.gate_pass(d)
        mags, ph, flags = self.read_candidates()
        if flags & 1:
            return None
        unsure = self.read_unsure()
        mt, pt = self.read_candidate_tags(len(mags), len(ph))
        return [(mags[mt == r], ph[pt == r]) for r in range(ranks)], unsure

    def read_unsure(self):
        idx, vals = self._host_buffers()[2:]
        n = ctypes.c_uint64(0)
        nat.check(nat.load().svb_unsure(self.handle, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                        nat.dptr(vals), _CAP, ctypes.byref(n)))
        k = n.value
        return idx[:k].copy(), vals[0:2 * k:2] + 1j * vals[1:2 * k:2]

    def reset(self):
        nat.check(nat.load().svb_reset(self.handle))

    def patch(self, idx, mi, pi, in_place: bool = False):
        """Host-encoded bytes into the pending planes (or the current ones after an
        in-place pass)."""
        if len(idx) == 0:
            return
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        mi = np.ascontiguousarray(mi, dtype=np.uint8)
        pi = np.ascontiguousarray(pi, dtype=np.uint8)
        fn = nat.load().svb_patch_in_place if in_place else nat.load().svb_patch
        nat.check(fn(self.handle, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                       mi.ctypes.data_as(ctypes.c_void_p), pi.ctypes.data_as(ctypes.c_void_p),
                                       idx.size))
        self.launches += 1

    def commit(self):
        nat.check(nat.load().svb_commit(self.handle))
        self.version += 1

    def gate_pass(self, desc: SvbGateDesc, in_place: bool = False):
        """One pass; in_place (diagonal write pass with fixed tables): only the selected
        amplitudes of the current planes are rewritten, no commit follows."""
        fn = nat.load().svb_gate_in_place if in_place else nat.load().svb_gate
        # all-zero phase planes: skip reading them, and writing them while the uploaded
        # phase table (the one this pass encodes with) still has one entry
        desc.ph_zero_in = 1 if self.ph_zero else 0
        desc.ph_zero_out = 1 if (self.ph_zero and self._tables_version is not None
                                 and self._tables_version[2] == 1) else 0
        if self.ph_zero and not desc.ph_zero_out and not desc.scan_only:
            self.ph_zero = False         # this pass writes real phase indices
        if getattr(self, "time_passes", False):
            e0, e1 = nat.Event(), nat.Event()
            e0.record(self.stream)
            nat.check(fn(self.handle, ctypes.byref(desc)))
            e1.record(self.stream)
            self.pass_events.append((desc.scan_only, e0, e1))
        else:
            nat.check(fn(self.handle, ctypes.byref(desc)))
        self.launches += 1

    def finish_gate(self, ui, uv, in_place: bool) -> int:
        """Patch the host-encoded uncertain amplitudes and publish the gate's planes."""
        self.reset()
        if len(ui):
            mi, pi = self.codebook.host_encode(uv)
            self.patch(ui, mi, pi, in_place)
        if in_place:
            self.version += 1
        else:
            self.commit()
        return len(ui)

    # -- array-level codec -----------------------------------------------------------
    def encode_values(self, v: np.ndarray):
        self.sync_tables()
        n = v.size
        mi = np.empty(n, dtype=np.uint8)
        pi = np.empty(n, dtype=np.uint8)
        self.reset()
        nat.check(nat.load().svb_encode_values(self.handle, v.view(np.float64).ctypes.data_as(
            ctypes.POINTER(ctypes.c_double)), n, mi.ctypes.data_as(ctypes.c_void_p),
            pi.ctypes.data_as(ctypes.c_void_p), 0))
        idx, vals = self.read_unsure()
        self.reset()
        if len(idx):
            fm, fp = self.codebook.host_encode(vals)
            mi[idx.astype(np.int64)] = fm
            pi[idx.astype(np.int64)] = fp
        return mi, pi

    def collect_values(self, v: np.ndarray):
        self.sync_tables()
        n = v.size
        mi = np.empty(max(n, 1), dtype=np.uint8)
        pi = np.empty(max(n, 1), dtype=np.uint8)
        self.reset()
        nat.check(nat.load().svb_encode_values(self.handle, v.view(np.float64).ctypes.data_as(
            ctypes.POINTER(ctypes.c_double)), n, mi.ctypes.data_as(ctypes.c_void_p),
            pi.ctypes.data_as(ctypes.c_void_p), 1))
        mags, ph, flags = self.read_candidates()
        self.reset()
        if flags & 1:
            raise RuntimeError("codebook candidate buffer overflow in propose()")
        return mags, ph

    def free(self):
        if getattr(self, "handle", None):
            nat.load(require_device=False).svb_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def set_logical_bits(d: SvbGateDesc, layout, pos, phys_base: int) -> None:
    """Where the logical bits the producer rule reads live physically (pos: logical ->
    physical qubit, None for the identity)."""
    loc = layout.local_qubits
    rank_bits = layout.total_qubits - loc
    d.rank_bits = rank_bits
    d.phys_base = phys_base
    for j in range(2 + rank_bits):
        lq = loc - 2 + j
        d.lbit[j] = 0 if lq < 0 else (lq if pos is None else pos[lq])


def _exchange_fields(desc: SvbGateDesc, gate, layout, plan) -> None:
    loc = layout.local_qubits
    desc.n_local = loc
    if plan.kind == "pairwise" and len(gate.qubits) == 1:
        desc.xkind, desc.xmask_a = 1, plan.masks[0]
    elif plan.kind == "pairwise":
        desc.xkind, desc.xmask_a = 2, plan.masks[0]
        (ql,) = [q for q in gate.qubits if q < loc]
        desc.qlow_top = 1 if ql == loc - 1 else 0
    elif plan.kind == "quad":
        desc.xkind, desc.xmask_a, desc.xmask_b = 3, plan.masks[0], plan.masks[1]
    else:
        desc.xkind = 0


class ByteEngineState(ByteDeviceState):
    """The engine's whole-register BYTE state (all rank slices in one buffer)."""

    track_support = True

    def __init__(self, n_qubits: int, layout, device: int = 0):
        super().__init__(n_qubits, Codebook(), device)
        self.layout = layout
        self.passes = 0
        self.reencodes = 0
        self.host_fixes = 0
        self.sup_free = (1 << n_qubits) - 1        # dense until zero() records a basis state
        self.sup_val = 0
        self.scan_first = False         # the previous gate grew a table: scan before encoding

    def _desc(self, gate, plan) -> SvbGateDesc:
        d = SvbGateDesc()
        if g.is_diagonal(gate):
            d.kind = nat.SV_OP_DIAG
            mask = 0
            for q in gate.qubits:
                mask |= 1 << q
            d.diag_mask = mask
            f = g.diagonal_factor(gate)
            d.m[0], d.m[1] = f.real, f.imag
        else:
            m = nat.mat_buffer(g.unitary_matrix(gate))
            for i, v in enumerate(m):
                d.m[i] = v
            d.kind = nat.SV_OP_1Q if len(gate.qubits) == 1 else nat.SV_OP_2Q
            d.qa = gate.qubits[0]
            d.qb = gate.qubits[1] if len(gate.qubits) == 2 else 0
        _exchange_fields(d, gate, self.layout, plan)
        set_logical_bits(d, self.layout, None, 0)
        d.producer = -1
        d.mag_cut = d.ph_cut = _BIG
        # support before the gate (csrc sv_byte.cu: the vector passes visit only its items; both
        # plane buffers hold zeros outside it, so it may only grow -- monomials free their qubits)
        all_bits = (1 << self.n_qubits) - 1
        d.sup_fixed = all_bits & ~self.sup_free
        d.sup_val = self.sup_val & d.sup_fixed
        return d

    def _collect_rank(self, d: SvbGateDesc, rank: int):
        """One pass restricted to `rank`'s work items; returns (mag cands, phase values, unsure)."""
        d.producer = rank
        d.collect = 1
        cb = self.codebook
        while True:
            self.reset()
            self.gate_pass(d)
            self.passes += 1
            mags, ph, flags = self.read_candidates()
            unsure = self.read_unsure()
            if not flags & 1:
                return mags, ph, unsure
            # candidate buffer overflowed: keep only the smallest values (merge can only
            # append the smallest `room` of them) and run again
            k = 4 * (CAPACITY + 1)
            um = np.unique(mags)
            if len(um) > k:
                d.mag_cut = float(um[k])
            _, th, _, _ = __import__("paper_2511_03359_b200.codec", fromlist=["canonicalize"]).canonicalize(ph)
            ut = np.unique(th)
            if len(ut) > k:
                d.ph_cut = float(ut[k]) + 1e-13
            if len(um) <= k and len(ut) <= k:
                raise RuntimeError("codebook candidate buffer overflow without a usable cut")

    def _write_pass(self, d: SvbGateDesc, in_place: bool = False):
        d.producer = -1
        d.collect = 0
        d.scan_only = 0
        self.reset()
        self.gate_pass(d, in_place)
        self.passes += 1
        return self.read_unsure()

    def apply_gate(self, gate, layout=None) -> None:
        """One gate with the reference's per-gate codebook barrier (engine.py:186-225).

        Pass policy: tables that can no longer change -> one encode pass; after a
        gate that grew a table -> candidate scan first (reads only), merge, then
        one encode pass; otherwise encode speculatively while collecting and
        re-encode only if the merge grew a table."""
        from .layout import plan_exchange
        from .state import PrecisionMode
        plan = plan_exchange(self.layout, gate, PrecisionMode.BYTE)
        cb = self.codebook
        self.sync_tables()
        sat_mag, sat_ph = cb.tables_saturated
        d = self._desc(gate, plan)
        d.want_mag = 0 if sat_mag else 1
        d.want_ph = 0 if sat_ph else 1
        # a diagonal gate's final write pass (tables fixed) rewrites only the amplitudes it
        # selects, in the current planes; the speculative encode-while-collecting pass
        # keeps its input intact (a table that grows forces a re-encode from it)
        in_place = IN_PLACE and d.kind == nat.SV_OP_DIAG
        final_in_place = False
        if sat_mag and sat_ph:
            ui, uv = self._write_pass(d, in_place)
            final_in_place = in_place
        else:
            # diagonal gates always scan first: the scan reads only the selected amplitudes
            # and the write pass then runs in place with the merged tables
            scan = self.scan_first or in_place
            proposals, unsure = [], []
            ranks = self.layout.rank_count
            d.scan_only = 1 if scan else 0
            tagged = self.collect_tagged(d, ranks) if 1 < ranks <= MAX_TAGGED_RANKS else None
            if tagged is not None:
                self.passes += 1
                per_rank, u = tagged
                proposals = [cb.finalize_proposal(m, p) for m, p in per_rank]
                unsure = [u]
            else:
                for r in range(ranks):
                    mags, ph, u = self._collect_rank(d, r if ranks > 1 else -1)
                    proposals.append(cb.finalize_proposal(mags, ph))
                    unsure.append(u)
            version = cb.version
            cb.merge(proposals)
            grew = cb.version != version
            self.scan_first = grew
            if scan or grew:
                self.sync_tables()
                ui, uv = self._write_pass(d, in_place)
                final_in_place = in_place
                if grew and not scan:
                    self.reencodes += 1
            else:
                ui = np.concatenate([u[0] for u in unsure])
                uv = np.concatenate([u[1] for u in unsure])
        self.host_fixes += self.finish_gate(ui, uv, final_in_place)
        if not g.is_diagonal(gate):
            for q in gate.qubits:
                self.sup_free |= 1 << q
