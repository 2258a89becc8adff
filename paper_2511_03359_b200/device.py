"""HBM-resident state vectors: the Python face of an ``sv_handle``.

A ``DeviceState`` is 2**n amplitudes in one B200's HBM (interleaved
complex128 for FP64, complex64 for FP32), with its own CUDA stream.  Every
mutation is a kernel of libsvb200.so launched on that stream; nothing here
computes on the host.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat

_DTYPE = {nat.SV_FP64: np.complex128, nat.SV_FP32: np.complex64}


def gate_op(kind: int, qa: int = 0, qb: int = 0, mask: int = 0, data=()) -> nat.SvOp:
    op = nat.SvOp()
    op.kind, op.qa, op.qb, op.diag_mask = kind, qa, qb, mask
    for i, v in enumerate(data):
        op.m[i] = float(v)
    return op


def ops_array(ops) -> ctypes.Array:
    arr = (nat.SvOp * max(1, len(ops)))()
    for i, o in enumerate(ops):
        arr[i] = o
    return arr


def jit_prepare(n_qubits: int, ops, tile_bits: int = 12, mode_code: int = nat.SV_FP64,
                combine_diag: bool = False) -> int:
    """Queue the specialised kernels (sv_jit.cu) of the fused passes `ops` will run on
    2**n_qubits amplitudes (FP64 or FP32 storage); returns how many new kernels were queued.
    combine_diag: the kernels of a state with combined diagonal runs (set_diag_combine)."""
    if not ops:
        return 0
    lib = nat.load(require_device=False)
    if combine_diag:
        rc = lib.sv_jit_prepare_opts(n_qubits, mode_code, ops_array(ops), len(ops), tile_bits, 1)
    else:
        rc = lib.sv_jit_prepare_mode(n_qubits, mode_code, ops_array(ops), len(ops), tile_bits)
    nat.check(min(rc, 0))
    return rc


def release_cached_memory() -> int:
    """Return the cached state slabs (sv_slab.cu) to the driver; returns the bytes released."""
    lib = nat.load(require_device=False)
    before = ctypes.c_uint64()
    nat.check(lib.sv_cached_bytes(ctypes.byref(before)))
    nat.check(lib.sv_release_cached())
    return int(before.value)


def jit_wait() -> None:
    nat.check(nat.load(require_device=False).sv_jit_wait())


def jit_stats() -> dict:
    out = np.zeros(8)
    nat.check(nat.load(require_device=False).sv_jit_stats(nat.dptr(out)))
    return {"compiled": int(out[0]), "failed": int(out[1]), "jit_launches": int(out[2]),
            "generic_fallbacks": int(out[3]), "compile_ms": round(float(out[4]), 1), "cached": int(out[5]),
            "disk_hits": int(out[6]), "disk_writes": int(out[7])}


class DeviceState:
    def __init__(self, n_qubits: int, mode, device: int = 0):
        lib = nat.load()
        self.n_qubits = int(n_qubits)
        self.mode_code = nat.mode_code(mode)
        if self.mode_code not in _DTYPE:
            raise ValueError("DeviceState holds FP64 or FP32 storage")
        self.device = device
        h = ctypes.c_void_p()
        nat.check(lib.sv_create(device, self.n_qubits, self.mode_code, ctypes.byref(h)))
        self.handle = h
        p, s = ctypes.c_void_p(), ctypes.c_void_p()
        nat.check(lib.sv_info(h, None, None, None, ctypes.byref(p), ctypes.byref(s)))
        self.ptr, self.stream = p, s
        self.version = 0
        self.launches = 0

    # -- properties -----------------------------------------------------------
    @property
    def size(self) -> int:
        return 1 << self.n_qubits

    @property
    def dtype(self):
        return _DTYPE[self.mode_code]

    @property
    def nbytes(self) -> int:
        return self.size * np.dtype(self.dtype).itemsize

    def set_diag_combine(self, on: bool) -> None:
        """FP64: runs of consecutive diagonal gates inside a fused pass multiply every
        amplitude by their combined factor (one rounding per register mask instead of per
        gate): amplitudes within 1e-12 relative of the reference -- the north star's FP64
        tolerance -- but not bit-identical.  Off by default."""
        nat.check(nat.load().sv_set_diag_combine(self.handle, 1 if on else 0))
        self.diag_combine = bool(on)

    def set_support_tracking(self, on: bool) -> None:
        """Record which index bits may differ from the initial basis state (sv_set_support_tracking):
        fused passes then skip the tiles that can only hold zeros.  Call before zero()."""
        nat.check(nat.load().sv_set_support_tracking(self.handle, 1 if on else 0))

    def support_info(self) -> dict:
        on, free, val, skipped = ctypes.c_int(0), ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_uint64(0)
        nat.check(nat.load().sv_support_info(self.handle, ctypes.byref(on), ctypes.byref(free), ctypes.byref(val),
                                             ctypes.byref(skipped)))
        return {"tracking": bool(on.value), "free_qubits": bin(free.value).count("1"),
                "tiles_skipped_total": int(skipped.value)}

    def _touch(self, launches: int = 1):
        self.version += 1
        self.launches += launches

    # -- initialisation / transfer ---------------------------------------------
    def zero(self, unit_index: int | None = 0, lazy: bool = False) -> None:
        """|unit_index> (None: all zeros).  lazy=True records it only: the first fused pass
        generates its tiles instead of reading them (sv_zero_state_lazy)."""
        fn = nat.load().sv_zero_state_lazy if lazy else nat.load().sv_zero_state
        nat.check(fn(self.handle, -1 if unit_index is None else unit_index))
        self._touch(0)

    def export(self, first: int = 0, count: int | None = None) -> np.ndarray:
        count = self.size - first if count is None else count
        out = np.empty(count, dtype=self.dtype)
        nat.check(nat.load().sv_export(self.handle, out.ctypes.data_as(ctypes.c_void_p), first, count))
        return out

    def import_(self, values: np.ndarray, first: int = 0) -> None:
        arr = np.ascontiguousarray(np.asarray(values), dtype=self.dtype)
        nat.check(nat.load().sv_import(self.handle, arr.ctypes.data_as(ctypes.c_void_p), first, arr.size))
        self._touch(0)

    # storage-level access used by LocalState mirrors (FP modes: one array)
    def export_storage(self, first: int, count: int) -> np.ndarray:
        return self.export(first, count)

    def import_storage(self, values, first: int = 0) -> None:
        self.import_(values, first)

    def element_ptr(self, index: int) -> ctypes.c_void_p:
        # sv_info with a pointer out-argument writes a lazily recorded basis state first
        p = ctypes.c_void_p()
        nat.check(nat.load().sv_info(self.handle, None, None, None, ctypes.byref(p), None))
        return ctypes.c_void_p(p.value + int(index) * np.dtype(self.dtype).itemsize)

    def measure_range(self, first: int, count: int):
        """(norm, ones, cross) of the sub-buffer [first, first + count), count = 2**k."""
        k = int(count).bit_length() - 1
        norm = np.zeros(1)
        ones = np.zeros(max(k, 1))
        cross = np.zeros(2 * max(k, 1))
        nat.check(nat.load().svk_measure(self.element_ptr(first), count, self.mode_code, nat.dptr(norm),
                                         nat.dptr(ones), nat.dptr(cross), self.stream))
        self.launches += 1
        return float(norm[0]), ones[:k].copy(), cross[0:2 * k:2] + 1j * cross[1:2 * k:2]

    def synchronize(self) -> None:
        nat.check(nat.load().sv_synchronize(self.handle))

    # -- gates ------------------------------------------------------------------
    def apply_1q(self, q: int, matrix) -> None:
        m = nat.mat_buffer(matrix)
        nat.check(nat.load().sv_apply_1q(self.handle, q, nat.dptr(m)))
        self._touch()

    def apply_2q(self, qa: int, qb: int, matrix) -> None:
        m = nat.mat_buffer(matrix)
        nat.check(nat.load().sv_apply_2q(self.handle, qa, qb, nat.dptr(m)))
        self._touch()

    def apply_diag(self, mask: int, factor: complex) -> None:
        f = np.array([complex(factor).real, complex(factor).imag])
        nat.check(nat.load().sv_apply_diag(self.handle, int(mask), nat.dptr(f)))
        self._touch()

    def apply_fused(self, ops, tile_bits: int = 12) -> None:
        if not ops:
            return
        arr = ops_array(ops)
        nat.check(nat.load().sv_apply_fused(self.handle, arr, len(ops), tile_bits))
        self._touch(max(1, len(ops)))

    # -- reductions ---------------------------------------------------------------
    def measure(self):
        """(norm, ones[n], cross[n] complex) over all n qubits of the buffer."""
        n = self.n_qubits
        norm = np.zeros(1)
        ones = np.zeros(max(n, 1))
        cross = np.zeros(2 * max(n, 1))
        nat.check(nat.load().sv_measure(self.handle, nat.dptr(norm), nat.dptr(ones), nat.dptr(cross)))
        self.launches += 1
        return float(norm[0]), ones[:n].copy(), (cross[0:2 * n:2] + 1j * cross[1:2 * n:2])

    def free(self) -> None:
        if getattr(self, "handle", None):
            nat.load(require_device=False).sv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
