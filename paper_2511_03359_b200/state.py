"""Per-rank amplitude storage (``svsim.state`` surface), resident in HBM.

Mirrors /root/reference/pkg/src/svsim/state.py: ``PrecisionMode`` (20-31:
16 / 8 / 2 bytes per element, norm tolerance 1e-5 for FP32 else 1e-12) and
``LocalState`` (34-103).  The difference is ownership: the amplitudes live in
device memory (a slice of a ``DeviceState``); ``psi`` / ``mag_idx`` /
``phase_idx`` are host mirrors exported on access and written back through
their setters (so ``state.psi *= 2.0`` behaves as in the reference).
"""
from __future__ import annotations

import enum

import numpy as np


class PrecisionMode(enum.Enum):
    FP64 = "fp64"
    FP32 = "fp32"
    BYTE = "be"

    @property
    def bytes_per_element(self) -> int:
        return {"fp64": 16, "fp32": 8, "be": 2}[self.value]

    @property
    def norm_tolerance(self) -> float:
        return 1e-5 if self is PrecisionMode.FP32 else 1e-12


class LocalState:
    """One partition's slice of the state vector, held on a B200."""

    def __init__(self, n_local: int, mode: PrecisionMode, *, _device_state=None, _offset: int = 0,
                 device: int = 0):
        self.n_local = n_local
        self.mode = mode
        if _device_state is None:
            _device_state = _new_storage(n_local, mode, device)
            _device_state.zero(None)
        self._dev = _device_state
        self._offset = _offset
        self._mirror = None
        self._mirror_version = -1

    @classmethod
    def zero_state(cls, n_local: int, mode: PrecisionMode, with_unit_amplitude: bool, device: int = 0):
        """All zeros; the partition owning global index 0 gets amplitude 1
        (in BYTE mode: magnitude index 1 = 1.0, phase index 0 = 0)."""
        dev = _new_storage(n_local, mode, device)
        dev.zero(0 if with_unit_amplitude else None)
        return cls(n_local, mode, _device_state=dev, _offset=0)

    @property
    def size(self) -> int:
        return 1 << self.n_local

    @property
    def storage_nbytes(self) -> int:
        return self.size * self.mode.bytes_per_element

    @property
    def device_state(self):
        return self._dev

    # -- host mirrors ------------------------------------------------------------
    def _storage(self):
        if self._mirror is None or self._mirror_version != self._dev.version:
            self._mirror = self._dev.export_storage(self._offset, self.size)
            self._mirror_version = self._dev.version
        return self._mirror

    def _write_storage(self, parts) -> None:
        self._dev.import_storage(parts, self._offset)
        self._mirror = None

    @property
    def psi(self) -> np.ndarray:
        if self.mode is PrecisionMode.BYTE:
            raise AttributeError("BYTE storage has mag_idx / phase_idx, not psi")
        return self._storage()

    @psi.setter
    def psi(self, values) -> None:
        if self.mode is PrecisionMode.BYTE:
            raise AttributeError("BYTE storage has mag_idx / phase_idx, not psi")
        self._write_storage(np.asarray(values))

    @property
    def mag_idx(self) -> np.ndarray:
        if self.mode is not PrecisionMode.BYTE:
            raise AttributeError("only BYTE storage has mag_idx")
        return self._storage()[0]

    @mag_idx.setter
    def mag_idx(self, values) -> None:
        self._write_storage((np.asarray(values, dtype=np.uint8), self.phase_idx.copy()))

    @property
    def phase_idx(self) -> np.ndarray:
        if self.mode is not PrecisionMode.BYTE:
            raise AttributeError("only BYTE storage has phase_idx")
        return self._storage()[1]

    @phase_idx.setter
    def phase_idx(self, values) -> None:
        self._write_storage((self.mag_idx.copy(), np.asarray(values, dtype=np.uint8)))

    # -- reference operations ------------------------------------------------------
    def working(self, codebook=None) -> np.ndarray:
        """Decoded complex128 copy of the slice (state.py:73-77)."""
        if self.mode is PrecisionMode.BYTE:
            return codebook.decode(self.mag_idx, self.phase_idx)
        return self.psi.astype(np.complex128)

    def store(self, values, codebook=None, where=None) -> None:
        """Write computed values back (state.py:79-99); BYTE re-encodes."""
        if self.mode is PrecisionMode.BYTE:
            mag, ph = codebook.encode(values)
            cur_m, cur_p = self.mag_idx.copy(), self.phase_idx.copy()
            sel = slice(None) if where is None else where
            cur_m[sel], cur_p[sel] = mag, ph
            self._write_storage((cur_m, cur_p))
            return
        cur = self.psi.copy()
        if where is None:
            cur[:] = values
        else:
            cur[where] = values
        self._write_storage(cur)

    def norm_squared(self, codebook=None) -> float:
        if self.mode is PrecisionMode.BYTE:
            w = self.working(codebook)
            from .kernels import norm_squared
            return norm_squared(w)
        norm, _, _ = self._dev.measure_range(self._offset, self.size)
        return norm


def _new_storage(n_local: int, mode: PrecisionMode, device: int):
    if mode is PrecisionMode.BYTE:
        from .byte_state import ByteDeviceState
        return ByteDeviceState(n_local, device=device)
    from .device import DeviceState
    return DeviceState(n_local, mode, device=device)
