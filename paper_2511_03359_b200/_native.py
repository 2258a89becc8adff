"""ctypes binding of libsvb200.so (the C ABI declared in include/svb200.h).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is visible, every device operation raises.  The product path runs on
the B200 or not at all.
"""
from __future__ import annotations

import atexit
import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsvb200.so")

SV_OK, SV_EINDEX, SV_EVALUE, SV_ECUDA, SV_ENOMEM = 0, -1, -2, -3, -4
SV_FP64, SV_FP32, SV_BYTE = 0, 1, 2
SV_OP_1Q, SV_OP_2Q, SV_OP_DIAG = 1, 2, 3


class NativeUnavailable(RuntimeError):
    """libsvb200.so could not be loaded or no CUDA device is present."""


class SvOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("qa", ctypes.c_int32), ("qb", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("diag_mask", ctypes.c_uint64),
                ("m", ctypes.c_double * 32)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_U64 = ctypes.c_uint64
_I = ctypes.c_int

_SIGNATURES = {
    "sv_abi_version": ([], _I),
    "sv_mem_info": ([_I, ctypes.POINTER(_U64), ctypes.POINTER(_U64)], _I),
    "sv_last_error": ([], ctypes.c_char_p),
    "sv_device_count": ([ctypes.POINTER(_I)], _I),
    "sv_sm_count": ([_I, ctypes.POINTER(_I)], _I),
    "sv_set_device": ([_I], _I),
    "svk_apply_1q": ([_P, _U64, _I, _I, _D, _P], _I),
    "svk_apply_2q": ([_P, _U64, _I, _I, _I, _D, _P], _I),
    "svk_apply_diag": ([_P, _U64, _I, _U64, _D, _P], _I),
    "svk_pair_update": ([_P, _P, _U64, _I, _D, _P], _I),
    "svk_quad_update": ([ctypes.POINTER(_P), _U64, _I, _D, _P], _I),
    "svk_apply_fused": ([_P, _U64, _I, ctypes.POINTER(SvOp), _I, _I, _P], _I),
    "svk_measure": ([_P, _U64, _I, _D, _D, _D, _P], _I),
    "sv_create": ([_I, _I, _I, ctypes.POINTER(_P)], _I),
    "sv_destroy": ([_P], _I),
    "sv_zero_state": ([_P, ctypes.c_int64], _I),
    "sv_zero_state_lazy": ([_P, ctypes.c_int64], _I),
    "sv_info": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I),
                 ctypes.POINTER(_P), ctypes.POINTER(_P)], _I),
    "sv_apply_1q": ([_P, _I, _D], _I),
    "sv_apply_2q": ([_P, _I, _I, _D], _I),
    "sv_apply_diag": ([_P, _U64, _D], _I),
    "sv_apply_fused": ([_P, ctypes.POINTER(SvOp), _I, _I], _I),
    "sv_measure": ([_P, _D, _D, _D], _I),
    "sv_export": ([_P, _P, _U64, _U64], _I),
    "sv_import": ([_P, _P, _U64, _U64], _I),
    "sv_synchronize": ([_P], _I),
    "svb_create": ([_I, _I, ctypes.POINTER(_P)], _I),
    "svb_destroy": ([_P], _I),
    "svb_info": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_P)], _I),
    "svb_zero_state": ([_P, ctypes.c_int64], _I),
    "svb_set_tables": ([_P, _D, _I, _D, _D, _D, _I], _I),
    "svb_gate": ([_P, _P], _I),
    "svb_gate_in_place": ([_P, _P], _I),
    "svb_candidate_tags": ([_P, ctypes.POINTER(ctypes.c_int32), _U64, ctypes.POINTER(ctypes.c_int32), _U64], _I),
    "svb_candidates": ([_P, _D, _U64, ctypes.POINTER(_U64), _D, _U64, ctypes.POINTER(_U64),
                        ctypes.POINTER(_I)], _I),
    "svb_unsure": ([_P, ctypes.POINTER(_U64), _D, _U64, ctypes.POINTER(_U64)], _I),
    "svb_reset": ([_P], _I),
    "svb_patch": ([_P, ctypes.POINTER(_U64), _P, _P, _U64], _I),
    "svb_patch_in_place": ([_P, ctypes.POINTER(_U64), _P, _P, _U64], _I),
    "svb_commit": ([_P], _I),
    "svb_export": ([_P, _P, _P, _U64, _U64], _I),
    "svb_import": ([_P, _P, _P, _U64, _U64], _I),
    "svb_decode": ([_P, _D, _U64, _U64], _I),
    "svb_measure": ([_P, _D, _D, _D], _I),
    "svb_measure_support": ([_P, _U64, _U64, _D, _D, _D], _I),
    "svb_encode_values": ([_P, _D, _U64, _P, _P, _I], _I),
    "sv_ipc_handle": ([_P, _P], _I),
    "sv_ipc_open": ([_I, _P, ctypes.POINTER(_P)], _I),
    "sv_ipc_close": ([_I, _P], _I),
    "sv_ipc_unexport_all": ([ctypes.POINTER(_U64)], _I),
    "svk_swap_peer": ([_P, _P, _U64, _I, _I, _I, _P], _I),
    "svk_pair_dot": ([_P, _P, _U64, _I, _I, _D, _P], _I),
    "svk_pair_dot_chunk": ([_P, _P, _U64, _I, _U64, _U64, _U64, _U64, _I, _D, _P], _I),
    "sv_release_cached": ([], _I),
    "sv_cached_bytes": ([ctypes.POINTER(_U64)], _I),
    "sv_jit_mode": ([_I], _I),
    "sv_jit_wait": ([], _I),
    "sv_jit_shutdown": ([], _I),
    "sv_jit_prepare": ([_I, _P, _I, _I], _I),
    "sv_jit_prepare_mode": ([_I, _I, _P, _I, _I], _I),
    "sv_jit_prepare_opts": ([_I, _I, _P, _I, _I, _I], _I),
    "sv_set_diag_combine": ([_P, _I], _I),
    "sv_set_support_tracking": ([_P, _I], _I),
    "sv_support_info": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_U64)], _I),
    "sv_set_support": ([_P, _U64, _U64], _I),
    "sv_support_advance": ([_P, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64)], _I),
    "sv_plan_passes": ([_I, _I, _P, _I, _I, ctypes.POINTER(_I), _I], _I),
    "sv_plan_pass_costs": ([_I, _I, _P, _I, _I, ctypes.POINTER(_I), _D, _I, _I], _I),
    "sv_jit_stats": ([_D], _I),
    "sv_jit_available": ([], _I),
    "sv_jit_probe": ([_P, _I, _I, ctypes.c_char_p, ctypes.c_size_t, _D], _I),
    "sv_swap_blocks": ([_I], _I),
    "sv_measure_reserve": ([_I], _I),
    "svk_swap_group_chunk": ([_P, _P, _U64, _I, _U64, _U64, _U64, _U64, _U64, _U64, _U64, _P], _I),
    "sv_apply_fused_chunk": ([_P, _P, _I, _I, _U64, _U64], _I),
    "sv_event_create_ipc": ([ctypes.POINTER(_P), _P], _I),
    "sv_event_open_ipc": ([_P, ctypes.POINTER(_P)], _I),
    "sv_stream_wait_event": ([_P, _P], _I),
    "svk_swap_group": ([_P, _P, _U64, _I, _U64, _U64, _U64, _U64, _U64, _P], _I),
    "svb_ipc_handles": ([_P, _P], _I),
    "svb_cur": ([_P], _I),
    "svb_planes": ([_P, ctypes.POINTER(_P), ctypes.POINTER(_P)], _I),
    "svb_swap_peer": ([_P, _P, _P, _I, _I], _I),
    "svb_clear_pending": ([_P], _I),
    "svb_swap_group": ([_P, _P, _P, _U64, _U64, _U64, _U64, _U64], _I),
    "svb_pair_dot": ([_P, _P, _P, _P, _P, _U64, _D], _I),
    "sv_buffer_alloc": ([_I, _U64, ctypes.POINTER(_P)], _I),
    "sv_buffer_free": ([_I, _P], _I),
    "sv_copy_h2d": ([_P, _P, _U64, _P], _I),
    "sv_copy_d2h": ([_P, _P, _U64, _P], _I),
    "sv_stream_create": ([_I, ctypes.POINTER(_P)], _I),
    "sv_stream_destroy": ([_P], _I),
    "sv_launch_count": ([ctypes.POINTER(_U64)], _I),
    "sv_transfer_bytes": ([ctypes.POINTER(_U64), ctypes.POINTER(_U64)], _I),
    "sv_fused_variant": ([_I], _I),
    "sv_fused_segment_limit": ([_I], _I),
    "sv_pass_timing": ([_I], _I),
    "sv_pass_timing_read": ([ctypes.POINTER(_U64), _D, _D], _I),
    "sv_event_create": ([ctypes.POINTER(_P)], _I),
    "sv_event_destroy": ([_P], _I),
    "sv_event_record": ([_P, _P], _I),
    "sv_event_elapsed_ms": ([_P, _P, ctypes.POINTER(ctypes.c_float)], _I),
    "sv_stream_synchronize": ([_P], _I),
    "svk_f32_round": ([_D, _D, _U64, _I], _I),
    "svt_create": ([_I, _I, _I, _I, _P, _I, ctypes.POINTER(_P)], _I),
    "svt_destroy": ([_P], _I),
    "svt_zero_state": ([_P, ctypes.c_int64], _I),
    "svt_apply_run": ([_P, _P, _I, _I], _I),
    "svt_apply_pairing": ([_P, _P], _I),
    "svt_measure": ([_P, _D, _D, _D], _I),
    "svt_export": ([_P, _P, _U64, _U64], _I),
    "svt_import": ([_P, _P, _U64, _U64], _I),
    "svt_synchronize": ([_P], _I),
    "svt_stats": ([_P, ctypes.POINTER(_U64)], _I),
}

_lib = None
_lock = threading.Lock()


def exported_symbols():
    return sorted(_SIGNATURES)


def load(require_device: bool = True):
    """Load libsvb200.so once; raise NativeUnavailable if it cannot run."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2511_03359_b200.build`")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
            # background NVRTC compiles must not outlive the interpreter: stop them
            # before Python and the CUDA runtime tear down (sv_jit.cu)
            atexit.register(lib.sv_jit_shutdown)
    if require_device:
        n = ctypes.c_int(0)
        if _lib.sv_device_count(ctypes.byref(n)) != SV_OK or n.value < 1:
            raise NativeUnavailable("no CUDA device visible: the B200 path has no CPU fallback")
    return _lib


def check(rc: int) -> None:
    """Map an SV_E* status to the reference's exception type."""
    if rc == SV_OK:
        return
    msg = _lib.sv_last_error().decode(errors="replace")
    if rc == SV_EINDEX:
        raise IndexError(msg)
    if rc == SV_EVALUE:
        raise ValueError(msg)
    if rc == SV_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def dptr(arr: np.ndarray):
    return arr.ctypes.data_as(_D)


def mat_buffer(matrix) -> np.ndarray:
    """Row-major complex matrix -> contiguous (re, im) doubles."""
    m = np.ascontiguousarray(np.asarray(matrix, dtype=np.complex128))
    return m.view(np.float64).ravel().copy()


def mode_code(mode) -> int:
    value = getattr(mode, "value", mode)
    return {"fp64": SV_FP64, "fp32": SV_FP32, "be": SV_BYTE}[value]


def launch_count() -> int:
    c = ctypes.c_uint64(0)
    check(load(require_device=False).sv_launch_count(ctypes.byref(c)))
    return int(c.value)


def transfer_bytes():
    """(h2d, d2h) bytes moved by the library so far."""
    a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
    check(load(require_device=False).sv_transfer_bytes(ctypes.byref(a), ctypes.byref(b)))
    return int(a.value), int(b.value)


def pass_timing(enable: bool) -> None:
    check(load(require_device=False).sv_pass_timing(1 if enable else 0))


def pass_timing_read():
    """(passes, device ms, algorithmic bytes) of the fused passes since the last read."""
    n = ctypes.c_uint64(0)
    ms = np.zeros(1)
    by = np.zeros(1)
    check(load(require_device=False).sv_pass_timing_read(ctypes.byref(n), dptr(ms), dptr(by)))
    return int(n.value), float(ms[0]), float(by[0])


class Stream:
    """A CUDA stream owned by the library (non-blocking)."""

    def __init__(self, device: int = 0):
        lib = load()
        p = ctypes.c_void_p()
        check(lib.sv_stream_create(device, ctypes.byref(p)))
        self.ptr = p
        self.device = device

    def synchronize(self):
        check(_lib.sv_stream_synchronize(self.ptr))

    def close(self):
        if self.ptr:
            _lib.sv_stream_synchronize(self.ptr)
            _lib.sv_stream_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceBuffer:
    """Raw device allocation, freed with the object."""

    def __init__(self, nbytes: int, device: int = 0):
        lib = load()
        p = ctypes.c_void_p()
        check(lib.sv_buffer_alloc(device, int(nbytes), ctypes.byref(p)))
        self.ptr = p
        self.nbytes = int(nbytes)
        self.device = device

    def upload(self, host: np.ndarray, stream: Stream):
        host = np.ascontiguousarray(host)
        assert host.nbytes <= self.nbytes
        check(_lib.sv_copy_h2d(self.ptr, host.ctypes.data_as(_P), host.nbytes, stream.ptr))

    def download(self, host: np.ndarray, stream: Stream):
        assert host.flags.c_contiguous and host.nbytes <= self.nbytes
        check(_lib.sv_copy_d2h(host.ctypes.data_as(_P), self.ptr, host.nbytes, stream.ptr))

    def offset(self, nbytes: int) -> ctypes.c_void_p:
        return ctypes.c_void_p(self.ptr.value + int(nbytes))

    def free(self):
        if self.ptr:
            _lib.sv_buffer_free(self.device, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Event:
    def __init__(self):
        lib = load()
        p = ctypes.c_void_p()
        check(lib.sv_event_create(ctypes.byref(p)))
        self.ptr = p

    def record(self, stream):
        check(_lib.sv_event_record(self.ptr, stream.ptr if isinstance(stream, Stream) else stream))

    def elapsed_ms(self, later: "Event") -> float:
        out = ctypes.c_float()
        check(_lib.sv_event_elapsed_ms(self.ptr, later.ptr, ctypes.byref(out)))
        return float(out.value)

    def __del__(self):
        try:
            _lib.sv_event_destroy(self.ptr)
        except Exception:
            pass
