"""ctypes binding of libofdmrx_b200.so (include/ofdmrx_b200.h).

The shared library is the product's compute path.  There is no fallback: if
it is missing or cannot be loaded every entry point raises DeviceError."""

import ctypes
import os
import threading

from .errors import (
    ConfigurationError,
    ContractError,
    DeviceError,
    InputError,
    NumericInputError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libofdmrx_b200.so")
ABI_VERSION = 2

OK, ERR_CONFIG, ERR_CONTRACT, ERR_INPUT, ERR_NUMERIC, ERR_CUDA = range(6)
FLAG_NONFINITE = 1
FLAG_ERASED = 2
FLAG_NOT_DETECTED = 4
FLAG_OUT_OF_RANGE = 8
OPT_PILOT_BPSK = 1
OPT_NO_SHARDS = 2
OPT_LATENCY = 4

_STATUS_EXC = {
    ERR_CONFIG: ConfigurationError,
    ERR_CONTRACT: ContractError,
    ERR_INPUT: InputError,
    ERR_NUMERIC: NumericInputError,
    ERR_CUDA: DeviceError,
}


class FrameDesc(ctypes.Structure):
    """ofdmrx_frame_desc."""

    _fields_ = [
        ("n_frames", ctypes.c_int32),
        ("n_antennas", ctypes.c_int32),
        ("fft_len", ctypes.c_int32),
        ("cp_len", ctypes.c_int32),
        ("n_data", ctypes.c_int32),
        ("qam_order", ctypes.c_int32),
        ("symbol0_offset", ctypes.c_int64),
        ("row_stride", ctypes.c_int64),
        ("frame_stride", ctypes.c_int64),
        ("eps", ctypes.c_float),
        ("options", ctypes.c_int32),
        ("rx_samples", ctypes.c_int64),
    ]


class Plan(ctypes.Structure):
    """ofdmrx_plan."""

    _fields_ = [(name, ctypes.c_int32) for name in
                ("kernel", "workers", "lanes_per_cta", "cluster", "ctas", "threads", "smem_bytes", "chunks")]


KERNEL_BALANCED, KERNEL_FUSED, KERNEL_ROWS = 1, 2, 3


_p = ctypes.c_void_p
_i32, _i64, _f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
_DESC = ctypes.POINTER(FrameDesc)


class SynthDesc(ctypes.Structure):
    """ofdmrx_synth_desc."""

    _fields_ = [
        ("n_frames", ctypes.c_int32),
        ("n_antennas", ctypes.c_int32),
        ("fft_len", ctypes.c_int32),
        ("cp_len", ctypes.c_int32),
        ("n_data", ctypes.c_int32),
        ("qam_order", ctypes.c_int32),
        ("pn_len", ctypes.c_int32),
        ("n_taps", ctypes.c_int32),
        ("resp_per_frame", ctypes.c_int32),
        ("noisy", ctypes.c_int32),
        ("snr_db", ctypes.c_float),
        ("timing_offset", ctypes.c_int64),
        ("n_samples", ctypes.c_int64),
        ("seed", ctypes.c_uint64),
    ]


_SDESC = ctypes.POINTER(SynthDesc)

# exported symbol -> (restype, argtypes); must match include/ofdmrx_b200.h
SIGNATURES = {
    "ofdmrx_abi_version": (ctypes.c_int, []),
    "ofdmrx_last_error": (ctypes.c_char_p, []),
    "ofdmrx_check_desc": (ctypes.c_int, [_DESC]),
    "ofdmrx_rx_plan": (ctypes.c_int, [_DESC, _i32, _i32, ctypes.POINTER(Plan)]),
    "ofdmrx_rx_frames": (ctypes.c_int, [_DESC, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "ofdmrx_rx_partials": (ctypes.c_int, [_DESC, _p, _p, _p, _p, _p, _p, _p]),
    "ofdmrx_rx_frames_profiled": (ctypes.c_int, [_DESC, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "ofdmrx_mrc_finish": (ctypes.c_int, [_i32, _i32, _i32, _i32, _i32, _p, _p, _f32, _p, _p, _p, _p, _p]),
    "ofdmrx_fft_shift": (ctypes.c_int, [_DESC, _i32, _i32, _p, _p, _p]),
    "ofdmrx_ls": (ctypes.c_int, [_i32, _i32, _i32, _p, _i64, _p, _p, _p]),
    "ofdmrx_mrc": (ctypes.c_int, [_i32, _i32, _i32, _i32, _p, _i64, _i64, _p, _f32, _i32, _p, _p, _p, _p]),
    "ofdmrx_demap": (ctypes.c_int, [_p, _i64, _i32, _p, _p]),
    "ofdmrx_stage_symbols": (ctypes.c_int, [_DESC, _p, _p, _p]),
    "ofdmrx_detect_scratch_bytes": (ctypes.c_int64, [_i32, _i32, _i64, _i32]),
    "ofdmrx_corr_metrics": (ctypes.c_int, [_p, _i32, _i32, _i64, _i64, _i64, _p, _i32, _p, _p]),
    "ofdmrx_detect": (ctypes.c_int, [_p, _i32, _i32, _i64, _i64, _i64, _p, _i32, _p, _p, _p, _p]),
    "ofdmrx_synth_bits": (ctypes.c_int, [_p, _i32, _i64, ctypes.c_uint64, _p]),
    "ofdmrx_synth_rayleigh": (ctypes.c_int, [_p, _i32, ctypes.c_uint64, _p]),
    "ofdmrx_synth_frames": (ctypes.c_int, [_SDESC, _p, _p, _p, _p, _p, _p]),
    "ofdmrx_rx_partials_routed": (ctypes.c_int, [_DESC, _p, _p, _p, _p, _p, _i32, _i32, _p, _p]),
    "ofdmrx_rx_frames_detected": (ctypes.c_int, [_DESC, _i64, _p, _p, _i32, _i32, ctypes.c_double, _p, _p, _p, _p, _p,
                                                 _p, _p, _p, _p]),
    "ofdmrx_peer_alloc": (ctypes.c_int, [_i64, ctypes.POINTER(ctypes.c_void_p), _p]),
    "ofdmrx_peer_open": (ctypes.c_int, [_p, ctypes.POINTER(ctypes.c_void_p)]),
    "ofdmrx_peer_close": (ctypes.c_int, [_p]),
    "ofdmrx_peer_free": (ctypes.c_int, [_p]),
    "ofdmrx_peer_signal": (ctypes.c_int, [_p, _i32, ctypes.c_uint64, _p]),
    "ofdmrx_peer_wait": (ctypes.c_int, [_p, _i32, ctypes.c_uint64, _p]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the native library; raise DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is not built; run `python -m paper_1901_07499_b200.build` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ofdmrx_abi_version() != ABI_VERSION:
            raise DeviceError("libofdmrx_b200.so ABI version mismatch; rebuild it")
        _lib = lib
    return _lib


def last_error():
    msg = load().ofdmrx_last_error()
    return msg.decode() if msg else ""


def check(rc):
    """Map a status code onto the errors.py taxonomy."""
    if rc == OK:
        return
    exc = _STATUS_EXC.get(rc, DeviceError)
    raise exc(last_error() or f"ofdmrx status {rc}")


def call(name, *args):
    check(getattr(load(), name)(*args))
