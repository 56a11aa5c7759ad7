"""Torch-facing wrappers over the C ABI (include/ofdmrx_b200.h).

PyTorch is plumbing here: it owns device memory and streams; every numeric
operation is one of the library's sm_100a kernels.  Inputs may be numpy
arrays (copied to the device as complex64) or CUDA tensors (used in place
when already complex64 and contiguous)."""

import math

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError, ContractError, DeviceError, NumericInputError

MRC_WEIGHT_FLOOR = 1e-12  # receiver.py:33


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 receive path has no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise DeviceError(f"device {dev} is not a CUDA device")
    _lib.load()
    return dev


class on_stream:
    """Run allocations and launches of one call on `stream` (None = the
    current stream).  The stream first waits for the current stream, so
    inputs produced there are ready, and tensors allocated inside belong to
    `stream` in the caching allocator (a scratch buffer freed on return is
    only reused by later work on the same stream, never while a kernel on
    `stream` may still touch it)."""

    def __init__(self, stream):
        self.stream = stream
        self.ctx = None

    def __enter__(self):
        if self.stream is not None and self.stream != torch.cuda.current_stream(self.stream.device):
            self.stream.wait_stream(torch.cuda.current_stream(self.stream.device))
            self.ctx = torch.cuda.stream(self.stream)
            self.ctx.__enter__()
        return self

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)


def stream_handle(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes_void(s.cuda_stream)


def ctypes_void(v):
    import ctypes

    return ctypes.c_void_p(int(v))


def ptr(t):
    return None if t is None else ctypes_void(t.data_ptr())


def as_c64(x, device):
    """complex64 contiguous CUDA tensor view/copy of x (numpy or torch)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.device != device:
            t = t.to(device, non_blocking=True)
        if t.dtype != torch.complex64:
            if not t.is_complex():
                raise ContractError(f"expected complex samples, got {t.dtype}")
            t = t.to(torch.complex64)
        return t.contiguous()
    a = np.asarray(x)
    if not np.iscomplexobj(a):
        a = a.astype(np.complex128)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex64)).to(device, non_blocking=False)


def qam_bits(order):
    return {4: 2, 16: 4, 64: 6}[order]


def make_desc(n_frames, n_antennas, fft_len, cp_len, n_data, qam_order, symbol0_offset, row_stride,
              frame_stride, eps=MRC_WEIGHT_FLOOR, options=0, *, rx_samples):
    """ofdmrx_frame_desc; rx_samples = complex samples readable at the capture
    pointer (the C side bounds-checks every call against it)."""
    return _lib.FrameDesc(int(n_frames), int(n_antennas), int(fft_len), int(cp_len), int(n_data),
                          int(qam_order), int(symbol0_offset), int(row_stride), int(frame_stride),
                          float(eps), int(options), int(rx_samples))


def pilot_options(pilot_values):
    """OFDMRX_OPT_PILOT_BPSK when every pilot value is exactly +-1 + 0j."""
    v = np.asarray(pilot_values)
    return _lib.OPT_PILOT_BPSK if np.all((v.imag == 0) & (np.abs(v.real) == 1)) else 0


def check_desc(desc):
    import ctypes

    _lib.check(_lib.load().ofdmrx_check_desc(ctypes.byref(desc)))


def rx_plan(desc, mode=0):
    """ofdmrx_rx_plan: the kernel, worker count (antenna-sum order) and CTA
    mapping a fused call with this descriptor uses on the current device."""
    import ctypes

    out = _lib.Plan()
    _lib.check(_lib.load().ofdmrx_rx_plan(ctypes.byref(desc), int(mode), 0, ctypes.byref(out)))
    return {name: getattr(out, name) for name, _ in _lib.Plan._fields_}


# ---------------------------------------------------------------------------
# staged stages
# ---------------------------------------------------------------------------

def fft_shift_rows(rows, device=None, stream=None):
    """FFT + fftshift of each row of a [R, M] matrix -> complex64 [R, M] CUDA tensor."""
    import ctypes

    dev = require_cuda(device)
    x = as_c64(rows, dev)
    if x.dim() == 1:
        x = x[None, :]
    r, m = x.shape
    out = torch.empty((r, m), dtype=torch.complex64, device=dev)
    # rows as frames of one antenna and one symbol without CP
    desc = make_desc(r, 1, m, 0, 0, 4, 0, m, m, rx_samples=r * m)
    _lib.call("ofdmrx_fft_shift", ctypes.byref(desc), 0, 1, ptr(x), ptr(out), stream_handle(stream))
    return out


def ls(freq, pilot_values, device=None, stream=None):
    """H = Y * conj(P) for Y [N, M] (or [F, N, M])."""
    dev = require_cuda(device)
    y = as_c64(freq, dev)
    squeeze = y.dim() == 2
    if squeeze:
        y = y[None]
    f, n, m = y.shape
    p = as_c64(pilot_values, dev).reshape(-1)
    if p.numel() != m:
        raise ContractError(f"matrix has {m} subcarriers, pilot has {p.numel()}")
    h = torch.empty_like(y)
    _lib.call("ofdmrx_ls", f, n, m, ptr(y), n * m, ptr(p), ptr(h), stream_handle(stream))
    return h[0] if squeeze else h


def mrc(freq, gains, eps=MRC_WEIGHT_FLOOR, tree=False, zf=False, device=None, stream=None):
    """MRC of Y [N, M] (or [F, D, N, M]) with H [N, M] (or [F, N, M]).
    Returns (s_hat, weights[, zf]) CUDA tensors."""
    dev = require_cuda(device)
    y = as_c64(freq, dev)
    h = as_c64(gains, dev)
    single = y.dim() == 2
    if single:
        y, h = y[None, None], h[None]
    f, d, n, m = y.shape
    if tuple(h.shape) != (f, n, m):
        raise ContractError(f"estimate shape {tuple(h.shape)} does not match symbol {tuple(y.shape)}")
    s_hat = torch.empty((f, d, m), dtype=torch.complex64, device=dev)
    w = torch.empty((f, d, m), dtype=torch.float32, device=dev)
    z = torch.empty((f, d, n, m), dtype=torch.complex64, device=dev) if zf else None
    _lib.call("ofdmrx_mrc", f, d, n, m, ptr(y), d * n * m, n * m, ptr(h), float(eps), int(bool(tree)),
              ptr(s_hat), ptr(w), ptr(z), stream_handle(stream))
    if single:
        s_hat, w = s_hat[0, 0], w[0, 0]
        z = z[0, 0] if z is not None else None
    return (s_hat, w, z) if zf else (s_hat, w)


def demap(symbols, order, device=None, stream=None):
    """qam_demap on the device.  numpy in -> numpy uint8 out."""
    host = not isinstance(symbols, torch.Tensor)
    dev = require_cuda(device)
    s = as_c64(symbols, dev).reshape(-1)
    qb = qam_bits(order)
    bits = torch.empty(s.numel() * qb, dtype=torch.uint8, device=dev)
    _lib.call("ofdmrx_demap", ptr(s), s.numel(), int(order), ptr(bits), stream_handle(stream))
    return bits.cpu().numpy() if host else bits


def raise_on_flags(flags):
    """Host check of per-frame flags (forces a sync): NumericInputError for
    frames that fed non-finite samples to the FFT (receiver.py:202-203)."""
    fl = flags.cpu().numpy() if isinstance(flags, torch.Tensor) else np.asarray(flags)
    bad = np.nonzero(fl & _lib.FLAG_NONFINITE)[0]
    if bad.size:
        raise NumericInputError(
            f"non-finite samples entering the FFT stage (frames {bad[:8].tolist()}"
            f"{'...' if bad.size > 8 else ''})")


def qam_scale(order):
    """waveform.py:138-143."""
    levels = 1 << (int(math.log2(order)) // 2)
    mean = np.mean([(levels - 1 - 2 * i) ** 2 for i in range(levels)])
    return 1.0 / math.sqrt(2.0 * mean)


def check_config(fft_len):
    if fft_len > 4096:
        raise ConfigurationError(f"fft length {fft_len} exceeds the device path limit 4096")
