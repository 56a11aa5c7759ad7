"""CPU-side checks of the C ABI: the library builds, loads without a GPU,
exports exactly what include/ofdmrx_b200.h declares, and its host-side
validation maps onto the reference exception taxonomy (errors.py)."""

import ctypes
import os
import re

import pytest

from paper_1901_07499_b200 import _lib, device
from paper_1901_07499_b200 import errors as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1901_07499_b200 import build

    build.build()
    return _lib.load()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ofdmrx_b200.h")).read()
    return set(re.findall(r"OFDMRX_API\s+[\w\s\*]+?\b(ofdmrx_\w+)\s*\(", text))


def test_exports_match_header(lib):
    declared = header_symbols()
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.ofdmrx_abi_version() == _lib.ABI_VERSION


def desc(**kw):
    base = dict(n_frames=1, n_antennas=4, fft_len=64, cp_len=16, n_data=10, qam_order=4,
                symbol0_offset=0, row_stride=880, frame_stride=3520, rx_samples=4 * 880)
    base.update(kw)
    return device.make_desc(**base)


@pytest.mark.parametrize("kw,exc", [
    (dict(fft_len=100), E.ConfigurationError),
    (dict(fft_len=8192), E.ConfigurationError),
    (dict(cp_len=64), E.ConfigurationError),
    (dict(cp_len=-1), E.ConfigurationError),
    (dict(n_antennas=0), E.ConfigurationError),
    (dict(qam_order=8), E.ConfigurationError),
    (dict(n_data=-1), E.ContractError),
    (dict(row_stride=100), E.ContractError),
    (dict(options=8), E.ContractError),
    (dict(rx_samples=-1), E.ContractError),
])
def test_check_desc_errors(lib, kw, exc):
    with pytest.raises(exc):
        device.check_desc(desc(**kw))


def test_check_desc_bounds_is_input_error(lib):
    """extract_slots' short-capture check (receiver.py:278-283) raises
    InputError; the C ABI bounds-checks against desc.rx_samples (ABI 2)."""
    device.check_desc(desc())
    with pytest.raises(E.InputError) as ei:
        device.check_desc(desc(rx_samples=4 * 880 - 1))
    assert "needed" in str(ei.value)
    # a later frame / antenna row / offset beyond the buffer is caught too
    with pytest.raises(E.InputError):
        device.check_desc(desc(n_frames=2, rx_samples=3520 + 3 * 880 - 1))
    with pytest.raises(E.InputError):
        device.check_desc(desc(n_antennas=1, symbol0_offset=1, rx_samples=880))


def test_short_capture_rejected_before_any_device_access(lib):
    """A raw C caller with a short buffer gets OFDMRX_ERR_INPUT from every
    capture-reading entry point, never an out-of-bounds TMA read."""
    d = desc(rx_samples=4 * 880 - 1)
    dummy = ctypes.c_void_p(0x10000)  # never dereferenced: validation fails first
    assert lib.ofdmrx_rx_frames(ctypes.byref(d), dummy, dummy, None, dummy, None, dummy, None, None,
                                None) == _lib.ERR_INPUT
    assert lib.ofdmrx_rx_partials(ctypes.byref(d), dummy, dummy, None, dummy, dummy, None, None) == _lib.ERR_INPUT
    assert lib.ofdmrx_fft_shift(ctypes.byref(d), 0, 11, dummy, dummy, None) == _lib.ERR_INPUT
    assert lib.ofdmrx_stage_symbols(ctypes.byref(d), dummy, dummy, None) == _lib.ERR_INPUT
    assert lib.ofdmrx_rx_partials_routed(ctypes.byref(d), dummy, dummy, None, dummy, dummy, 1, 0, None,
                                         None) == _lib.ERR_INPUT
    dd = desc(row_stride=1000, frame_stride=4000, rx_samples=4 * 1000 - 1)
    assert lib.ofdmrx_rx_frames_detected(ctypes.byref(dd), 1000, dummy, dummy, 1, 255, 0.6, dummy, dummy, None,
                                         dummy, None, dummy, None, dummy, None) == _lib.ERR_INPUT
    with pytest.raises(E.InputError):
        _lib.check(_lib.ERR_INPUT)


def test_entry_points_validate_before_touching_the_device(lib):
    d = desc(fft_len=48)
    rc = lib.ofdmrx_rx_frames(ctypes.byref(d), None, None, None, None, None, None, None, None, None)
    assert rc == _lib.ERR_CONFIG and "power of two" in _lib.last_error()
    d = desc()
    rc = lib.ofdmrx_rx_frames(ctypes.byref(d), None, None, None, None, None, None, None, None, None)
    assert rc == _lib.ERR_CONTRACT and "rx is NULL" in _lib.last_error()
    assert lib.ofdmrx_demap(None, 10, 32, None, None) == _lib.ERR_CONFIG
    assert lib.ofdmrx_mrc(1, 1, 1, 64, None, 0, 0, None, 1e-12, 2, None, None, None, None) == _lib.ERR_CONFIG
    assert lib.ofdmrx_mrc_finish(1, 1, 64, 4, 0, None, None, 1e-12, None, None, None, None, None) == _lib.ERR_CONTRACT


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(E.DeviceError):
        device.require_cuda()
