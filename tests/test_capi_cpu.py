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
                symbol0_offset=0, row_stride=880, frame_stride=3520)
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
    (dict(options=4), E.ContractError),
])
def test_check_desc_errors(lib, kw, exc):
    with pytest.raises(exc):
        device.check_desc(desc(**kw))


def test_check_desc_bounds_is_framing_error(lib):
    device.check_desc(desc(), 4 * 880)
    with pytest.raises(E.FramingError) as ei:
        device.check_desc(desc(), 4 * 880 - 1)
    assert "needed" in str(ei.value)


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
