"""Capture-file ingest (paper_1901_07499_b200.ingest): the reference's
rx_meta.txt + rx_ant<k>.cf32 layout (io_formats.py, cli._load_capture) read
straight into one complex64 [N, S] buffer, with the reference's errors."""

import os
import sys

import numpy as np
import pytest

from paper_1901_07499_b200 import OfdmConfig, ingest
from paper_1901_07499_b200.errors import InputError

REF = "/root/reference/pkg/src"


def _streams(n=3, s=517, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))).astype(np.complex64)


def test_roundtrip(tmp_path):
    cfg = OfdmConfig(64, 16, 3, qam_order=16)
    x = _streams()
    ingest.write_capture(str(tmp_path), x, cfg)
    meta, cfg2, st = ingest.load_capture(str(tmp_path), pinned=False)
    assert cfg2 == cfg and meta["format_version"] == "1"
    assert np.array_equal(st.numpy(), x)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")
def test_reads_files_written_by_the_reference_io_layer(tmp_path):
    sys.path.insert(0, REF)
    try:
        from ofdmrx import io_formats
    finally:
        sys.path.remove(REF)
    x = _streams(2, 301, 5).astype(np.complex128)
    for k in range(2):
        io_formats.write_cf32(os.path.join(tmp_path, f"rx_ant{k}.cf32"), x[k])
    io_formats.write_meta(os.path.join(tmp_path, "rx_meta.txt"),
                          {"n_antennas": 2, "fft_len": 64, "cp_len": 16, "qam_order": 4, "pn_len": 255,
                           "sample_rate_hz": 1e7})
    meta, cfg, st = ingest.load_capture(str(tmp_path), pinned=False)
    ref = np.stack([io_formats.read_cf32(os.path.join(tmp_path, f"rx_ant{k}.cf32")) for k in range(2)])
    assert np.array_equal(st.numpy().astype(np.complex128), ref)
    assert cfg.n_antennas == 2 and cfg.fft_len == 64


def test_errors(tmp_path):
    cfg = OfdmConfig(64, 16, 2, qam_order=4)
    with pytest.raises(InputError):
        ingest.load_capture(str(tmp_path), pinned=False)  # no rx_meta.txt
    ingest.write_capture(str(tmp_path), _streams(2, 100), cfg)
    os.remove(os.path.join(tmp_path, "rx_ant1.cf32"))
    with pytest.raises(InputError, match="missing antenna"):
        ingest.load_capture(str(tmp_path), pinned=False)
    np.zeros(202, dtype="<f4").tofile(os.path.join(tmp_path, "rx_ant1.cf32"))  # 101 samples != 100
    with pytest.raises(InputError, match="disagree"):
        ingest.load_capture(str(tmp_path), pinned=False)
    np.zeros(201, dtype="<f4").tofile(os.path.join(tmp_path, "rx_ant0.cf32"))
    np.zeros(201, dtype="<f4").tofile(os.path.join(tmp_path, "rx_ant1.cf32"))
    with pytest.raises(InputError, match="odd float count"):
        ingest.load_capture(str(tmp_path), pinned=False)
    with open(os.path.join(tmp_path, "rx_meta.txt"), "a") as fh:
        fh.write("not a key value line\n")
    with pytest.raises(InputError, match="key=value"):
        ingest.load_capture(str(tmp_path), pinned=False)


def test_load_captures_pads_to_the_longest(tmp_path):
    cfg = OfdmConfig(64, 16, 2, qam_order=4)
    a, b = _streams(2, 300, 1), _streams(2, 340, 2)
    ingest.write_capture(str(tmp_path / "a"), a, cfg)
    ingest.write_capture(str(tmp_path / "b"), b, cfg)
    metas, cfg2, st = ingest.load_captures([str(tmp_path / "a"), str(tmp_path / "b")], pinned=False)
    x = st.numpy()
    assert x.shape == (2, 2, 340) and cfg2 == cfg
    assert np.array_equal(x[0, :, :300], a) and not x[0, :, 300:].any() and np.array_equal(x[1], b)
    ingest.write_capture(str(tmp_path / "c"), _streams(2, 300, 3), OfdmConfig(128, 16, 2, qam_order=4))
    with pytest.raises(InputError, match="disagree on the configuration"):
        ingest.load_captures([str(tmp_path / "a"), str(tmp_path / "c")], pinned=False)
