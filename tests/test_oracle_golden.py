"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py, reference numpy backend).  Bit equality is
required wherever the oracle restates the same numpy operations."""

import hashlib
import os

import numpy as np
import pytest

from oracle import ofdm_oracle as orc


@pytest.fixture(scope="module")
def unit(golden_dir):
    return dict(np.load(os.path.join(golden_dir, "unit_vectors.npz")))


@pytest.mark.parametrize("n", [2, 64, 1024])
def test_fft_rows_bit_exact(unit, n):
    x = unit[f"fft_in_{n}"]
    y = orc.fft_rows(x)
    assert np.array_equal(y, unit[f"fft_out_{n}"])
    assert np.array_equal(orc.fft_rows(y, inverse=True), unit[f"ifft_out_{n}"])
    for r in range(x.shape[0]):  # reference test_kernels.py:27-35 bound
        assert np.max(np.abs(y[r] - orc.dft_direct(x[r]))) < 1e-9


def test_fftshift_example(unit):
    assert np.array_equal(orc.fftshift(unit["shift_in"]), unit["shift_out"])
    assert np.array_equal(orc.fftshift(np.arange(4)), [2, 3, 0, 1])


@pytest.mark.parametrize("rows", [1, 2, 5, 16])
def test_tree_reduce_bit_exact(unit, rows):
    assert np.array_equal(orc.tree_reduce_rows(unit[f"tree_in_{rows}"]), unit[f"tree_out_{rows}"])


@pytest.mark.parametrize("rows", [1, 3, 16, 64])
def test_mrc_bit_exact(unit, rows):
    y, h = unit[f"mrc_y_{rows}"], unit[f"mrc_h_{rows}"]
    s, w = orc.mrc_seq(y, h)
    assert np.array_equal(s, unit[f"mrc_seq_s_{rows}"]) and np.array_equal(w, unit[f"mrc_seq_w_{rows}"])
    s, w = orc.mrc_tree(y, h)
    assert np.array_equal(s, unit[f"mrc_tree_s_{rows}"]) and np.array_equal(w, unit[f"mrc_tree_w_{rows}"])


@pytest.mark.parametrize("order", [4, 16, 64])
def test_demap_and_constellation(unit, order):
    assert np.array_equal(orc.qam_demap(unit["demap_in"], order), unit[f"demap_out_{order}"])
    assert np.array_equal(orc.build_constellation(order)[0], unit[f"const_{order}"])


def test_pilot_pn_and_modulate(unit):
    for m in (64, 256, 1024, 2048):
        assert np.array_equal(orc.make_pilot(m), unit[f"pilot_{m}"])
    assert np.array_equal(orc.generate_pn(), unit["pn"])
    assert np.array_equal(orc.ofdm_modulate(orc.make_pilot(64), 16)[0], unit["pilot_symbol_64"])


FRAME_SETS = ["C1", "C1_0dB", "C2", "C3", "C3_0dB", "C4", "C4_0dB"]


@pytest.mark.parametrize("name", FRAME_SETS)
def test_frames_bit_exact(golden_dir, name):
    g = dict(np.load(os.path.join(golden_dir, f"frames_{name}.npz")))
    n_ant, m, cp, qam, d = (int(v) for v in g["spec"])
    for f in g["seeds"]:
        tag = f"f{int(f)}"
        streams, bits, s0 = orc.synth_capture(m, cp, n_ant, qam, d, int(f), snr_db=float(g["snr_db"]))
        assert hashlib.sha256(streams.tobytes()).digest() == g[f"{tag}_rx_sha256"].tobytes()
        assert np.array_equal(np.packbits(bits), g[f"{tag}_tx_bits"])
        H, s_hat, w, out_bits = orc.receive_frame(streams, s0, m, cp, d, qam)
        assert np.array_equal(np.packbits(out_bits), g[f"{tag}_bits"])
        assert np.array_equal(w, g[f"{tag}_weights"])
        if f"{tag}_H" in g:
            assert np.array_equal(H, g[f"{tag}_H"])
            assert np.array_equal(s_hat, g[f"{tag}_s_hat"])
            _, s_tree, _, bits_tree = orc.receive_frame(streams, s0, m, cp, d, qam, order="tree")
            assert np.array_equal(s_tree, g[f"{tag}_s_hat_tree"])
            assert np.array_equal(np.packbits(bits_tree), g[f"{tag}_bits_tree"])
        else:
            rows = g[f"{tag}_H_rows"]
            assert np.array_equal(H[rows].astype(np.complex64), g[f"{tag}_H_sub"])
            assert np.array_equal(s_hat.astype(np.complex64), g[f"{tag}_s_hat"])
        assert np.allclose(np.linalg.norm(H, axis=1), g[f"{tag}_H_norm"], rtol=0, atol=0)


@pytest.fixture(scope="module")
def sync(golden_dir):
    return dict(np.load(os.path.join(golden_dir, "sync_vectors.npz")))


def test_corr_metrics_bit_exact(sync):
    assert np.array_equal(orc.corr_metrics(sync["corr_stream"], sync["corr_chips"]), sync["corr_out"])
    emb = orc.corr_metrics(sync["emb_stream"], sync["emb_chips"])
    assert np.array_equal(emb, sync["emb_out"])
    assert int(np.argmax(emb)) == 300


@pytest.mark.parametrize("case", orc.SYNC_CASES, ids=lambda c: c[0])
def test_detect_packet_bit_exact(sync, case):
    name = case[0]
    streams = orc.sync_capture(*case[1:])
    assert hashlib.sha256(streams.tobytes()).digest() == sync[f"{name}_sha256"].tobytes()
    det, start, s0, peak, peaks = orc.detect_packet(streams, orc.generate_pn())
    assert np.array_equal([p[0] for p in peaks], sync[f"{name}_peaks"])
    assert np.array_equal([p[1] for p in peaks], sync[f"{name}_metrics"])
    assert det == bool(sync[f"{name}_detected"]) and s0 == start + 255


def test_noise_only_detection_bit_exact(sync):
    pn = orc.generate_pn()
    for i, row in enumerate(sync["noise_streams"]):
        det, start, _, peak, _ = orc.detect_packet(row[None, :], pn)
        assert start == sync["noise_peaks"][i] and peak == sync["noise_metrics"][i] and not det
