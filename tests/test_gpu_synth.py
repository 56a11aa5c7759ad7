"""Device frame synthesizer (synth.synth_frames) against
the oracle's restatement of waveform.build_frame + channel.apply_channel.

Deterministic stages (QAM map, IFFT + CP, PN preamble, channel response,
timing offset) are compared on noiseless captures with the reference's own
payload bits: within 2e-6 relative (fp32 inverse FFT vs the reference's fp64
radix-2).  The random stages (bits, Rayleigh gains, AWGN) use counter-based
device RNG streams, so they are checked statistically and end to end (sync +
receive decode the synthesized frames)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ofdm_oracle as orc  # noqa: E402

TOL = 2e-6


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.complex128) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def P():
    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import device

    device.require_cuda()
    return P


def ref_bits(m, qam, d, f):
    return np.random.default_rng(f).integers(0, 2, size=d * m * int(np.log2(qam)), dtype=np.uint8)


@pytest.mark.parametrize("m,cp,qam,d", [(64, 16, 4, 10), (256, 32, 16, 4), (1024, 72, 16, 3), (2048, 256, 64, 2),
                                        (8, 1, 16, 5)])
def test_noiseless_identity_matches_oracle_frame(P, m, cp, qam, d):
    from paper_1901_07499_b200 import synth

    cfg = P.OfdmConfig(m, cp, 2, qam_order=qam)
    bits = np.stack([ref_bits(m, qam, d, f) for f in range(3)])
    out = synth.synth_frames(cfg, d, 3, mode="identity", snr_db=None, bits=bits)
    rx = out.rx.cpu().numpy()
    for f in range(3):
        tx, _, nd = orc.build_frame_samples(m, cp, qam, orc.make_pilot(m), bits[f], orc.generate_pn())
        assert nd == d and rx.shape[2] == tx.size
        for a in range(2):
            assert rel(rx[f, a], tx) < TOL
    assert torch.equal(out.bits.cpu(), torch.from_numpy(bits))
    assert out.symbol0_offset == 255


def test_fixed_gains_multipath_and_offset_match_oracle(P):
    from paper_1901_07499_b200 import synth

    m, cp, qam, d, n = 64, 16, 16, 4, 3
    cfg = P.OfdmConfig(m, cp, n, qam_order=qam)
    bits = ref_bits(m, qam, d, 9)[None]
    tx, _, _ = orc.build_frame_samples(m, cp, qam, orc.make_pilot(m), bits[0], orc.generate_pn())
    gains = [0.5 + 0.25j, -1.0 + 0.0j, 0.1 - 2.0j]
    out = synth.synth_frames(cfg, d, 1, mode="fixed_gains", gains=gains, snr_db=None, bits=bits, timing_offset=37)
    ref, _ = orc.apply_channel(tx, n, mode="fixed_gains", gains=gains, timing_offset=37)
    assert rel(out.rx[0].cpu().numpy(), ref) < TOL and out.symbol0_offset == 37 + 255
    taps = np.array([[1.0, 0.3 - 0.2j, 0.05j], [0.7j, 0.0, 0.2], [1.0, 0.0, 0.0]])
    out = synth.synth_frames(cfg, d, 1, mode="multipath", taps=taps, snr_db=None, bits=bits)
    ref, _ = orc.apply_channel(tx, n, mode="multipath", taps=taps)
    assert rel(out.rx[0].cpu().numpy(), ref) < TOL


def test_awgn_power_gain_statistics_and_reproducibility(P):
    from paper_1901_07499_b200 import synth

    m, cp, qam, d, n, F = 256, 32, 16, 4, 8, 64
    cfg = P.OfdmConfig(m, cp, n, qam_order=qam)
    clean = synth.synth_frames(cfg, d, F, mode="flat_rayleigh", snr_db=None, seed=11)
    noisy = synth.synth_frames(cfg, d, F, mode="flat_rayleigh", snr_db=10.0, seed=11)
    assert torch.equal(clean.bits, noisy.bits) and torch.equal(clean.response, noisy.response)
    x, y = clean.rx.to(torch.complex128), noisy.rx.to(torch.complex128)
    p_sig = (x.abs() ** 2).mean(dim=2)
    p_noise = ((y - x).abs() ** 2).mean(dim=2)
    snr = 10 * torch.log10(p_sig / p_noise)
    assert abs(float(snr.mean()) - 10.0) < 0.05 and float(snr.std()) < 0.2
    g = clean.response.reshape(-1).to(torch.complex128)
    assert abs(float((g.abs() ** 2).mean()) - 1.0) < 0.12 and abs(complex(g.mean())) < 0.12
    b = clean.bits.double().mean()
    assert abs(float(b) - 0.5) < 0.01
    again = synth.synth_frames(cfg, d, F, mode="flat_rayleigh", snr_db=10.0, seed=11)
    other = synth.synth_frames(cfg, d, F, mode="flat_rayleigh", snr_db=10.0, seed=12)
    assert torch.equal(again.rx, noisy.rx) and not torch.equal(other.rx, noisy.rx)


def test_synthesized_frames_sync_and_decode(P):
    """Device TX -> device channel (timing offset, Rayleigh, 10 dB) -> device
    PN detection -> fused receive recovers the payload."""
    from paper_1901_07499_b200 import frames, sync, synth

    m, cp, qam, d, n, F = 1024, 72, 16, 10, 16, 32
    cfg = P.OfdmConfig(m, cp, n, qam_order=qam)
    out = synth.synth_frames(cfg, d, F, mode="flat_rayleigh", snr_db=10.0, seed=3, timing_offset=123,
                             n_samples=123 + 255 + 11 * (m + cp) + 50)
    det = sync.detect_frames(out.rx, orc.generate_pn())
    assert bool((det.frame_start == 123).all()) and bool(det.detected.all())
    res = frames.receive_frames(out.rx, cfg, symbol0_offset=int(det.symbol0_offset[0]), n_data=d)
    ber = float((res.bits != out.bits).double().mean())
    # same link on reference-synthesised captures (numpy RNG): BER must agree
    caps = [orc.synth_capture(m, cp, n, qam, d, s, snr_db=10.0) for s in range(4)]
    x = torch.from_numpy(np.stack([c[0] for c in caps]).astype(np.complex64)).cuda()
    r2 = frames.receive_frames(x, cfg, symbol0_offset=caps[0][2], n_data=d)
    ber_ref = float((r2.bits.cpu().numpy() != np.stack([c[1] for c in caps])).mean())
    assert 0.5 < ber / ber_ref < 2.0, (ber, ber_ref)
    # noiseless: exact
    out0 = synth.synth_frames(cfg, d, 4, mode="flat_rayleigh", snr_db=None, seed=4)
    res0 = frames.receive_frames(out0.rx, cfg, symbol0_offset=out0.symbol0_offset, n_data=d)
    assert torch.equal(res0.bits, out0.bits)


def test_bad_arguments(P):
    from paper_1901_07499_b200 import synth
    from paper_1901_07499_b200.errors import ConfigurationError

    cfg = P.OfdmConfig(64, 16, 2)
    with pytest.raises(ConfigurationError):
        synth.synth_frames(cfg, 2, 1, mode="bogus")
    with pytest.raises(ConfigurationError):
        synth.synth_frames(cfg, 2, 1, mode="fixed_gains", gains=[1.0])
    with pytest.raises(ConfigurationError):
        synth.synth_frames(cfg, 2, 1, timing_offset=-1)
