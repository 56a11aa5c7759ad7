"""Capture files -> (pinned) host memory, the front of the ingest path
(SURVEY.md §8(f) #2).

Mirrors the reference's file layer for received captures:
``io_formats.read_cf32`` / ``read_meta`` (io_formats.py:26-30,72-89) and
``cli._load_capture`` (cli.py:249-271): a directory holds ``rx_meta.txt``
(``key=value`` lines with ``format_version``, ``n_antennas``, ``fft_len``,
``cp_len``, ``qam_order``, ``pn_len``, ``sample_rate_hz``) and one
``rx_ant<k>.cf32`` file per antenna (little-endian interleaved float32 I/Q).
Same errors (InputError for a missing meta file or antenna file, an odd float
count, antennas of different lengths, a malformed meta line).

Differences by design: samples stay complex64 (the device path's cf32) and
are read straight into one [N, S] buffer - page-locked when ``pinned`` - so
``ofdmrx_stage_symbols`` / ``frames.StreamingReceiver`` can DMA them to the
GPU without an extra host copy."""

import os

import numpy as np

from .errors import InputError
from .waveform import OfdmConfig


def read_meta(path):
    """io_formats.read_meta (io_formats.py:72-89)."""
    entries = {}
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, 1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if "=" not in line:
                raise InputError(f"{path}:{lineno}: expected key=value, got {line!r}")
            key, value = line.split("=", 1)
            entries[key.strip()] = value.strip()
    if "format_version" not in entries:
        raise InputError(f"{path}: missing format_version")
    return entries


def _alloc(shape, pinned):
    import torch

    return torch.empty(shape, dtype=torch.complex64, pin_memory=bool(pinned))


def _read_into(path, dst):
    """Interleaved <f4 I/Q of `path` into the complex64 row `dst` (numpy view)."""
    nbytes = os.path.getsize(path)
    if nbytes % 8:
        raise InputError(f"{path}: odd float count, not interleaved I/Q")  # io_formats.py:28-29
    if nbytes != dst.nbytes:
        raise InputError(f"{path}: {nbytes // 8} samples, expected {dst.size}")
    with open(path, "rb") as fh:
        got = fh.readinto(memoryview(dst.view(np.uint8)))
    if got != nbytes:
        raise InputError(f"{path}: short read ({got} of {nbytes} bytes)")


def capture_files(in_dir, n_antennas):
    return [os.path.join(in_dir, f"rx_ant{k}.cf32") for k in range(n_antennas)]


def load_capture(in_dir, pinned=True):
    """cli._load_capture (cli.py:249-271) -> (meta, OfdmConfig, streams).

    streams: torch complex64 [N, S] (page-locked when ``pinned``)."""
    meta_path = os.path.join(in_dir, "rx_meta.txt")
    if not os.path.exists(meta_path):
        raise InputError(f"missing {meta_path}")
    meta = read_meta(meta_path)
    n_antennas = int(meta["n_antennas"])
    cfg = OfdmConfig(int(meta["fft_len"]), int(meta["cp_len"]), n_antennas, int(meta["qam_order"]),
                     pn_len=int(meta["pn_len"]), sample_rate_hz=float(meta["sample_rate_hz"]))
    files = capture_files(in_dir, n_antennas)
    missing = [p for p in files if not os.path.exists(p)]
    if missing:
        raise InputError("missing antenna files: " + ", ".join(missing))
    sizes = {os.path.getsize(p) for p in files}
    if len(sizes) != 1:
        raise InputError(f"antenna files disagree on length: {sorted(s // 8 for s in sizes)}")
    s = sizes.pop() // 8
    streams = _alloc((n_antennas, s), pinned)
    view = streams.numpy()
    for k, p in enumerate(files):
        _read_into(p, view[k])
    return meta, cfg, streams


def load_captures(in_dirs, pinned=True):
    """Several capture directories of one configuration -> (metas, cfg,
    streams [F, N, S]) in one (pinned) buffer, the batch layout of
    frames.receive_frames / receive_captures / StreamingReceiver.  Captures
    of different lengths are zero-padded to the longest (the tail beyond a
    capture is never a valid symbol window: ofdmrx_rx_frames_detected flags
    frames that would need it)."""
    metas, cfgs, lens = [], [], []
    for d in in_dirs:
        meta_path = os.path.join(d, "rx_meta.txt")
        if not os.path.exists(meta_path):
            raise InputError(f"missing {meta_path}")
        meta = read_meta(meta_path)
        n = int(meta["n_antennas"])
        files = capture_files(d, n)
        missing = [p for p in files if not os.path.exists(p)]
        if missing:
            raise InputError("missing antenna files: " + ", ".join(missing))
        sizes = {os.path.getsize(p) for p in files}
        if len(sizes) != 1:
            raise InputError(f"antenna files disagree on length: {sorted(s // 8 for s in sizes)}")
        metas.append(meta)
        cfgs.append((int(meta["fft_len"]), int(meta["cp_len"]), n, int(meta["qam_order"]), int(meta["pn_len"])))
        lens.append(sizes.pop())
    if len(set(cfgs)) != 1:
        raise InputError(f"captures disagree on the configuration: {sorted(set(cfgs))}")
    m, cp, n, q, pn = cfgs[0]
    cfg = OfdmConfig(m, cp, n, q, pn_len=pn, sample_rate_hz=float(metas[0]["sample_rate_hz"]))
    if any(length % 8 for length in lens):
        raise InputError("odd float count, not interleaved I/Q")
    s = max(lens) // 8
    streams = _alloc((len(in_dirs), n, s), pinned)
    view = streams.numpy()
    for f, d in enumerate(in_dirs):
        view[f, :, lens[f] // 8:] = 0
        for k, p in enumerate(capture_files(d, n)):
            _read_into(p, view[f, k, :lens[f] // 8])
    return metas, cfg, streams


def write_capture(out_dir, streams, cfg, extra=None):
    """Write a capture directory in the reference layout (io_formats.write_cf32
    + write_meta, io_formats.py:18-23,59-69; cli.py:219-234): for tests and
    tools."""
    os.makedirs(out_dir, exist_ok=True)
    x = np.asarray(streams)
    for k in range(x.shape[0]):
        inter = np.empty(2 * x.shape[1], dtype="<f4")
        inter[0::2] = x[k].real
        inter[1::2] = x[k].imag
        inter.tofile(os.path.join(out_dir, f"rx_ant{k}.cf32"))
    meta = {"n_antennas": cfg.n_antennas, "fft_len": cfg.fft_len, "cp_len": cfg.cp_len,
            "qam_order": cfg.qam_order, "pn_len": cfg.pn_len, "sample_rate_hz": repr(float(cfg.sample_rate_hz))}
    meta.update(extra or {})
    with open(os.path.join(out_dir, "rx_meta.txt"), "w", encoding="utf-8") as fh:
        fh.write("format_version=1\n")
        for k, v in meta.items():
            fh.write(f"{k}={v}\n")
