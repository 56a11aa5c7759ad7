"""The device antenna-sharded receive (SURVEY.md §8(e), C4's split) with two
ranks on one GPU: each rank runs the fused partial-sum kernel on its antenna
half, the partials are exchanged (gloo: staged through host memory; NCCL on a
multi-GPU box moves them device to device), and the finish kernel combines
them in rank order.  Modes "gather" (every rank finishes every frame) and
"scatter" (all-to-all, each rank finishes its own frames, chunked so the
exchange of chunk i overlaps chunk i+1's kernel).  Bits must equal the
oracle's, s_hat within 1e-4."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

SHAPE = (256, 32, 16, 16, 6, 8)  # M, CP, N, QAM, D, frames


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    from oracle import ofdm_oracle as orc

    m, cp, n, qam, d, nf = SHAPE
    caps = [orc.synth_capture(m, cp, n, qam, d, 40 + i, snr_db=10.0) for i in range(nf)]
    return np.stack([c[0] for c in caps]), caps[0][2]


def _worker(rank, world, port, mode, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import sharding

    try:
        dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
        torch.cuda.set_device(0)
        m, cp, n, qam, d, nf = SHAPE
        streams, s0 = _inputs()
        cfg = P.OfdmConfig(m, cp, n, qam_order=qam)
        rx = sharding.AntennaShardedReceiver(cfg, d, symbol0_offset=s0, mode=mode,
                                             chunk_frames=4 if mode == "scatter" else None)
        x = torch.from_numpy(streams[:, rx.ant_lo:rx.ant_hi].astype(np.complex64)).cuda()
        s_hat, w, bits, fl, _ = rx.receive(x)
        torch.cuda.synchronize()
        owned = rx.owned_frames(nf) if mode == "scatter" else list(range(nf))
        q.put((rank, (owned, s_hat.cpu().numpy(), w.cpu().numpy(), bits.cpu().numpy(), fl.cpu().numpy()), None))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("mode", ["gather", "scatter"])
def test_device_antenna_sharded_two_ranks(mode):
    import multiprocessing as mp

    from oracle import ofdm_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, out, err = q.get(timeout=300)
        assert err is None, err
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
    m, cp, n, qam, d, nf = SHAPE
    streams, s0 = _inputs()
    seen = []
    for rank in (0, 1):
        owned, s_hat, w, bits, fl = res[rank]
        assert len(owned) == bits.shape[0] and not fl.any()
        seen += owned
        for i, f in enumerate(owned):
            _, s_ref, w_ref, b_ref = orc.receive_frame(streams[f], s0, m, cp, d, qam)
            assert np.array_equal(bits[i], b_ref), (rank, f)
            assert np.linalg.norm(s_hat[i] - s_ref) / np.linalg.norm(s_ref) < 1e-4
            assert np.linalg.norm(w[i] - w_ref) / np.linalg.norm(w_ref) < 1e-4
    if mode == "scatter":  # every frame finished exactly once
        assert sorted(seen) == list(range(nf))
    else:  # gather: both ranks hold every frame, bit-identical
        assert np.array_equal(res[0][3], res[1][3]) and np.array_equal(res[0][1], res[1][1])
