"""Antenna-sharded exchange over peer memory (sharding mode "peer",
SURVEY.md §8(e)): two ranks on one GPU (separate processes, CUDA IPC
mappings of each other's inboxes, gloo only for the handle exchange).  The
fused kernel stores the partial sums into the owners' inboxes; flags hand
them over; each owner finishes its frames.  Bits must equal the oracle's,
s_hat within 1e-4, over several back-to-back epochs (inbox reuse)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    from oracle import ofdm_oracle as orc

    m, cp, n_ant, qam, d, nf = 256, 32, 16, 16, 5, 4
    caps = [orc.synth_capture(m, cp, n_ant, qam, d, s, snr_db=10.0) for s in range(nf)]
    return (m, cp, n_ant, qam, d, nf), np.stack([c[0] for c in caps]), caps[0][2]


def _worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import sharding

    try:
        dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
        torch.cuda.set_device(0)
        (m, cp, n_ant, qam, d, nf), streams, s0 = _inputs()
        cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
        rx = sharding.AntennaShardedReceiver(cfg, d, symbol0_offset=s0, mode="peer")
        x = torch.from_numpy(streams[:, rx.ant_lo:rx.ant_hi].astype(np.complex64)).cuda()
        outs = []
        for _ in range(3):  # several epochs through the same inboxes
            s_hat, w, bits, fl, _ = rx.receive(x)
            outs.append((s_hat.cpu().numpy(), w.cpu().numpy(), bits.cpu().numpy(), fl.cpu().numpy()))
        torch.cuda.synchronize()
        rx.close()
        dist.destroy_process_group()
        q.put((rank, outs, None))
    except Exception as exc:  # noqa: BLE001
        import traceback

        q.put((rank, None, traceback.format_exc()))


def test_peer_exchange_two_ranks_one_gpu():
    import multiprocessing as mp

    from oracle import ofdm_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, outs, err = q.get(timeout=300)
        assert err is None, err
        res[rank] = outs
    for p in procs:
        p.join(timeout=60)
    (m, cp, n_ant, qam, d, nf), streams, s0 = _inputs()
    fpo = nf // 2
    for rank in (0, 1):
        for s_hat, w, bits, fl in res[rank]:
            assert not fl.any()
            for i in range(fpo):
                f = rank * fpo + i
                H, s_ref, w_ref, b_ref = orc.receive_frame(streams[f], s0, m, cp, d, qam)
                assert np.array_equal(bits[i], b_ref)
                assert np.linalg.norm(s_hat[i] - s_ref) / np.linalg.norm(s_ref) < 1e-4
                assert np.linalg.norm(w[i] - w_ref) / np.linalg.norm(w_ref) < 1e-4
        # epochs agree bit for bit (deterministic tree over the two slots)
        assert all(np.array_equal(res[rank][0][2], o[2]) for o in res[rank][1:])
