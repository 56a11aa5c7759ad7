"""Multi-process (gloo, world size 2) checks of the sharding host logic: frame
and antenna partitioning, the partial-sum exchange in both modes, and the
pairwise-tree combine — against the CPU oracle's full-array MRC."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ofdm_oracle as orc
from paper_1901_07499_b200 import sharding


def test_frame_shard_partitions():
    for n in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [sharding.frame_shard(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_antenna_shard_even_split():
    assert sharding.antenna_shard(256, 3, 8) == (96, 128)
    with pytest.raises(Exception):
        sharding.antenna_shard(10, 0, 4)


def test_tree_sum_parts_matches_reference_plan():
    rng = np.random.default_rng(0)
    for g in range(1, 12):
        x = rng.standard_normal((g, 5)) + 1j * rng.standard_normal((g, 5))
        got = sharding.tree_sum_parts(torch.from_numpy(x)).numpy()
        assert np.array_equal(got, orc.tree_reduce_rows(x))


def test_pack_roundtrip():
    num = torch.randn(3, 4, 8, dtype=torch.complex64)
    den = torch.rand(3, 8)
    n2, d2 = sharding.unpack_partials(sharding.pack_partials(num, den), 3, 4, 8)
    assert torch.equal(n2, num) and torch.equal(d2, den)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, cp, n_ant, qam, d = 64, 16, 8, 16, 4
        streams, _, s0 = orc.synth_capture(m, cp, n_ant, qam, d, 5, snr_db=10.0)
        lo, hi = sharding.antenna_shard(n_ant, rank, world)
        # this rank's partial sums, computed with the oracle's stages
        H = orc.ls_divide(orc.freq_transform(streams[lo:hi, s0 + cp: s0 + cp + m]), orc.make_pilot(m))
        Y = np.stack([orc.freq_transform(streams[lo:hi, s0 + (k + 1) * (m + cp) + cp: s0 + (k + 1) * (m + cp) + cp + m])
                      for k in range(d)])
        num, den = sharding.host_partials(Y, H)
        nump, denp = sharding.exchange_partials(torch.from_numpy(num[None]), torch.from_numpy(den[None]), mode)
        if mode == "gather":
            assert nump.shape[0] == world
            num_t = sharding.tree_sum_parts(nump)[0].numpy()
            den_t = sharding.tree_sum_parts(denp)[0].numpy()
        else:
            num_t, den_t = nump[0, 0].numpy(), denp[0, 0].numpy()
        s_hat = num_t / np.maximum(den_t, 1e-12)
        bits = orc.qam_demap(s_hat, qam)
        _, s_ref, w_ref, b_ref = orc.receive_frame(streams, s0, m, cp, d, qam)
        ok = (np.array_equal(bits, b_ref) and np.allclose(s_hat, s_ref, rtol=1e-10, atol=1e-12)
              and np.allclose(den_t, w_ref, rtol=1e-12))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["gather", "allreduce"])
def test_antenna_sharded_exchange_gloo_world2(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in procs)
    assert res == {0: True, 1: True}


def test_scatter_pack_roundtrip():
    num = torch.randn(6, 4, 8, dtype=torch.complex64)
    den = torch.rand(6, 8)
    buf = sharding.scatter_pack(num, den, 3)
    assert buf.shape == (3, 2 * (4 * 8 * 2 + 8))
    n2, d2 = sharding.scatter_unpack(buf, 4, 8)  # as if every row came from a different rank
    assert torch.equal(n2.reshape(6, 4, 8), num) and torch.equal(d2.reshape(6, 8), den)


def _scatter_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, cp, n_ant, qam, d, nf = 64, 16, 8, 16, 4, 4
        caps = [orc.synth_capture(m, cp, n_ant, qam, d, 20 + i, snr_db=10.0) for i in range(nf)]
        s0 = caps[0][2]
        lo, hi = sharding.antenna_shard(n_ant, rank, world)
        nums, dens = [], []
        for streams, _, _ in caps:  # this rank's antenna shard of every frame
            H = orc.ls_divide(orc.freq_transform(streams[lo:hi, s0 + cp: s0 + cp + m]), orc.make_pilot(m))
            Y = np.stack([orc.freq_transform(streams[lo:hi, s0 + (k + 1) * (m + cp) + cp:
                                                     s0 + (k + 1) * (m + cp) + cp + m]) for k in range(d)])
            num, den = sharding.host_partials(Y, H)
            nums.append(num)
            dens.append(den)
        num = torch.from_numpy(np.stack(nums)).to(torch.complex128)
        den = torch.from_numpy(np.stack(dens))
        recv, work = sharding.scatter_partials(num.to(torch.complex64), den.float(), async_op=True)
        work.wait()
        nump, denp = sharding.scatter_unpack(recv, d, m)
        fpo = nf // world
        assert nump.shape == (world, fpo, d, m) and denp.shape == (world, fpo, m)
        ok = True
        for j in range(fpo):
            f = rank * fpo + j
            num_t = sharding.tree_sum_parts(nump[:, j]).numpy().astype(np.complex128)
            den_t = sharding.tree_sum_parts(denp[:, j]).numpy().astype(np.float64)
            s_hat = num_t / np.maximum(den_t, 1e-12)
            _, s_ref, w_ref, b_ref = orc.receive_frame(caps[f][0], s0, m, cp, d, qam)
            ok = ok and np.array_equal(orc.qam_demap(s_hat, qam), b_ref)
            ok = ok and np.linalg.norm(s_hat - s_ref) / np.linalg.norm(s_ref) < 1e-5
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_scatter_exchange_gloo_world2():
    """Mode "scatter": each owner receives every rank's partials of its own
    frames (all-to-all), tree-sums them in rank order and decodes its frames
    exactly as the oracle does."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_scatter_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in procs)
    assert res == {0: True, 1: True}
