"""Multi-GPU distribution of the receive path.

* Frame sharding ("DP" analogue): frames are independent (each carries its own
  pilot and H), so F frames are split contiguously over the ranks and each GPU
  runs the fused kernel on its slice.  There is no collective on the data path.
* Antenna sharding (for arrays too large for one GPU's frame budget, C4 =
  256 antennas): every rank FFTs and LS-estimates its contiguous antenna shard
  of the same frames, producing the un-normalised MRC partial sums
  num[F,D,M] = sum_n conj(H_n) Y_n and den[F,M] = sum_n |H_n|^2
  (frames.receive_partials); one exchange step combines them, then each rank
  divides and demaps (frames.finish_partials).  Two exchange modes:
    - "gather": all-gather of the partials and a fixed-order pairwise tree over
      ranks inside the finish kernel — deterministic, bit-identical on every
      rank and matching the reference ReductionPlan order over shards
      (numerics.py:85-106) when the shard size is a power of two;
    - "allreduce": one NCCL sum all-reduce of the packed partials (half the
      bytes on the wire, association order left to NCCL).
    - "scatter": reduce-scatter shaped.  Rank o owns frames [o F/G, (o+1) F/G)
      of every chunk; one all-to-all sends each owner the partials of its
      frames (each rank receives F/G x G partial sets instead of F x G), the
      owner runs the same rank-ordered pairwise tree over them and finishes
      only its frames.  Chunked: the exchange of chunk i runs on NCCL's stream
      while chunk i+1's partial-sum kernel runs (AntennaShardedReceiver
      chunk_frames).
    - "peer": no collective on the data path.  Each rank owns F/G frames; the
      fused partial-sum kernel stores every frame's (num, den) straight into
      the owner's inbox over peer memory (CUDA IPC mappings: NVLink stores
      between GPUs), release/acquire flags hand the inbox to its owner, which
      runs the same pairwise-tree finish over the G slots (PeerExchange).
      Each rank returns its own F/G frames (reduce-scatter semantics).
  "gather"/"allreduce" only use torch.distributed collectives, so they run
  unchanged on the gloo backend for the CPU tests; "peer" uses
  torch.distributed only once, to exchange the 64-byte IPC handles.
"""

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigurationError, ContractError

EXCHANGE_MODES = ("gather", "allreduce", "scatter", "peer")


def frame_shard(n_frames, rank, world):
    """Contiguous [start, stop) of the frames owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ContractError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def antenna_shard(n_antennas, rank, world):
    """Contiguous antenna range of `rank`; requires an even split so that every
    shard's partial sums cover the same number of antennas."""
    if n_antennas % world:
        raise ConfigurationError(f"{n_antennas} antennas do not split evenly over {world} ranks")
    per = n_antennas // world
    return rank * per, (rank + 1) * per


def pack_partials(num, den):
    """[F,D,M] complex64 + [F,M] float32 -> one flat float32 buffer (one collective)."""
    return torch.cat([torch.view_as_real(num).reshape(-1), den.reshape(-1)])


def unpack_partials(buf, n_frames, n_data, fft_len):
    nn = n_frames * n_data * fft_len * 2
    num = torch.view_as_complex(buf[..., :nn].reshape(buf.shape[:-1] + (n_frames, n_data, fft_len, 2)).contiguous())
    den = buf[..., nn:].reshape(buf.shape[:-1] + (n_frames, fft_len))
    return num, den


def _host_staged(t, group):
    """gloo moves CPU tensors only: device buffers go through host memory
    (the multi-process code-path tests on one GPU); NCCL takes them as is."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def exchange_partials(num, den, mode="gather", group=None):
    """Combine the antenna shards' partial sums across the process group.

    mode="gather": returns ([G,F,D,M], [G,F,M]) stacked partials of all ranks
    (rank order) for the deterministic tree in the finish kernel.
    mode="allreduce": returns ([1,F,D,M], [1,F,M]) summed partials."""
    if mode not in EXCHANGE_MODES:
        raise ConfigurationError(f"exchange mode must be one of {EXCHANGE_MODES}")
    f, d, m = num.shape
    buf = pack_partials(num, den)
    world = dist.get_world_size(group)
    if _host_staged(buf, group):
        n, dd = exchange_partials(num.cpu(), den.cpu(), mode, group)
        return n.to(num.device), dd.to(num.device)
    if mode == "allreduce":
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        n, dd = unpack_partials(buf, f, d, m)
        return n[None], dd[None]
    if buf.is_cuda:
        out = torch.empty((world,) + tuple(buf.shape), dtype=buf.dtype, device=buf.device)
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        out = torch.stack(parts)
    return unpack_partials(out, f, d, m)


def scatter_pack(num, den, world):
    """[F,D,M] c64 + [F,M] f32 -> [G, F/G * (2DM + M)] f32: row o holds the
    partials of owner o's contiguous frame block (the all-to-all send buffer)."""
    f, d, m = num.shape
    if f % world:
        raise ConfigurationError(f"{f} frames do not split evenly over {world} owners")
    return torch.cat([torch.view_as_real(num).reshape(world, -1), den.reshape(world, -1)], dim=1).contiguous()


def scatter_unpack(recv, n_data, fft_len):
    """Inverse of scatter_pack on the receive side: [G, fpo*(2DM+M)] ->
    (num [G, fpo, D, M], den [G, fpo, M]), row g = rank g's partials."""
    g = recv.shape[0]
    per = 2 * n_data * fft_len + fft_len
    fpo = recv.shape[1] // per
    nn = fpo * n_data * fft_len * 2
    num = torch.view_as_complex(recv[:, :nn].reshape(g, fpo, n_data, fft_len, 2).contiguous())
    den = recv[:, nn:].reshape(g, fpo, fft_len)
    return num, den


def scatter_partials(num, den, group=None, async_op=False):
    """Reduce-scatter shaped exchange (mode "scatter"): all-to-all of the
    owner blocks.  Returns (recv [G, fpo*(2DM+M)], work) -- recv row g holds
    rank g's partial sums of this rank's frames (scatter_unpack)."""
    world = dist.get_world_size(group)
    send = scatter_pack(num, den, world)
    if _host_staged(send, group):
        recv = torch.empty_like(send, device="cpu")
        dist.all_to_all_single(recv, send.cpu(), group=group)
        return recv.to(send.device), None
    recv = torch.empty_like(send)
    work = dist.all_to_all_single(recv, send, group=group, async_op=async_op)
    return recv, work


def tree_sum_parts(x):
    """Reference pairwise tree over axis 0 (numerics.ReductionPlan order); the
    host twin of the finish kernel's reduction, used by the CPU tests."""
    acc = x
    while acc.shape[0] > 1:
        cnt = acc.shape[0]
        half = cnt // 2
        merged = acc[0:2 * half:2] + acc[1:2 * half:2]
        if cnt % 2:
            merged = torch.cat([merged, acc[-1:]], dim=0)
        acc = merged
    return acc[0]


class PeerExchange:
    """Inboxes and flags of the peer-memory exchange for one rank.

    Inbox of rank r (one ofdmrx_peer_alloc allocation, zero-initialised):
      num [G, fpo, D, M] cf32 | den [G, fpo, M] f32 | ready [G] u64 | consumed u64
    slot g of num/den holds producer g's partial sums of r's frames; ready[g]
    is producer g's epoch flag; consumed is r's "inbox read" epoch."""

    def __init__(self, n_frames, n_data, fft_len, group=None, device=None):
        import ctypes

        from . import _lib
        from . import device as dv

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if n_frames % self.world:
            raise ConfigurationError(f"{n_frames} frames do not split evenly over {self.world} owners")
        self.fpo = n_frames // self.world
        self.n_frames, self.n_data, self.fft_len = n_frames, n_data, fft_len
        g, fpo, d, m = self.world, self.fpo, n_data, fft_len
        self.num_bytes = g * fpo * d * m * 8
        self.den_off = self.num_bytes
        self.ready_off = (self.den_off + g * fpo * m * 4 + 15) // 16 * 16
        self.consumed_off = self.ready_off + 8 * g
        nbytes = self.consumed_off + 64
        self.dev = dv.require_cuda(device)
        lib = _lib.load()
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        _lib.check(lib.ofdmrx_peer_alloc(nbytes, ctypes.byref(ptr), handle))
        self.own = ptr.value
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=group)
        self.bases, self.opened = [], []
        for r, h in enumerate(handles):
            if r == self.rank:
                self.bases.append(self.own)
                continue
            q = ctypes.c_void_p()
            _lib.check(lib.ofdmrx_peer_open(ctypes.create_string_buffer(h, 64), ctypes.byref(q)))
            self.bases.append(q.value)
            self.opened.append(q.value)
        b = self.bases
        tab = lambda xs: torch.tensor(xs, dtype=torch.int64, device=self.dev)  # noqa: E731
        self.num_dst = tab(b)
        self.den_dst = tab([x + self.den_off for x in b])
        self.ready_dst = tab([x + self.ready_off + 8 * self.rank for x in b])  # my flag at every owner
        self.ready_src = tab([self.own + self.ready_off + 8 * i for i in range(g)])  # producers' flags here
        self.consumed_src = tab([x + self.consumed_off for x in b])
        self.consumed_dst = tab([self.own + self.consumed_off])
        self.epoch = 0
        self.group = group

    def inbox(self):
        """(num [G, fpo, D, M], den [G, fpo, M]) views of this rank's inbox as
        raw pointers for ofdmrx_mrc_finish."""
        return self.own, self.own + self.den_off

    def close(self):
        from . import _lib

        lib = _lib.load()
        for q in self.opened:
            lib.ofdmrx_peer_close(ctypes_void(q))
        self.opened = []
        if self.own:
            lib.ofdmrx_peer_free(ctypes_void(self.own))
            self.own = None


def ctypes_void(v):
    import ctypes

    return ctypes.c_void_p(int(v))


class AntennaShardedReceiver:
    """Antenna-sharded fused receive for one rank of a process group.

    receive(rx_shard) takes this rank's antenna rows [F, N/G, S] of the frames
    and returns (s_hat, weights, bits, flags, H) for all F frames on every rank
    (modes "gather" / "allreduce") or for the frames this rank owns (modes
    "scatter" / "peer": owned_frames(F))."""

    def __init__(self, cfg, n_data, symbol0_offset=0, pilot=None, mode="gather", group=None, chunk_frames=None):
        from .waveform import OfdmConfig

        if mode not in EXCHANGE_MODES:
            raise ConfigurationError(f"exchange mode must be one of {EXCHANGE_MODES}")
        self.cfg = cfg
        self.n_data = n_data
        self.symbol0_offset = symbol0_offset
        self.pilot = pilot
        self.mode = mode
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ant_lo, self.ant_hi = antenna_shard(cfg.n_antennas, self.rank, self.world)
        self.chunk_frames = chunk_frames
        self.shard_cfg = OfdmConfig(cfg.fft_len, cfg.cp_len, self.ant_hi - self.ant_lo, qam_order=cfg.qam_order,
                                    pn_len=cfg.pn_len)
        self.peer = None

    def receive(self, rx_shard, want_h=False, stream=None):
        from . import frames

        if self.mode == "peer":
            return self._receive_peer(rx_shard, want_h, stream)
        if self.mode == "scatter":
            return self._receive_scatter(rx_shard, want_h)
        H, num, den, flags = frames.receive_partials(rx_shard, self.shard_cfg, self.pilot,
                                                     symbol0_offset=self.symbol0_offset, n_data=self.n_data,
                                                     want_h=want_h, stream=stream)
        nump, denp = exchange_partials(num, den, self.mode, self.group)
        s_hat, weights, bits, fflags = frames.finish_partials(nump, denp, self.cfg.qam_order, stream=stream)
        return s_hat, weights, bits, fflags | flags, H

    def _receive_peer(self, rx_shard, want_h, stream):
        """Fused partials -> owners' inboxes (peer stores) -> flags -> finish of
        the own frames.  Returns (s_hat, weights, bits, flags, H) for frames
        [rank * F/G, (rank + 1) * F/G)."""
        import ctypes

        from . import _lib, device as dv, frames

        x = dv.as_c64(rx_shard, dv.require_cuda(rx_shard.device if isinstance(rx_shard, torch.Tensor) else None))
        if x.dim() == 2:
            x = x[None]
        f, n, s = x.shape
        ex = self.peer
        if ex is None or ex.n_frames != f:
            if ex is not None:
                ex.close()
            ex = self.peer = PeerExchange(f, self.n_data, self.cfg.fft_len, self.group, x.device)
        ex.epoch += 1
        e = ex.epoch
        st = dv.stream_handle(stream)
        g, m, d = ex.world, self.cfg.fft_len, self.n_data
        lib = _lib.load()
        # owners have read epoch e-1 from their inboxes
        _lib.check(lib.ofdmrx_peer_wait(dv.ptr(ex.consumed_src), g, e - 1, st))
        pvals = frames._pilot_values(self.pilot, m)
        desc = dv.make_desc(f, n, m, self.cfg.cp_len, d, self.cfg.qam_order, self.symbol0_offset, s, n * s,
                            options=dv.pilot_options(pvals), rx_samples=x.numel())
        H = torch.empty((f, n, m), dtype=torch.complex64, device=x.device) if want_h else None
        flags = torch.zeros((f,), dtype=torch.int32, device=x.device)
        pv = frames._PILOTS.get(pvals, x.device)
        _lib.call("ofdmrx_rx_partials_routed", ctypes.byref(desc), dv.ptr(x), dv.ptr(pv), dv.ptr(H),
                  dv.ptr(ex.num_dst), dv.ptr(ex.den_dst), ex.fpo, ex.rank, dv.ptr(flags), st)
        _lib.check(lib.ofdmrx_peer_signal(dv.ptr(ex.ready_dst), g, e, st))
        _lib.check(lib.ofdmrx_peer_wait(dv.ptr(ex.ready_src), g, e, st))
        qb = dv.qam_bits(self.cfg.qam_order)
        fo = ex.fpo
        s_hat = torch.empty((fo, d, m), dtype=torch.complex64, device=x.device)
        weights = torch.empty((fo, m), dtype=torch.float32, device=x.device)
        bits = torch.empty((fo, d * m * qb), dtype=torch.uint8, device=x.device)
        fflags = torch.zeros((fo,), dtype=torch.int32, device=x.device)
        num_p, den_p = ex.inbox()
        _lib.call("ofdmrx_mrc_finish", fo, d, m, int(self.cfg.qam_order), g, ctypes_void(num_p), ctypes_void(den_p),
                  float(dv.MRC_WEIGHT_FLOOR), dv.ptr(s_hat), dv.ptr(weights), dv.ptr(bits), dv.ptr(fflags), st)
        _lib.check(lib.ofdmrx_peer_signal(dv.ptr(ex.consumed_dst), 1, e, st))
        own = slice(ex.rank * fo, (ex.rank + 1) * fo)
        return s_hat, weights, bits, fflags | flags[own], (H[own] if H is not None else None)

    def owned_frames(self, n_frames):
        """Frame indices this rank returns in mode "scatter" (and "peer"):
        block rank of every chunk of chunk_frames frames."""
        c = self.chunk_frames or n_frames
        fpo = c // self.world
        return [ci * c + self.rank * fpo + j for ci in range(n_frames // c) for j in range(fpo)]

    def _receive_scatter(self, rx_shard, want_h):
        """Chunked partials -> all-to-all of the owner blocks -> finish of the
        owned frames.  The all-to-all of chunk i is issued async (NCCL's own
        stream waits for chunk i's partial kernel) and chunk i+1's partial
        kernel is enqueued before the current stream waits for it, so the
        exchange overlaps the next chunk's compute.  Returns (s_hat, weights,
        bits, flags, H) for owned_frames(F), in that order."""
        from . import device as dv, frames

        x = rx_shard
        if isinstance(x, torch.Tensor) and x.dim() == 2:
            x = x[None]
        f = x.shape[0]
        c = self.chunk_frames or f
        if c % self.world or f % c:
            raise ConfigurationError(f"chunk of {c} frames must divide {f} frames and split over {self.world} owners")
        d, m = self.n_data, self.cfg.fft_len
        pending, outs = [], []

        def finish(item):
            recv, work, flags, H = item
            if work is not None:
                work.wait()
            nump, denp = scatter_unpack(recv, d, m)
            s_hat, w, bits, ff = frames.finish_partials(nump, denp, self.cfg.qam_order)
            fpo = c // self.world
            own = slice(self.rank * fpo, (self.rank + 1) * fpo)
            outs.append((s_hat, w, bits, ff | flags[own], H[own] if H is not None else None))

        for ci in range(f // c):
            H, num, den, flags = frames.receive_partials(x[ci * c:(ci + 1) * c], self.shard_cfg, self.pilot,
                                                         symbol0_offset=self.symbol0_offset, n_data=d,
                                                         want_h=want_h)
            recv, work = scatter_partials(num, den, self.group, async_op=True)
            pending.append((recv, work, flags, H))
            if len(pending) > 1:  # chunk ci's kernel is queued: finish chunk ci-1
                finish(pending.pop(0))
        while pending:
            finish(pending.pop(0))
        cat = lambda i: torch.cat([o[i] for o in outs]) if outs[0][i] is not None else None  # noqa: E731
        return cat(0), cat(1), cat(2), cat(3), cat(4)

    def close(self):
        if getattr(self, "peer", None) is not None:
            self.peer.close()
            self.peer = None

    def exchange_bytes(self, n_frames):
        """Bytes each rank contributes to the exchange per call."""
        return n_frames * (self.n_data * self.cfg.fft_len * 8 + self.cfg.fft_len * 4)


def host_partials(Y, H):
    """CPU (numpy) partial sums of one shard, for tests: Y [D,N,M], H [N,M]."""
    num = np.einsum("nm,dnm->dm", np.conj(H), Y)
    den = np.sum(H.real ** 2 + H.imag ** 2, axis=0)
    return num, den
