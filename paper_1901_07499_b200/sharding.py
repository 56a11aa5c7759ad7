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
  The exchange functions only use torch.distributed collectives, so they run
  unchanged on the gloo backend for the CPU tests.
"""

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigurationError, ContractError

EXCHANGE_MODES = ("gather", "allreduce")


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


class AntennaShardedReceiver:
    """Antenna-sharded fused receive for one rank of a process group.

    receive(rx_shard) takes this rank's antenna rows [F, N/G, S] of the frames
    and returns (s_hat, weights, bits, flags) for all F frames on every rank."""

    def __init__(self, cfg, n_data, symbol0_offset=0, pilot=None, mode="gather", group=None):
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
        self.shard_cfg = OfdmConfig(cfg.fft_len, cfg.cp_len, self.ant_hi - self.ant_lo, qam_order=cfg.qam_order,
                                    pn_len=cfg.pn_len)

    def receive(self, rx_shard, want_h=False, stream=None):
        from . import frames

        H, num, den, flags = frames.receive_partials(rx_shard, self.shard_cfg, self.pilot,
                                                     symbol0_offset=self.symbol0_offset, n_data=self.n_data,
                                                     want_h=want_h, stream=stream)
        nump, denp = exchange_partials(num, den, self.mode, self.group)
        s_hat, weights, bits, fflags = frames.finish_partials(nump, denp, self.cfg.qam_order, stream=stream)
        return s_hat, weights, bits, fflags | flags, H

    def exchange_bytes(self, n_frames):
        """Bytes each rank contributes to the exchange per call."""
        return n_frames * (self.n_data * self.cfg.fft_len * 8 + self.cfg.fft_len * 4)


def host_partials(Y, H):
    """CPU (numpy) partial sums of one shard, for tests: Y [D,N,M], H [N,M]."""
    num = np.einsum("nm,dnm->dm", np.conj(H), Y)
    den = np.sum(H.real ** 2 + H.imag ** 2, axis=0)
    return num, den
