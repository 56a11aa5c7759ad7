"""paper_1901_07499_b200 — B200-native (sm_100a) uplink OFDM receive path.

CP drop + FFT + fftshift, LS channel estimation, MRC combining (with a
per-antenna ZF option) and hard QAM demapping, fused into one CUDA kernel
behind a C ABI (include/ofdmrx_b200.h), with the reference ``ofdmrx``
receiver API mirrored in ``receiver`` (Gokalgandhi et al., arXiv:1901.07499).
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    ConfigurationError,
    ContractError,
    DeviceError,
    FramingError,
    InputError,
    NumericInputError,
    PipelineOrderError,
    ReceiverError,
)
from .waveform import OfdmConfig, PilotDefinition, default_cp, make_pilot  # noqa: F401


def __getattr__(name):
    # heavy (torch) modules load lazily
    if name in ("receiver", "frames", "device", "synth", "sharding", "sync", "ingest"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    if name in ("receive_frames", "receive_partials", "finish_partials", "FrameBatch", "receive_captures"):
        from . import frames

        return getattr(frames, name)
    raise AttributeError(name)
