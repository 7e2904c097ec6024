"""Device plumbing: torch owns device memory and streams; the kernels are ours."""

from __future__ import annotations

import torch

from . import _native as N


def require_cuda() -> torch.device:
    """The GPU path has no CPU fallback: fail loudly without a CUDA device."""
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2411_09336_b200 needs a CUDA (sm_100a) device; there is no CPU fallback"
        )
    N.lib()  # load the native library now so a missing build fails here
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def dptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


class Timer:
    """CUDA-event timer on the current stream."""

    def __init__(self):
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.a.record()
        return self

    def __exit__(self, *exc):
        self.b.record()

    def seconds(self) -> float:
        self.b.synchronize()
        return 1e-3 * self.a.elapsed_time(self.b)
