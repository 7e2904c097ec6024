"""Truncated SVD on the GPU — the hot-path piece of ``mpskernel.tensor``.

``svd_truncated`` (tensor.py:87-123) runs the same batched one-sided Jacobi
kernel the simulator uses for every two-qubit gate, so the truncation rule
(noise floor 10*eps*s0, longest tail within the budget, at least one value)
can be checked in isolation against the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._device import dptr, require_cuda, stream_ptr

NOISE_FLOOR = 10.0 * np.finfo(np.float64).eps  # tensor.py:17


@dataclass(frozen=True)
class SvdResult:
    left: np.ndarray
    singular_values: np.ndarray
    right: np.ndarray
    discarded_weight: float


def svd_truncated_batched(mats: np.ndarray, budget: float, chi_max: int = 0):
    """(U, s, Vh, keep, discarded) for a (batch, rows, cols) complex stack.
    Only the first keep[b] columns / values / rows of each item are the result."""
    require_cuda()
    mats = np.ascontiguousarray(mats, dtype=np.complex128)
    if mats.ndim != 3:
        raise ValueError("expected a (batch, rows, cols) stack")
    if budget < 0:
        raise ValueError("budget must be non-negative")
    b, rows, cols = mats.shape
    k = min(rows, cols)
    dev = torch.device("cuda")
    A = torch.from_numpy(mats.view(np.float64).reshape(b, -1)).to(dev)
    U = torch.empty((b, rows * k * 2), dtype=torch.float64, device=dev)
    S = torch.empty((b, k), dtype=torch.float64, device=dev)
    V = torch.empty((b, k * cols * 2), dtype=torch.float64, device=dev)
    keep = torch.empty(b, dtype=torch.int32, device=dev)
    disc = torch.empty(b, dtype=torch.float64, device=dev)
    status = torch.zeros(b, dtype=torch.int32, device=dev)
    N.check(N.lib().mpskq_svd_truncated_batched(rows, cols, b, dptr(A), float(budget), int(chi_max), dptr(U),
                                                dptr(S), dptr(V), dptr(keep), dptr(disc), dptr(status),
                                                stream_ptr()))
    if np.any(status.cpu().numpy() == N.STATE_NONFINITE):
        raise ValueError("tensor has non-finite entries")
    return (U.cpu().numpy().view(np.complex128).reshape(b, rows, k), S.cpu().numpy(),
            V.cpu().numpy().view(np.complex128).reshape(b, k, cols), keep.cpu().numpy(), disc.cpu().numpy())


def svd_truncated(t, left_axes: int, budget: float) -> SvdResult:
    """Truncated SVD of ``t`` split after its first ``left_axes`` axes (tensor.py:87-123)."""
    t = np.asarray(t, dtype=np.complex128)
    if t.ndim == 0:
        t = t.reshape(1)
    if not 0 < left_axes < t.ndim:
        raise ValueError("split must leave a non-empty axis group on each side")
    if budget < 0:
        raise ValueError("budget must be non-negative")
    if not np.all(np.isfinite(t)):
        raise ValueError("tensor has non-finite entries")
    ls, rs = t.shape[:left_axes], t.shape[left_axes:]
    u, s, v, keep, disc = svd_truncated_batched(t.reshape(1, math.prod(ls), math.prod(rs)), budget)
    kk = int(keep[0])
    return SvdResult(u[0, :, :kk].reshape(*ls, kk), s[0, :kk].copy(), v[0, :kk].reshape(kk, *rs), float(disc[0]))
