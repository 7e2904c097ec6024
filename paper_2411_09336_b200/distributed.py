"""Multi-GPU Gram assembly: one process per GPU over torch.distributed (NCCL).

SURVEY.md section 8(e): the rows are block-partitioned across ranks and each
rank simulates its shard (the units are independent); the packed MPS slabs
and bond-dim tables are all-gathered ONCE (the path's only real exchange —
the reference's analogue is the round-robin ring of serialized states,
kernel.py:188-266 / :400-420); every rank then evaluates the block-cyclic
share of overlap tiles (tile t on rank t % world, see mpskq_overlap_tiles)
into a zero matrix, and a SUM-reduce to rank 0 assembles K exactly (the
shares are disjoint, so the sum only ever adds zeros).

The host-side pieces (row sharding, ragged all-gather, tile ownership) are
plain torch.distributed code and are exercised on CPU with gloo in
tests/test_distributed.py.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _native as N


# Run the exchange steps even for a single rank (tests drive the NCCL
# collectives on a one-GPU box this way; multi-GPU runs take them anyway).
FORCE_COLLECTIVES = False


def _exchange(world: int) -> bool:
    return world > 1 or FORCE_COLLECTIVES


def rank_world(group=None) -> tuple:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard(n: int, world: int, rank: int) -> tuple:
    """Contiguous row block of `rank` (earlier ranks one longer)."""
    q, rem = divmod(n, world)
    lo = rank * q + min(rank, rem)
    return lo, lo + q + (rank < rem)


def _host_collectives(group=None) -> bool:
    """gloo runs the collectives on host copies (tests / CPU); NCCL on device."""
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def allgather_rows(local: torch.Tensor, counts: list, group=None) -> torch.Tensor:
    """Concatenate every rank's rows (ragged along dim 0) on every rank."""
    import torch.distributed as dist

    dev = local.device
    if _host_collectives(group):
        local = local.cpu()
    mx = max(counts)
    pad = local.new_zeros((mx,) + tuple(local.shape[1:]))
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in counts]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0).to(dev)


def _all_reduce_max(t: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist

    h = t.cpu() if _host_collectives(group) else t
    dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
    return h.to(t.device)


def _reduce_sum_to0(t: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist

    h = t.cpu() if _host_collectives(group) else t
    dist.reduce(h, dst=0, op=dist.ReduceOp.SUM, group=group)
    return h.to(t.device)


def tiles_of(kind: str, chi_cap: int, n_bras: int, n_kets: int, rank: int, world: int) -> tuple:
    """(tiles int32 (T, 2), row_block, col_block) the library assigns to `rank`."""
    lib = N.lib()
    kid = N.KIND_TRAIN if kind == "train" else N.KIND_TEST
    nt, rb, cb = N.C.c_int64(0), N.C.c_int32(0), N.C.c_int32(0)
    N.check(lib.mpskq_overlap_tiles(kid, chi_cap, n_bras, n_kets, rank, world, None, 0, N.C.byref(nt),
                                    N.C.byref(rb), N.C.byref(cb)))
    out = np.zeros((nt.value, 2), dtype=np.int32)
    N.check(lib.mpskq_overlap_tiles(kid, chi_cap, n_bras, n_kets, rank, world, N.ptr(out, N.C.c_int32),
                                    nt.value, N.C.byref(nt), N.C.byref(rb), N.C.byref(cb)))
    return out, int(rb.value), int(cb.value)


def gram(X_bras, X_kets, cfg, kind: str, budget: float, chi_max: int = 0, group=None):
    """Kernel matrix for run_distributed; returns (K or empty on ranks > 0, RunReport)."""
    import torch.distributed as dist

    from ._device import Timer, require_cuda
    from .kernel import RunReport, simulate_rows
    from .mps import MpsBatch

    require_cuda()
    rank, world = rank_world(group)
    train = kind == "train"
    X_all = X_kets if train else np.vstack([X_bras, X_kets])
    n_all = X_all.shape[0]
    nb = X_kets.shape[0] if train else X_bras.shape[0]
    nk = X_kets.shape[0]
    rep = RunReport()
    lo, hi = shard(n_all, world, rank)
    with Timer() as t_sim:
        local = simulate_rows(X_all[lo:hi], cfg, budget, chi_max) if hi > lo else None
        if _exchange(world):
            cap = torch.tensor([local.chi_cap if local is not None else 0], device="cuda")
            cap = int(_all_reduce_max(cap, group).item())
            if local is not None and local.chi_cap != cap:
                local = simulate_rows(X_all[lo:hi], cfg, budget, chi_max, chi_cap=cap)
    rep.n_simulations = n_all
    if _exchange(world):
        from .mps import batch_layout

        off, stride = batch_layout(cfg.m, cap)
        counts = [shard(n_all, world, r)[1] - shard(n_all, world, r)[0] for r in range(world)]
        dev = torch.device("cuda")
        mine = local if local is not None else None
        sites_l = mine.sites if mine is not None else torch.zeros((0, 2 * stride), dtype=torch.float64, device=dev)
        chi_l = mine.chi if mine is not None else torch.zeros((0, cfg.m + 1), dtype=torch.int32, device=dev)
        disc_l = mine.discard if mine is not None else torch.zeros(0, dtype=torch.float64, device=dev)
        peak_l = mine.peak if mine is not None else torch.zeros(0, dtype=torch.int32, device=dev)
        with Timer() as t_comm:
            sites = allgather_rows(sites_l, counts, group)
            chi = allgather_rows(chi_l, counts, group)
            disc = allgather_rows(disc_l, counts, group)
            peak = allgather_rows(peak_l, counts, group)
        ref = mine if mine is not None else None
        full = MpsBatch(cfg.m, cap, off, stride, sites, chi, disc, peak, budget,
                        ref.gate_count_1q if ref else 0, ref.gate_count_2q if ref else 0,
                        ref.ortho_center if ref else None)
        rep._add("communication", t_comm.seconds())
    else:
        full = local
    from .mps import overlap_matrix

    with Timer() as t_ov:
        bras = full.rows(0, nb) if not train else full
        kets = full if train else full.rows(nb, nb + nk)
        K_dev = torch.zeros((nb, nk), dtype=torch.float64, device="cuda")
        overlap_matrix(bras, kets, kind, rank=rank, world=world, out=K_dev)
    t0 = time.perf_counter()
    if _exchange(world):
        K_dev = _reduce_sum_to0(K_dev, group)
    K = K_dev.cpu().numpy() if rank == 0 else np.empty((0, 0))
    rep._add("simulation", t_sim.seconds())
    rep._add("inner_products", t_ov.seconds())
    rep._add("merge", time.perf_counter() - t0)
    rep.n_inner_products = nk * (nk - 1) // 2 if train else nb * nk
    return K, rep
