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

# How the ranks share MPS: "allgather" (every rank holds all slabs: one
# exchange, fastest while the slabs fit), "ring" (each rank holds its own
# shard plus one visiting shard; world-1 point-to-point ring steps, the
# reference's round-robin schedule kernel.py:188-266, for sets that exceed
# HBM), or "auto" (ring when the gathered slabs would take more than
# RING_FRACTION of the smallest free device memory).
EXCHANGE = "auto"
RING_FRACTION = 0.4


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


def exact_offsets(chi: torch.Tensor) -> tuple:
    """Complex offsets of every state in the exact (unpadded) packing and the
    total: state i holds sum_s 2 chi_s chi_{s+1} entries (mps.py:61-62)."""
    ent = (2 * chi[:, :-1].long() * chi[:, 1:].long()).sum(1)
    return torch.cumsum(ent, 0) - ent, int(ent.sum().item()) if ent.numel() else 0


def _pack_native(sites, chi, off, total, m, stride, site_off_dev):
    from ._device import dptr, stream_ptr

    out = sites.new_empty(max(2 * total, 2))
    N.check(N.lib().mpskq_pack_exact(m, chi.shape[0], dptr(sites), dptr(site_off_dev), stride, dptr(chi), dptr(off),
                                     dptr(out), stream_ptr()))
    return out[: 2 * total]


def _unpack_native(packed, off, chi, m, stride, site_off_dev):
    from ._device import dptr, stream_ptr

    sites = packed.new_empty((chi.shape[0], 2 * stride))
    N.check(N.lib().mpskq_unpack_exact(m, chi.shape[0], dptr(packed), dptr(off), dptr(chi), dptr(sites),
                                       dptr(site_off_dev), stride, None, stream_ptr()))
    return sites


def exact_allgather(sites, chi, counts, m, stride, site_off_dev, group=None, pack=None, unpack=None) -> tuple:
    """All-gather every rank's states WITHOUT the layout padding: each rank
    packs its site tensors back to back (mpskq_pack_exact), the packed
    buffers (padded only to the largest rank's byte count) and the bond-dim
    tables are all-gathered, and every rank unpacks all states into the batch
    layout (mpskq_unpack_exact).  Returns (sites_all, chi_all, bytes this rank
    received).  `pack` / `unpack` default to the native kernels (the CPU
    tests pass torch stand-ins)."""
    import torch.distributed as dist

    rank, world = rank_world(group)
    chi_all = allgather_rows(chi, counts, group)
    off, total = exact_offsets(chi)
    packed = (pack or _pack_native)(sites, chi, off, total, m, stride, site_off_dev)
    dev = sites.device
    sz = torch.tensor([[total]], dtype=torch.int64, device=dev)
    sizes = [int(x) for x in allgather_rows(sz, [1] * world, group)[:, 0].tolist()]
    mx = max(max(sizes), 1)
    host = _host_collectives(group)
    pad = torch.zeros(2 * mx, dtype=torch.float64, device="cpu" if host else dev)
    pad[: 2 * total] = packed.to(pad.device)
    parts = torch.empty(world * 2 * mx, dtype=torch.float64, device=pad.device)
    dist.all_gather_into_tensor(parts, pad, group=group) if not host else dist.all_gather(
        list(parts.view(world, 2 * mx).unbind(0)), pad, group=group)
    parts = parts.to(dev)
    offs, s0 = [], 0
    for r, c in enumerate(counts):
        o_r, _ = exact_offsets(chi_all[s0 : s0 + c])
        offs.append(o_r + r * mx)
        s0 += c
    state_off = torch.cat(offs) if offs else torch.zeros(0, dtype=torch.int64, device=dev)
    sites_all = (unpack or _unpack_native)(parts, state_off, chi_all, m, stride, site_off_dev)
    nloc = chi.shape[0]
    received = 16 * (sum(sizes) - total) + 4 * (m + 1) * (sum(counts) - nloc)
    return sites_all, chi_all, received


def gather_rows_to0(rows: torch.Tensor, ids: torch.Tensor, group=None) -> tuple:
    """Rank 0 receives every rank's owned K rows (and their caller row ids);
    other ranks get (None, None).  Shorter row sets are padded with id -1."""
    import torch.distributed as dist

    rank, world = rank_world(group)
    dev = rows.device
    host = _host_collectives(group)
    n = torch.tensor([[rows.shape[0]]], dtype=torch.int64, device=dev)
    counts = [int(x) for x in allgather_rows(n, [1] * world, group)[:, 0].tolist()]
    mx = max(max(counts), 1)
    nk = rows.shape[1] if rows.ndim == 2 else 0
    tdev = "cpu" if host else dev
    pr = torch.zeros((mx, nk), dtype=rows.dtype, device=tdev)
    pi = torch.full((mx,), -1, dtype=torch.int32, device=tdev)
    pr[: rows.shape[0]] = rows.to(tdev)
    pi[: ids.shape[0]] = ids.to(tdev)
    gr = [torch.empty_like(pr) for _ in range(world)] if rank == 0 else None
    gi = [torch.empty_like(pi) for _ in range(world)] if rank == 0 else None
    dist.gather(pr, gr, dst=0, group=group)
    dist.gather(pi, gi, dst=0, group=group)
    if rank != 0:
        return None, None
    return torch.cat(gr).to(dev), torch.cat(gi).to(dev)


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


def _exchange_mode(n_all: int, local, cap: int, cfg, world: int, group=None) -> str:
    """The EXCHANGE setting resolved identically on every rank."""
    if world == 1 or EXCHANGE in ("allgather", "ring"):
        return EXCHANGE if EXCHANGE != "auto" else "allgather"
    from .mps import batch_layout

    _, stride = batch_layout(cfg.m, cap)
    gathered = n_all * 2 * stride * 8
    free = torch.tensor([float(torch.cuda.mem_get_info()[0])], dtype=torch.float64, device="cuda")
    import torch.distributed as dist

    h = free.cpu() if _host_collectives(group) else free
    dist.all_reduce(h, op=dist.ReduceOp.MIN, group=group)
    return "ring" if gathered > RING_FRACTION * float(h.item()) else "allgather"


def _gram_ring(X_bras, X_kets, cfg, kind, budget, chi_max, group, rank, world, local, cap, t_sim, rep):
    """Ring exchange: bras and kets sharded separately; the ket shards travel."""
    from ._device import Timer
    from .kernel import simulate_rows

    train = kind == "train"
    nb, nk = X_bras.shape[0], X_kets.shape[0]
    blo, bhi = shard(nb, world, rank)
    klo, khi = shard(nk, world, rank)
    with Timer() as t_sim2:
        if train:
            kets = local  # the all-gather sharding of the train rows is the same
            if kets is None or kets.chi_cap != cap:
                kets = simulate_rows(X_kets[klo:khi], cfg, budget, chi_max, chi_cap=cap)
            bras = kets
        else:
            rows = np.vstack([X_bras[blo:bhi], X_kets[klo:khi]])
            both = simulate_rows(rows, cfg, budget, chi_max, chi_cap=cap)
            bras, kets = both.rows(0, bhi - blo), both.rows(bhi - blo, len(both))
    counts = [shard(nk, world, r)[1] - shard(nk, world, r)[0] for r in range(world)]
    with Timer() as t_ov:
        K_dev = torch.zeros((nb, nk), dtype=torch.float64, device="cuda")
        comm = _ring_gram(kets, bras, blo, counts, cfg, kind, rank, world, group, K_dev)
    t0 = time.perf_counter()
    K_dev = _reduce_sum_to0(K_dev, group)
    K = K_dev.cpu().numpy() if rank == 0 else np.empty((0, 0))
    rep._add("simulation", t_sim.seconds() + t_sim2.seconds())
    rep._add("communication", comm)
    rep._add("inner_products", t_ov.seconds() - comm)
    rep._add("merge", time.perf_counter() - t0)
    rep.n_inner_products = nk * (nk - 1) // 2 if train else nb * nk
    return K, rep


def ring_plan(world: int, rank: int, kind: str) -> list:
    """(step, held shard, block) for every ring step of `rank`.  At step t the
    rank holds ket shard (rank - t) mod world.  block is "diag" (train, own
    shard: triangle + unit diagonal), "full" (bras of this rank x held kets;
    train mirrors it) or None.  For train each unordered shard pair is
    computed exactly once: ring distance t < world/2 by the holder, and at
    t == world/2 (even world) only by ranks < world/2."""
    plan = []
    for t in range(world):
        held = (rank - t) % world
        if kind != "train":
            plan.append((t, held, "full"))
        elif t == 0:
            plan.append((t, held, "diag"))
        elif 2 * t < world or (2 * t == world and rank < world // 2):
            plan.append((t, held, "full"))
        else:
            plan.append((t, held, None))
    return plan


def _ring_shift_start(tensors: list, rank: int, world: int, group=None) -> tuple:
    """Post the sends of every tensor to rank+1 and the receives of same-shaped
    ones from rank-1; returns the pending (works, received, device) for
    _ring_shift_finish.  On NCCL the transfer runs on the communicator's
    stream, so kernels launched before the finish overlap it."""
    import torch.distributed as dist

    host = _host_collectives(group)
    src = [t.cpu() if host else t for t in tensors]
    dst = [torch.empty_like(t) for t in src]
    ops = []
    for a, b in zip(src, dst):
        ops.append(dist.P2POp(dist.isend, a, (rank + 1) % world, group))
        ops.append(dist.P2POp(dist.irecv, b, (rank - 1) % world, group))
    return dist.batch_isend_irecv(ops), dst, tensors[0].device


def _ring_shift_finish(pending: tuple) -> list:
    works, dst, dev = pending
    for w in works:
        w.wait()
    return [b.to(dev) for b in dst]


def _ring_shift(tensors: list, rank: int, world: int, group=None) -> list:
    """Send every tensor to rank+1 and receive same-shaped ones from rank-1."""
    return _ring_shift_finish(_ring_shift_start(tensors, rank, world, group))


def _ring_gram(full_kets, bras, nb_lo, kets_counts, cfg, kind, rank, world, group, K_dev):
    """Fill this rank's ring blocks of K_dev; returns host seconds spent posting
    and waiting on the shifts (the transfer itself overlaps the block)."""
    from .mps import MpsBatch, overlap_matrix

    mx = max(kets_counts)
    pad_sites = full_kets.sites.new_zeros((mx, full_kets.sites.shape[1]))
    pad_chi = full_kets.chi.new_zeros((mx, full_kets.chi.shape[1]))
    pad_sites[: len(full_kets)] = full_kets.sites
    pad_chi[: len(full_kets)] = full_kets.chi
    offs = np.concatenate([[0], np.cumsum(kets_counts)])
    comm = 0.0
    # every rank shifts the same number of times: train needs ring distances
    # up to world // 2, test all of them
    plan = ring_plan(world, rank, kind)[: (world // 2 + 1 if kind == "train" else world)]
    for t, held, block in plan:
        # post the shift of the held shard before computing on it, so the
        # next shard travels while this block's overlaps run (reference
        # analogue: round-robin step 0 computing the local block, kernel.py:225-227)
        pending = None
        if t < len(plan) - 1:
            t0 = time.perf_counter()
            pending = _ring_shift_start([pad_sites, pad_chi], rank, world, group)
            comm += time.perf_counter() - t0
        c = kets_counts[held]
        if block is not None and c > 0 and len(bras) > 0:
            kets = MpsBatch(cfg.m, full_kets.chi_cap, full_kets.site_off, full_kets.stride, pad_sites[:c],
                            pad_chi[:c], pad_sites.new_zeros(c), pad_chi.new_zeros(c), full_kets.budget,
                            full_kets.gate_count_1q, full_kets.gate_count_2q, full_kets.ortho_center)
            k0, k1 = int(offs[held]), int(offs[held + 1])
            if block == "diag":  # step 0: the held shard is this rank's own (bras)
                K_dev[nb_lo : nb_lo + len(bras), k0:k1] = overlap_matrix(bras, bras, "train")
            elif kind == "train" and held < rank:
                # bra = the lower row index, as compute_gram does (kernel.py:169-175)
                blk = overlap_matrix(kets, bras, "test")
                K_dev[k0:k1, nb_lo : nb_lo + len(bras)] = blk
                K_dev[nb_lo : nb_lo + len(bras), k0:k1] = blk.T
            else:
                blk = overlap_matrix(bras, kets, "test")
                K_dev[nb_lo : nb_lo + len(bras), k0:k1] = blk
                if kind == "train":
                    K_dev[k0:k1, nb_lo : nb_lo + len(bras)] = blk.T
        if pending is not None:
            t0 = time.perf_counter()
            pad_sites, pad_chi = _ring_shift_finish(pending)
            comm += time.perf_counter() - t0
    return comm


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


def _gram_single(X_bras, X_kets, cfg, kind: str, budget: float, chi_max: int = 0):
    """One GPU: the whole path in one native call (mpskq_gram_host: rows in,
    encode + simulate with per-state capacity escalation + overlap, K
    streamed into a page-locked host matrix under the overlap)."""
    import ctypes as C

    from .kernel import RunReport
    from .mps import pinned_matrix
    from ._device import stream_ptr

    train = kind == "train"
    Xb = np.ascontiguousarray(X_bras, dtype=np.float64)
    Xk = np.ascontiguousarray(X_kets, dtype=np.float64)
    nb, nk = (Xk.shape[0], Xk.shape[0]) if train else (Xb.shape[0], Xk.shape[0])
    rep = RunReport()
    if nb == 0 or nk == 0:
        return (np.eye(nk) if train else np.empty((nb, nk))), rep
    K = pinned_matrix(nb, nk)
    secs = np.zeros(4)
    f64 = C.POINTER(C.c_double)
    N.check(N.lib().mpskq_gram_host(
        N.KIND_TRAIN if train else N.KIND_TEST, cfg.m, cfg.r, cfg.d, float(cfg.gamma), float(budget), int(chi_max), 0,
        N.ptr(Xk if train else Xb, C.c_double), nb, None if train else N.ptr(Xk, C.c_double), 0 if train else nk,
        C.cast(K.data_ptr(), f64), stream_ptr(), N.ptr(secs, C.c_double)))
    for phase, dt in zip(("simulation", "inner_products", "communication", "merge"), secs):
        rep._add(phase, float(dt))
    rep.n_simulations = nk if train else nb + nk
    rep.n_inner_products = nk * (nk - 1) // 2 if train else nb * nk
    return K.numpy(), rep


def gram(X_bras, X_kets, cfg, kind: str, budget: float, chi_max: int = 0, group=None):
    """Kernel matrix for run_distributed; returns (K or empty on ranks > 0, RunReport)."""
    import torch.distributed as dist

    from ._device import Timer, require_cuda
    from .kernel import RunReport, simulate_rows
    from .mps import MpsBatch

    require_cuda()
    rank, world = rank_world(group)
    if world == 1 and not FORCE_COLLECTIVES:
        return _gram_single(X_bras, X_kets, cfg, kind, budget, chi_max)
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
    mode = _exchange_mode(n_all, local, cap if _exchange(world) else (local.chi_cap if local else 4), cfg, world,
                          group)
    if mode == "ring" and world > 1 and min(nb, nk) >= world:
        return _gram_ring(X_bras, X_kets, cfg, kind, budget, chi_max, group, rank, world, local, cap, t_sim, rep)
    if _exchange(world):
        from .mps import batch_layout

        off, stride = batch_layout(cfg.m, cap)
        counts = [shard(n_all, world, r)[1] - shard(n_all, world, r)[0] for r in range(world)]
        dev = torch.device("cuda")
        off_d = torch.from_numpy(off).to(dev)
        mine = local if local is not None else None
        sites_l = mine.sites if mine is not None else torch.zeros((0, 2 * stride), dtype=torch.float64, device=dev)
        chi_l = mine.chi if mine is not None else torch.zeros((0, cfg.m + 1), dtype=torch.int32, device=dev)
        disc_l = mine.discard if mine is not None else torch.zeros(0, dtype=torch.float64, device=dev)
        peak_l = mine.peak if mine is not None else torch.zeros(0, dtype=torch.int32, device=dev)
        with Timer() as t_comm:
            sites, chi, _ = exact_allgather(sites_l, chi_l, counts, cfg.m, stride, off_d, group)
            disc = allgather_rows(disc_l, counts, group)
            peak = allgather_rows(peak_l, counts, group)
        ref = mine if mine is not None else None
        full = MpsBatch(cfg.m, cap, off, stride, sites, chi, disc, peak, budget,
                        ref.gate_count_1q if ref else 0, ref.gate_count_2q if ref else 0,
                        ref.ortho_center if ref else None)
        rep._add("communication", t_comm.seconds())
    else:
        full = local
    from ._device import dptr, stream_ptr

    kind_id = N.KIND_TRAIN if train else N.KIND_TEST
    with Timer() as t_ov:
        bras = full.rows(0, nb) if not train else full
        kets = full if train else full.rows(nb, nb + nk)
        n_own = N.C.c_int64(0)
        N.check(N.lib().mpskq_owned_rows(full.chi_cap, nb, rank, world, N.C.byref(n_own)))
        rows = torch.empty((n_own.value, nk), dtype=torch.float64, device="cuda")
        ids = torch.empty(n_own.value, dtype=torch.int32, device="cuda")
        pos = torch.empty(nk, dtype=torch.int32, device="cuda")
        N.check(N.lib().mpskq_overlap_owned_rows(
            kind_id, cfg.m, full.chi_cap, dptr(full.site_off_dev), full.stride, dptr(bras.sites), dptr(bras.chi), nb,
            dptr(kets.sites), dptr(kets.chi), nk, rank, world, dptr(rows), dptr(ids), dptr(pos), stream_ptr()))
    t0 = time.perf_counter()
    all_rows, all_ids = gather_rows_to0(rows, ids, group)
    K = np.empty((0, 0))
    if rank == 0:
        from .mps import pinned_matrix

        K_dev = torch.empty((nb, nk), dtype=torch.float64, device="cuda")
        N.check(N.lib().mpskq_assemble_rows(kind_id, nb, nk, dptr(all_rows), dptr(all_ids), all_ids.shape[0],
                                            dptr(pos) if train else None, dptr(K_dev), nk, stream_ptr()))
        Kp = pinned_matrix(nb, nk)
        Kp.copy_(K_dev)
        K = Kp.numpy()
    rep._add("simulation", t_sim.seconds())
    rep._add("inner_products", t_ov.seconds())
    rep._add("merge", time.perf_counter() - t0)
    rep.n_inner_products = nk * (nk - 1) // 2 if train else nb * nk
    return K, rep
