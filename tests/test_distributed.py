"""Multi-rank host logic of the GPU path on CPU: world_size-2 gloo processes
exercise row sharding, the ragged all-gather of MPS slabs and the disjoint
block-cyclic tile shares whose SUM-reduce assembles K (distributed.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mps_oracle as O
        from paper_2411_09336_b200.distributed import allgather_rows, shard, tiles_of

        # ragged all-gather: rank r contributes rows [lo, hi) of a global table
        n = 7
        lo, hi = shard(n, world, rank)
        full = torch.arange(n * 3, dtype=torch.float64).reshape(n, 3)
        counts = [shard(n, world, r)[1] - shard(n, world, r)[0] for r in range(world)]
        got = allgather_rows(full[lo:hi].clone(), counts)
        ok_gather = torch.equal(got, full)

        # tile shares evaluated with the oracle as the stand-in compute (test only),
        # then SUM-reduced: must equal the single-process Gram bitwise
        rng = np.random.default_rng(5)
        X = rng.uniform(0, 2, (9, 5))
        sites = [O.simulate_row(x, 5, 2, 2, 0.5, 1e-24).sites for x in X]
        K = torch.zeros(9, 9, dtype=torch.float64)
        tiles, rb, cb = tiles_of("train", 4, 9, 9, rank, world)
        for I, J in tiles:
            for i in range(I * rb, min(9, (I + 1) * rb)):
                for j in range(J * cb, min(9, (J + 1) * cb)):
                    if i < j:
                        K[i, j] = K[j, i] = abs(O.overlap(sites[i], sites[j])) ** 2
        if rank == 0:
            K.diagonal().fill_(1.0)
        dist.all_reduce(K, op=dist.ReduceOp.SUM)
        ok_k = np.array_equal(K.numpy(), O.gram(sites, sites, "train"))
        q.put((rank, ok_gather, ok_k, len(tiles)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_gather_and_tile_reduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] and r[2] for r in res), res
    assert sum(r[3] for r in res) > 0


def test_shard_partition():
    from paper_2411_09336_b200.distributed import shard

    for n in (0, 1, 7, 6400):
        for w in (1, 2, 3, 8):
            parts = [shard(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
def test_ring_plan_covers_every_block_once(world):
    """Ring exchange (the reference's round-robin, kernel.py:188-266): train
    computes each unordered shard pair once (own shard as a triangle), test
    every (bra shard, ket shard) block once."""
    from paper_2411_09336_b200.distributed import ring_plan

    steps = world // 2 + 1
    seen = {}
    for r in range(world):
        plan = ring_plan(world, r, "train")[:steps]
        for t, held, block in plan:
            assert held == (r - t) % world
            if block is not None:
                key = frozenset((r, held))
                seen[key] = seen.get(key, 0) + 1
                assert (block == "diag") == (held == r)
    assert len(seen) == world * (world + 1) // 2 and set(seen.values()) == {1}
    test = [(r, held) for r in range(world) for _, held, b in ring_plan(world, r, "test") if b == "full"]
    assert sorted(test) == [(r, s) for r in range(world) for s in range(world)]


def _ring_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_09336_b200.distributed import _ring_shift

        a = torch.full((3, 2), float(rank), dtype=torch.float64)
        b = torch.full((4,), rank, dtype=torch.int32)
        for step in range(1, world):
            a, b = _ring_shift([a, b], rank, world)
            ok = bool((a == float((rank - step) % world)).all() and (b == (rank - step) % world).all())
            if not ok:
                break
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_ring_shift_gloo_three_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ring_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res


def _torch_pack(sites, chi, off, total, m, stride, site_off):
    """Test stand-in of mpskq_pack_exact (host torch; the product path uses the kernel)."""
    out = torch.zeros(2 * total, dtype=torch.float64)
    so = site_off.tolist()
    for i in range(chi.shape[0]):
        o = int(off[i]) * 2
        for s in range(m):
            ln = 2 * 2 * int(chi[i, s]) * int(chi[i, s + 1])
            out[o : o + ln] = sites[i, 2 * so[s] : 2 * so[s] + ln]
            o += ln
    return out


def _torch_unpack(packed, off, chi, m, stride, site_off):
    sites = torch.zeros((chi.shape[0], 2 * stride), dtype=torch.float64)
    so = site_off.tolist()
    for i in range(chi.shape[0]):
        o = int(off[i]) * 2
        for s in range(m):
            ln = 2 * 2 * int(chi[i, s]) * int(chi[i, s + 1])
            sites[i, 2 * so[s] : 2 * so[s] + ln] = packed[o : o + ln]
            o += ln
    return sites


def _exchange_worker(rank, world, port, q):
    """The multi-GPU exchange of distributed.gram with gloo on CPU: exact
    (unpadded) all-gather of ragged MPS shards, row-ownership of K rows and
    their gather to rank 0 (the kernels are replaced by host stand-ins)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mps_oracle as O
        from paper_2411_09336_b200 import _native as N
        from paper_2411_09336_b200.distributed import exact_allgather, gather_rows_to0, shard
        from paper_2411_09336_b200.mps import batch_layout

        m, n = 6, 11
        X = np.random.default_rng(3).uniform(0, 2, (n, m))
        states = [O.simulate_row(x, m, 2, 2, 0.5, 1e-24).sites for x in X]
        cap = 8
        off, stride = batch_layout(m, cap)
        lay = np.zeros((n, stride), dtype=np.complex128)
        chi = np.zeros((n, m + 1), dtype=np.int32)
        for i, st in enumerate(states):
            chi[i] = [t.shape[0] for t in st] + [1]
            for s, t in enumerate(st):
                lay[i, off[s] : off[s] + t.size] = t.reshape(-1)
        lay_t = torch.from_numpy(lay.view(np.float64).copy())
        chi_t = torch.from_numpy(chi)
        counts = [shard(n, world, r)[1] - shard(n, world, r)[0] for r in range(world)]
        lo, hi = shard(n, world, rank)
        got, got_chi, recv = exact_allgather(lay_t[lo:hi].clone(), chi_t[lo:hi].clone(), counts, m, stride,
                                             torch.from_numpy(off), pack=_torch_pack, unpack=_torch_unpack)
        ok_sites = torch.equal(got, lay_t) and torch.equal(got_chi, chi_t)
        exact_bytes = 16 * int(sum((2 * chi[i, :-1] * chi[i, 1:]).sum() for i in range(n) if not lo <= i < hi))
        ok_bytes = recv == exact_bytes + 4 * (m + 1) * (n - (hi - lo))

        # row ownership: this rank's rows (oracle stand-in for the overlap),
        # gathered on rank 0 and assembled (upper triangle + mirror + diag)
        n_own = N.C.c_int64(0)
        N.check(N.lib().mpskq_owned_rows(cap, n, rank, world, N.C.byref(n_own)))
        own = [b for b in range(n) if b % world == rank]  # single-row bands off the chi <= 4 path
        assert n_own.value == len(own)
        rows = torch.zeros((len(own), n), dtype=torch.float64)
        for k, a in enumerate(own):
            for b in range(a + 1, n):
                rows[k, b] = abs(O.overlap(states[a], states[b])) ** 2
        ids = torch.tensor(own, dtype=torch.int32)
        all_rows, all_ids = gather_rows_to0(rows, ids)
        ok_k = True
        if rank == 0:
            K = torch.zeros((n, n), dtype=torch.float64)
            for r, a in zip(all_rows, all_ids.tolist()):
                if a >= 0:
                    K[a] = r
            K = torch.triu(K, 1) + torch.triu(K, 1).T + torch.eye(n, dtype=torch.float64)
            ok_k = np.array_equal(K.numpy(), O.gram(states, states, "train"))
        q.put((rank, ok_sites, ok_bytes, ok_k))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_exact_allgather_and_row_gather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] and r[2] and r[3] for r in res), res


def test_owned_rows_partition_every_row_once():
    """Row ownership (mpskq_owned_rows / mpskq_overlap_owned_rows): bands of 8
    ordered rows at capacity 4, single rows otherwise, band b on rank b % world."""
    from paper_2411_09336_b200 import _native as N

    for cap, rb in ((4, 8), (8, 1), (48, 1)):
        for n in (1, 7, 8, 9, 100, 6400):
            for world in (1, 2, 3, 8):
                tot = 0
                for r in range(world):
                    c = N.C.c_int64(0)
                    N.check(N.lib().mpskq_owned_rows(cap, n, r, world, N.C.byref(c)))
                    bands = [b for b in range((n + rb - 1) // rb) if b % world == r]
                    assert c.value == len(bands) * rb
                    tot += sum(min(rb, n - b * rb) for b in bands)
                assert tot == n
