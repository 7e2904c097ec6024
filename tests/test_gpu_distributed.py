"""run_distributed over processes sharing one GPU (gloo collectives on host
copies; the ranks' kernels never wait on each other): the sharded
simulation, exact (unpadded) all-gather, band-cyclic row ownership and the
gather + assembly on rank 0 must reproduce the single-process kernel
matrix bitwise."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, kind, q, exchange="allgather"):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2411_09336_b200 as P
        from paper_2411_09336_b200 import distributed as D

        D.EXCHANGE = exchange

        torch.cuda.set_device(0)
        g = golden("headline_m165_d1.npz")
        cfg = P.FeatureMapConfig(165, 2, 1, 0.1)
        Xb = g["X"] if kind == "train" else g["X_test"]
        sched = P.make_schedule(len(Xb), len(g["X"]), world, "round_robin", kind)
        rep = P.RunReport()
        K = P.run_distributed(Xb, g["X"], cfg, sched, budget=1e-24, report=rep).entries
        q.put((rank, K, rep.n_simulations, rep.n_inner_products))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["train", "test"])
def test_two_ranks_on_one_gpu_match_single_process(kind):
    import paper_2411_09336_b200 as P

    g = golden("headline_m165_d1.npz")
    cfg = P.FeatureMapConfig(165, 2, 1, 0.1)
    Xb = g["X"] if kind == "train" else g["X_test"]
    ref = P.run_distributed(Xb, g["X"], cfg, P.make_schedule(len(Xb), len(g["X"]), 1, "round_robin", kind)).entries
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (K, ns, ni)) for r, K, ns, ni in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    K0 = out[0][0]
    assert np.array_equal(K0, ref)
    assert np.abs(K0 - (g["K_train"] if kind == "train" else g["K_test"])).max() < 1e-10


@pytest.mark.parametrize("world,kind", [(2, "train"), (3, "train"), (3, "test")])
def test_ring_exchange_matches_single_process(world, kind):
    """Ring exchange (each rank keeps its own shard plus one travelling ket
    shard; for MPS sets beyond HBM) over processes sharing one GPU.  Off-
    diagonal shard blocks take the lower row index as the bra (the
    reference's rule) while the single-process train kernel takes the lower
    position of its ket ordering, so |<a|b>|^2 and |<b|a>|^2 may differ in the
    last bits: equal to 1e-15, exact unit diagonal and symmetry."""
    import paper_2411_09336_b200 as P

    g = golden("headline_m165_d1.npz")
    cfg = P.FeatureMapConfig(165, 2, 1, 0.1)
    Xb = g["X"] if kind == "train" else g["X_test"]
    ref = P.run_distributed(Xb, g["X"], cfg, P.make_schedule(len(Xb), len(g["X"]), 1, "round_robin", kind)).entries
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, kind, q, "ring")) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (K, ns, ni)) for r, K, ns, ni in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    K0 = out[0][0]
    assert np.abs(K0 - ref).max() < 1e-15
    assert np.abs(K0 - (g["K_train"] if kind == "train" else g["K_test"])).max() < 1e-10
    if kind == "train":
        assert np.array_equal(K0, K0.T) and np.all(np.diag(K0) == 1.0)
    else:
        assert np.array_equal(K0, ref)  # test blocks: same roles, same tiles
    assert out[0][2] == (len(g["X"]) * (len(g["X"]) - 1) // 2 if kind == "train" else len(Xb) * len(g["X"]))


def _nccl_single(kind, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        import paper_2411_09336_b200 as P
        from paper_2411_09336_b200 import distributed as D

        D.FORCE_COLLECTIVES = True  # all-gather / all-reduce / reduce through NCCL on device tensors
        g = golden("headline_m165_d1.npz")
        cfg = P.FeatureMapConfig(165, 2, 1, 0.1)
        Xb = g["X"] if kind == "train" else g["X_test"]
        sched = P.make_schedule(len(Xb), len(g["X"]), 1, "round_robin", kind)
        K = P.run_distributed(Xb, g["X"], cfg, sched, budget=1e-24).entries
        q.put((dist.get_backend(), K))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["train", "test"])
def test_nccl_exchange_path_single_gpu(kind):
    """The NCCL branch of the exchange (device all-gather of the exactly
    packed MPS and bond dims, all-reduce of the capacity, gather of the owned
    K rows and assembly) on one rank:
    the only NCCL configuration a one-GPU box can run."""
    import paper_2411_09336_b200 as P

    g = golden("headline_m165_d1.npz")
    cfg = P.FeatureMapConfig(165, 2, 1, 0.1)
    Xb = g["X"] if kind == "train" else g["X_test"]
    ref = P.run_distributed(Xb, g["X"], cfg, P.make_schedule(len(Xb), len(g["X"]), 1, "round_robin", kind)).entries
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_single, args=(kind, q))
    p.start()
    backend, K = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert backend == "nccl"
    assert np.array_equal(K, ref)


def test_bench_multirank_step_four_ranks_share_gpu():
    """bench.py's N>1 step (exact all-gather, owned K rows, gather + assemble
    on rank 0) with 4 ranks sharing one GPU over gloo
    (MPSKQ_BENCH_SHARE_GPU=1): the rank-0 K must pass the run's own oracle
    spot check and the public-API e2e must equal the device step bitwise."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, MPSKQ_BENCH_SHARE_GPU="1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(ROOT / "bench.py"), "--gpus", "4",
           "--rows", "200", "--steps", "1", "--warmup", "3", "--test-rows", "0", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 4
    assert line["parity_spot_check"]["bond_dims_equal"]
    assert line["parity_spot_check"]["max_abs_err_vs_oracle_6x6"] < 1e-10
    assert line["e2e"]["k_bitwise_equal_device_path"]
    comm = line["communication_bytes_per_step"]
    assert comm["allgather_bytes_received"] > 0 and comm["gather_bytes_to_rank0"] > 0
