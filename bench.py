#!/usr/bin/env python
"""Headline benchmark: the 165-qubit, N=6400 train kernel matrix.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[3] / SURVEY.md 8(d) row 4): m=165 qubits,
interaction distance d=1, 2 layers, gamma=0.1, per-gate budget 1e-24,
N=6400 synthetic rows uniform in [0, 2] (seed 0).  One step = encode every
row, simulate every MPS, fill the whole train kernel (20,476,800 computed
entries; diagonal and mirror are free).  On N GPUs the rows are sharded, the
MPS all-gathered once over NCCL without the layout padding, every rank
computes the K rows of the bra bands it owns (band b -> rank b % N) and rank
0 gathers and assembles them (total work fixed: strong scaling).

`value` is entries/s with the feature rows already in HBM; `e2e` is the same
metric through the public API run_distributed (host rows in, host K out, every
copy inside the timed region; `e2e_c_abi` is the C ABI mpskq_gram_host under
it).  `test_kernel` times the headline TEST kernel (1600 test rows x 6400
train states) with its own roofline.  The reference arm (--impl reference)
times the CPU oracle (a numpy restatement of the reference that is bitwise
identical to it, oracle/mps_oracle.py) on every host core over a bounded
sample and projects the same metric.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import multiprocessing as mp  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "kernel entries/s + train-kernel wall time (165 qubits, N=6400) at 1/2/4/8 B200"
UNIT = "entries/s"
M, R, D, GAMMA, BUDGET = 165, 2, 1, 0.1, 1e-24
WORKLOAD = "headline train kernel: 165 qubits, d=1, 2 layers, gamma=0.1, budget=1e-24, N=6400 (BASELINE configs[3])"
# ~3 h for the N=6400 train kernel on 32x A100
PUBLISHED_ENTRIES_PER_S = 6400 * 6399 / 2 / (3 * 3600.0)


def feature_rows(n: int, m: int = M, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 2.0, (n, m))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ CPU (oracle)
def _cpu_worker(job):
    rows, seconds = job
    from oracle import mps_oracle as O

    t0 = time.perf_counter()
    states = [O.simulate_row(x, M, R, D, GAMMA, BUDGET).sites for x in rows]
    t_sim = time.perf_counter() - t0
    pairs = [(a, b) for a in range(len(states)) for b in range(a + 1, len(states))]
    count, t1 = 0, time.perf_counter()
    while True:
        for a, b in pairs:
            O.overlap(states[a], states[b])
            count += 1
        if time.perf_counter() - t1 >= seconds:
            break
    return len(rows), t_sim, count, time.perf_counter() - t1


def cpu_sample(n: int, seconds: float, cores: int | None = None) -> dict:
    """Time the oracle on `cores` processes over a bounded sample (4 simulations
    + `seconds` of overlaps per process) and project the N-row train kernel."""
    cores = cores or host_cores()
    X = feature_rows(max(4 * cores, 4))
    jobs = [(X[4 * i : 4 * i + 4], seconds) for i in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_cpu_worker, jobs)
    sims_per_s = sum(k / t for k, t, _, _ in res)
    pairs_per_s = sum(c / t for _, _, c, t in res)
    entries = n * (n - 1) / 2
    wall = n / sims_per_s + entries / pairs_per_s
    return {
        "value": entries / wall,
        "unit": UNIT,
        "cores": cores,
        "kind": "port",
        "sample": (
            f"{cores} processes x (4 MPS simulations + {seconds:.0f} s of overlaps) at the headline shape, "
            f"projected to the N={n} train kernel ({sims_per_s:.1f} MPS/s, {pairs_per_s:.0f} overlaps/s)"
        ),
        "mps_states_per_s": sims_per_s,
        "projected_train_wall_s": wall,
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.lines: list = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ roofline helpers
def train_flops(chi: np.ndarray) -> float:
    """sum_{i<j} F(i,j), F = sum_s 16 chi^b_s chi^a_{s+1} (chi^a_s + chi^b_{s+1}) with
    bra a = row i, ket b = row j, via prefix sums over i."""
    c = chi.astype(np.float64)
    total = 0.0
    for s in range(c.shape[1] - 1):
        u1 = c[:, s + 1] * c[:, s]  # bra factor of the first term
        u2 = c[:, s + 1]  # bra factor of the second term
        v1 = c[:, s]  # ket factor of the first term
        v2 = c[:, s] * c[:, s + 1]  # ket factor of the second term
        p1 = np.concatenate([[0.0], np.cumsum(u1)[:-1]])  # sum over i < j
        p2 = np.concatenate([[0.0], np.cumsum(u2)[:-1]])
        total += 16.0 * float(np.dot(p1, v1) + np.dot(p2, v2))
    return total


def fp64_peak_tflops(lib, torch) -> float:
    """Measured FFMA64 throughput (no FP64 entry in MEASURED_PEAKS.json)."""
    from paper_2411_09336_b200 import _native as N

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 8, 100_000
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    N.check(lib.mpskq_fp64_probe(blocks, 1000, out.data_ptr(), st))
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        N.check(lib.mpskq_fp64_probe(blocks, iters, out.data_ptr(), st))
        b.record()
        b.synchronize()
        flops = 2.0 * 16 * iters * blocks * 256
        best = max(best, flops / (1e-3 * a.elapsed_time(b)) / 1e12)
    return best


# ------------------------------------------------------------------ GPU arm
def test_flops(chi_b: np.ndarray, chi_k: np.ndarray) -> float:
    """sum over ALL (bra i, ket j) of F(i,j) (test kind, kernel.py:176-181)."""
    cb, ck = chi_b.astype(np.float64), chi_k.astype(np.float64)
    total = 0.0
    for s in range(cb.shape[1] - 1):
        # F = 16 chi^k_s chi^b_{s+1} chi^b_s + 16 chi^k_s chi^k_{s+1} chi^b_{s+1}
        total += 16.0 * (float((cb[:, s + 1] * cb[:, s]).sum()) * float(ck[:, s].sum())
                         + float(cb[:, s + 1].sum()) * float((ck[:, s] * ck[:, s + 1]).sum()))
    return total


def config_dict(n: int) -> dict:
    """The workload keys both arms report (identical key sets)."""
    return {"workload": WORKLOAD, "m": M, "d": D, "layers": R, "gamma": GAMMA, "budget": BUDGET, "N": n,
            "computed_entries": n * (n - 1) // 2}


def gpu_main(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.rows
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(n, args.cpu_seconds)  # before CUDA init (forked workers)

    # MPSKQ_BENCH_SHARE_GPU=1 maps every rank onto cuda:0 and uses gloo (host
    # collectives): a functional check of the multi-rank path on a 1-GPU box.
    # The ranks' kernels never wait on each other.  Real runs use NCCL.
    share = os.environ.get("MPSKQ_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            # communicator setup (ranks, NVLS / channels) in the log for the scaling run
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200 import _native as N
    from paper_2411_09336_b200.ansatz import feature_map_topology
    from paper_2411_09336_b200.distributed import _all_reduce_max, exact_allgather, gather_rows_to0, shard
    from paper_2411_09336_b200.kernel import simulate_rows
    from paper_2411_09336_b200.mps import batch_layout, compile_program

    lib = N.lib()
    cfg = P.FeatureMapConfig(M, R, D, GAMMA)
    X = feature_rows(n)
    lo, hi = shard(n, world, rank)
    nloc = hi - lo
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    X_loc = torch.from_numpy(X[lo:hi]).to(dev)
    prog = compile_program(feature_map_topology(M, R, D))
    ops = prog.device_ops
    # capacity the states need (public path, also warms the library up)
    cap = simulate_rows(X[lo:hi], cfg, BUDGET).chi_cap
    if world > 1:
        cap = int(_all_reduce_max(torch.tensor([cap], device=dev)).item())
    off, stride = batch_layout(M, cap)
    off_d = torch.from_numpy(off).to(dev)
    coef = torch.empty((nloc, prog.n_params, 2), dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    sites_loc = torch.empty((nloc, 2 * stride), dtype=torch.float64, device=dev)
    chi_loc = torch.empty((nloc, M + 1), dtype=torch.int32, device=dev)
    disc = torch.empty(nloc, dtype=torch.float64, device=dev)
    peak = torch.empty(nloc, dtype=torch.int32, device=dev)
    status = torch.zeros(nloc, dtype=torch.int32, device=dev)
    counts = [shard(n, world, r)[1] - shard(n, world, r)[0] for r in range(world)]
    K = torch.empty((n, n), dtype=torch.float64, device=dev)
    if world > 1:
        n_own = N.C.c_int64(0)
        N.check(lib.mpskq_owned_rows(cap, n, rank, world, N.C.byref(n_own)))
        rows = torch.empty((n_own.value, n), dtype=torch.float64, device=dev)
        ids = torch.empty(n_own.value, dtype=torch.int32, device=dev)
        pos = torch.empty(n, dtype=torch.int32, device=dev)
    comm = {"allgather_bytes_received": 0, "gather_bytes_to_rank0": 0}
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    # ours per step: encode, simulate, ket key, chi=4 clustering, block bounds,
    # inverse order, pack bras, pack kets, overlap, un-permute / owned rows,
    # diagonal (N=1); N>1 adds exact pack + unpack and, on rank 0, scatter +
    # mirror.  The ket key sort is CUB's radix sort (library, not counted).
    launches_per_step = (11 if world == 1 else 12 + (2 if rank == 0 else 0))
    state = {"sites_all": sites_loc, "chi_all": chi_loc}

    def step(e):
        e[0].record()
        N.check(lib.mpskq_feature_map_coefficients_device(X_loc.data_ptr(), nloc, M, R, D, GAMMA, coef.data_ptr(),
                                                          bad.data_ptr(), sp))
        N.check(lib.mpskq_simulate(M, cap, ops.data_ptr(), prog.ops.shape[0], prog.n_gates, coef.data_ptr(),
                                   prog.n_params, nloc, BUDGET, 0, off_d.data_ptr(), stride, sites_loc.data_ptr(),
                                   chi_loc.data_ptr(), disc.data_ptr(), peak.data_ptr(), status.data_ptr(), None, sp))
        e[1].record()
        if world > 1:  # the one exchange: exact (unpadded) all-gather of the MPS
            sa, ca, recv = exact_allgather(sites_loc, chi_loc, counts, M, stride, off_d)
            state["sites_all"], state["chi_all"] = sa, ca
            comm["allgather_bytes_received"] = recv
        e[2].record()
        sa, ca = state["sites_all"], state["chi_all"]
        if world == 1:
            N.check(lib.mpskq_overlap(N.KIND_TRAIN, N.OUT_KERNEL, M, cap, off_d.data_ptr(), stride, sa.data_ptr(),
                                      ca.data_ptr(), n, sa.data_ptr(), ca.data_ptr(), n, 0, 1, K.data_ptr(), n, sp))
            e[3].record()
        else:
            N.check(lib.mpskq_overlap_owned_rows(N.KIND_TRAIN, M, cap, off_d.data_ptr(), stride, sa.data_ptr(),
                                                 ca.data_ptr(), n, sa.data_ptr(), ca.data_ptr(), n, rank, world,
                                                 rows.data_ptr(), ids.data_ptr(), pos.data_ptr(), sp))
            e[3].record()
            all_rows, all_ids = gather_rows_to0(rows, ids)
            if rank == 0:
                comm["gather_bytes_to_rank0"] = int(all_rows.numel() * 8 - rows.numel() * 8)
                N.check(lib.mpskq_assemble_rows(N.KIND_TRAIN, n, n, all_rows.data_ptr(), all_ids.data_ptr(),
                                                all_ids.shape[0], pos.data_ptr(), K.data_ptr(), n, sp))
        e[4].record()

    for _ in range(args.warmup):
        step(ev[0])
    torch.cuda.synchronize()
    if int(status.max().item()) != 0 or int(bad.item()) != 0:
        raise RuntimeError("simulation reported a bad state during warm-up")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip().isdigit()]
    gpu_index = int(vis[local]) if local < len(vis) else local
    with ClockSampler(gpu_index) as clocks:
        t0.record()
        for k in range(args.steps):
            step(ev[k])
        t1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / args.steps
    sim_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    comm_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    ov_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    red_ms = float(np.mean([e[3].elapsed_time(e[4]) for e in ev]))
    if world > 1:
        t = torch.tensor([ms, sim_ms, comm_ms, ov_ms, red_ms], dtype=torch.float64, device=dev)
        ms, sim_ms, comm_ms, ov_ms, red_ms = _all_reduce_max(t).tolist()

    # parity spot check of this very run against the CPU oracle (rows 0..5)
    spot = chi_ok = None
    chi_all = state["chi_all"]
    if rank == 0:
        from oracle import mps_oracle as O

        sub = [O.simulate_row(x, M, R, D, GAMMA, BUDGET) for x in X[:6]]
        Ko = O.gram([s.sites for s in sub], [s.sites for s in sub], "train")
        spot = float(np.abs(K[:6, :6].cpu().numpy() - Ko).max())
        chi_ok = bool(np.array_equal(chi_all[:6].cpu().numpy(), np.array([s.bond_dims() for s in sub])))
    K_dev_np = K.cpu().numpy() if rank == 0 else None

    # e2e through the public API: run_distributed (kernel.py:443-512) with
    # host rows in and the host K out (N=1: one native call that streams K
    # into page-locked memory under the overlap; N>1: sharded + gathered)
    sched = P.make_schedule(n, n, world, "round_robin", "train")
    for _ in range(max(1, args.warmup)):
        g = P.run_distributed(X, X, cfg, sched, budget=BUDGET)
    del g
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record()
    k_equal = None
    for k in range(args.steps):
        g = P.run_distributed(X, X, cfg, sched, budget=BUDGET)
        if k == args.steps - 1 and rank == 0:
            last = g
        del g
    b.record()
    b.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = a.elapsed_time(b) / args.steps
    wall_ms = 1e3 * (time.perf_counter() - w0) / args.steps
    if world > 1:
        e2e_ms, wall_ms = _all_reduce_max(torch.tensor([e2e_ms, wall_ms], dtype=torch.float64, device=dev)).tolist()
    if rank == 0:
        k_equal = bool(np.array_equal(last.entries, K_dev_np))
        del last
    e2e = {"value": n * (n - 1) / 2 / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": X.nbytes,
           "d2h_bytes_per_step": n * n * 8, "ms_per_step": e2e_ms, "host_wall_ms_per_step": wall_ms,
           "path": "public API run_distributed(X, X, cfg, make_schedule(N, N, n_gpus, 'round_robin', 'train')): "
                   "host rows -> host K (N=1: mpskq_gram_host streams K row bands into page-locked memory "
                   "under the overlap)",
           "k_bitwise_equal_device_path": k_equal}

    # the C ABI itself (what a non-Python binding calls), N=1
    e2e_c = None
    if world == 1:
        import ctypes as C

        Xp = torch.from_numpy(X).pin_memory()
        Kp = torch.empty((n, n), dtype=torch.float64).pin_memory()
        secs = np.zeros(4)

        def host_call():
            N.check(lib.mpskq_gram_host(N.KIND_TRAIN, M, R, D, GAMMA, BUDGET, 0, 0,
                                        C.cast(Xp.data_ptr(), C.POINTER(C.c_double)), n, None, 0,
                                        C.cast(Kp.data_ptr(), C.POINTER(C.c_double)), sp,
                                        N.ptr(secs, C.c_double)))

        for _ in range(max(1, args.warmup)):
            host_call()
        a.record()
        for _ in range(args.steps):
            host_call()
        b.record()
        b.synchronize()
        ms_c = a.elapsed_time(b) / args.steps
        e2e_c = {"value": n * (n - 1) / 2 / (ms_c / 1e3), "ms_per_step": ms_c,
                 "path": "C ABI mpskq_gram_host (pinned host rows -> pinned host K)"}
        del Kp

    # the headline TEST kernel (BASELINE configs[3]: M=1600 test rows x N
    # train states, kernel.py:176-181): simulate the test rows and fill M x N
    # against the resident train states (the inference use)
    test_line = None
    if world == 1 and args.test_rows > 0:
        mt = args.test_rows
        Xt = feature_rows(mt, seed=1)
        Xt_d = torch.from_numpy(Xt).to(dev)
        coef_t = torch.empty((mt, prog.n_params, 2), dtype=torch.float64, device=dev)
        sites_t = torch.empty((mt, 2 * stride), dtype=torch.float64, device=dev)
        chi_t = torch.empty((mt, M + 1), dtype=torch.int32, device=dev)
        disc_t = torch.empty(mt, dtype=torch.float64, device=dev)
        peak_t = torch.empty(mt, dtype=torch.int32, device=dev)
        status_t = torch.zeros(mt, dtype=torch.int32, device=dev)
        Kt = torch.empty((mt, n), dtype=torch.float64, device=dev)
        evt = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]

        def tstep(e):
            e[0].record()
            N.check(lib.mpskq_feature_map_coefficients_device(Xt_d.data_ptr(), mt, M, R, D, GAMMA,
                                                              coef_t.data_ptr(), bad.data_ptr(), sp))
            N.check(lib.mpskq_simulate(M, cap, ops.data_ptr(), prog.ops.shape[0], prog.n_gates, coef_t.data_ptr(),
                                       prog.n_params, mt, BUDGET, 0, off_d.data_ptr(), stride, sites_t.data_ptr(),
                                       chi_t.data_ptr(), disc_t.data_ptr(), peak_t.data_ptr(), status_t.data_ptr(),
                                       None, sp))
            e[1].record()
            N.check(lib.mpskq_overlap(N.KIND_TEST, N.OUT_KERNEL, M, cap, off_d.data_ptr(), stride,
                                      sites_t.data_ptr(), chi_t.data_ptr(), mt, sites_loc.data_ptr(),
                                      chi_loc.data_ptr(), n, 0, 1, Kt.data_ptr(), n, sp))
            e[2].record()

        for _ in range(args.warmup):
            tstep(evt[0])
        torch.cuda.synchronize()
        if int(status_t.max().item()) != 0:
            raise RuntimeError("test-row simulation reported a bad state")
        a.record()
        for k in range(args.steps):
            tstep(evt[k])
        b.record()
        b.synchronize()
        t_ms = a.elapsed_time(b) / args.steps
        t_ov = float(np.mean([e[1].elapsed_time(e[2]) for e in evt]))
        t_sim = float(np.mean([e[0].elapsed_time(e[1]) for e in evt]))
        tfl = test_flops(chi_t.cpu().numpy(), chi_loc.cpu().numpy())
        from oracle import mps_oracle as O

        sub_t = [O.simulate_row(x, M, R, D, GAMMA, BUDGET) for x in Xt[:3]]
        sub = [O.simulate_row(x, M, R, D, GAMMA, BUDGET) for x in X[:4]]
        Kto = O.gram([s.sites for s in sub_t], [s.sites for s in sub], "test")
        # end to end through the public API (test rows and train rows in, M x N K
        # out: run_distributed also simulates the train rows, kernel.py:443-512)
        tsched = P.make_schedule(mt, n, 1, "round_robin", "test")
        for _ in range(max(1, args.warmup)):
            del_g = P.run_distributed(Xt, X, cfg, tsched, budget=BUDGET)
        del del_g
        a.record()
        for _ in range(args.steps):
            g = P.run_distributed(Xt, X, cfg, tsched, budget=BUDGET)
            del g
        b.record()
        b.synchronize()
        te2e_ms = a.elapsed_time(b) / args.steps
        test_line = {
            "workload": f"headline test kernel: {mt} test rows (seed 1) x {n} train states (BASELINE configs[3])",
            "e2e": {"value": mt * n / (te2e_ms / 1e3), "unit": UNIT, "ms_per_step": te2e_ms,
                    "h2d_bytes_per_step": Xt.nbytes + X.nbytes, "d2h_bytes_per_step": mt * n * 8,
                    "path": "public API run_distributed(X_test, X_train, cfg, make_schedule(M, N, 1, 'round_robin', "
                            "'test')): simulates the test AND train rows, K streamed to page-locked host memory"},
            "entries": mt * n, "value": mt * n / (t_ms / 1e3), "unit": UNIT, "ms_per_step": t_ms,
            "phases_ms": {"simulate_test_rows": t_sim, "overlap": t_ov},
            "roofline": None,  # filled below with the same peak
            "algorithmic_flops_per_launch": tfl,
            "parity_spot_check": {"max_abs_err_vs_oracle_3x4": float(np.abs(Kt[:3, :4].cpu().numpy() - Kto).max())},
        }
        del Kt, sites_t

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    chi_np = chi_all.cpu().numpy()
    flops = train_flops(chi_np)
    peak_tf = fp64_peak_tflops(lib, torch)
    achieved = flops / world / (ov_ms / 1e3) / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("overlap_o1_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    if test_line is not None:
        ach_t = test_line["algorithmic_flops_per_launch"] / (test_line["phases_ms"]["overlap"] / 1e3) / 1e12
        test_line["roofline"] = {"bound": "fp64", "achieved": ach_t, "peak": peak_tf, "unit": "TFLOP/s",
                                 "frac": ach_t / peak_tf if peak_tf else None,
                                 "kernel": "overlap_o1_kernel, test kind (whole mpskq_overlap call)"}
    entries = n * (n - 1) / 2
    line = {
        "metric": METRIC,
        "value": entries / (ms / 1e3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": entries / (ms / 1e3) / PUBLISHED_ENTRIES_PER_S,
        "dtype": "c128",
        "data": "synthetic: rows uniform [0,2] (seed 0); no trained weights exist for this path",
        "config": config_dict(n),
        "layout": {
            "parallelism": (f"rows sharded x{world}, MPS all-gathered once (exact, unpadded), K rows owned "
                            f"band-cyclically and gathered to rank 0" if world > 1 else "one GPU"),
            "l2": "working set (540 MB padded MPS + 328 MB K) larger than L2; no flush needed",
            "chi_cap": cap,
        },
        "train_wall_s": ms / 1e3,
        "mps_states_per_s": n / (sim_ms / 1e3),
        "phases_ms": {"simulate": sim_ms, "all_gather": comm_ms, "overlap": ov_ms, "gather_assemble": red_ms},
        "communication_bytes_per_step": comm if world > 1 else None,
        "roofline": {
            "bound": "fp64",
            "kernel": "overlap_o1_kernel (timed as the whole mpskq_overlap call: ket ordering + 2 packs + overlap + diagonal)",
            "achieved": achieved,
            "peak": peak_tf,
            "unit": "TFLOP/s",
            "frac": achieved / peak_tf if peak_tf else None,
            "traffic": traffic,
            "algorithmic_flops_per_launch": flops / world,
            "peak_source": "measured in-run: FP64 FMA probe (mpskq_fp64_probe), burst; MEASURED_PEAKS.json has no FP64",
        },
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "e2e": e2e,
        "e2e_c_abi": e2e_c,
        "test_kernel": test_line,
        "gpu_launches": launches_per_step * args.steps,
        "parity_spot_check": {"max_abs_err_vs_oracle_6x6": spot, "bond_dims_equal": chi_ok},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ reference arm
def as_shipped_sample(rows: int) -> dict | None:
    """The unmodified reference as shipped (BASELINE.md section 2 mode 1):
    kernel.run_distributed(k=1) from baseline/_ref on `rows` headline rows
    (its worker threads are GIL-bound, k > 1 is slower), entries/s."""
    ref = ROOT / "baseline" / "_ref"
    if rows <= 1 or not (ref / "mpskernel").exists():
        return None
    import importlib

    sys.path.insert(0, str(ref))
    try:
        K = importlib.import_module("mpskernel.kernel")
        A = importlib.import_module("mpskernel.ansatz")
        X = feature_rows(rows)
        cfg = A.FeatureMapConfig(M, R, D, GAMMA)
        t0 = time.perf_counter()
        K.run_distributed(X, X, cfg, K.make_schedule(rows, rows, 1, "round_robin", "train"), budget=BUDGET)
        dt = time.perf_counter() - t0
    finally:
        sys.path.remove(str(ref))
    entries = rows * (rows - 1) / 2
    return {"value": entries / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"mpskernel.kernel.run_distributed(k=1), unmodified, on {rows} headline rows "
                      f"({rows} simulations + {int(entries)} overlaps in {dt:.1f} s)"}


def reference_main(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.rows
    seconds = max(2.0, args.ref_seconds)
    for _ in range(args.warmup):
        cpu_sample(n, 0.5)
    vals, walls = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = cpu_sample(n, seconds)
        vals.append(s["value"])
        walls.append(s["projected_train_wall_s"])
    elapsed = (time.perf_counter() - t0) / args.steps
    v = float(np.median(vals))
    shipped = as_shipped_sample(args.shipped_rows)
    line = {
        "metric": METRIC,
        "impl": "reference",
        "value": v,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * elapsed,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": v / PUBLISHED_ENTRIES_PER_S,
        "dtype": "c128",
        "data": "synthetic: rows uniform [0,2] (seed 0)",
        "config": config_dict(n),
        "train_wall_s": float(np.median(walls)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": s["cores"], "kind": "port", "sample": s["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "as_shipped": shipped,
        "note": "reference is pure Python/numpy (nothing to compile); timed through oracle/mps_oracle.py, "
                "which is bitwise identical to it (tests/test_oracle.py), in a process pool over every host "
                "core; `as_shipped` times the unmodified reference's own run_distributed(k=1) from baseline/_ref",
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--rows", type=int, default=6400, help="N feature rows (train kernel N x N)")
    ap.add_argument("--test-rows", type=int, default=1600, help="M test rows of the headline test kernel (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--shipped-rows", type=int, default=48, help="rows of the as-shipped reference sample (0: skip)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        reference_main(args)
    else:
        gpu_main(args)


if __name__ == "__main__":
    main()
