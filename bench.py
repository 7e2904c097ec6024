#!/usr/bin/env python
"""Headline benchmark: the 165-qubit, N=6400 train kernel matrix.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[3] / SURVEY.md 8(d) row 4): m=165 qubits,
interaction distance d=1, 2 layers, gamma=0.1, per-gate budget 1e-24,
N=6400 synthetic rows uniform in [0, 2] (seed 0).  One step = encode every
row, simulate every MPS, fill the whole train kernel (20,476,800 computed
entries; diagonal and mirror are free) — on N GPUs the rows are sharded,
the MPS all-gathered once over NCCL and the tiles split block-cyclically
(total work fixed: strong scaling).

`value` is entries/s with the feature rows already in HBM; `e2e` is the same
metric through the C ABI (mpskq_gram_host: pinned host rows in, pinned host K
out, copies inside the timed region) at N=1 and through the public
run_distributed API at N>1.  The reference arm (--impl reference) times the
CPU oracle (a numpy restatement of the reference that is bitwise identical
to it, oracle/mps_oracle.py) on every host core over a bounded sample and
projects the same metric.
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
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200 import _native as N
    from paper_2411_09336_b200.ansatz import feature_map_topology
    from paper_2411_09336_b200.distributed import _all_reduce_max, _reduce_sum_to0, allgather_rows, shard
    from paper_2411_09336_b200.kernel import encode_device, simulate_rows
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
    mx = max(counts)
    nccl = world > 1 and dist.get_backend() == "nccl"
    if nccl:
        pad_sites = torch.zeros((mx, 2 * stride), dtype=torch.float64, device=dev)
        pad_chi = torch.ones((mx, M + 1), dtype=torch.int32, device=dev)
        g_sites = torch.empty((world * mx, 2 * stride), dtype=torch.float64, device=dev)
        g_chi = torch.empty((world * mx, M + 1), dtype=torch.int32, device=dev)
    if world > 1:
        sites_all = torch.empty((n, 2 * stride), dtype=torch.float64, device=dev)
        chi_all = torch.empty((n, M + 1), dtype=torch.int32, device=dev)
    else:
        sites_all, chi_all = sites_loc, chi_loc
    K = torch.empty((n, n), dtype=torch.float64, device=dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    # ours per step: encode, simulate, ket key, chi=4 clustering, block bounds, inverse
    # order, pack bras, pack kets, overlap, un-permute, diagonal (rank 0); the ket
    # key sort is CUB's radix sort (library, not counted)
    launches_per_step = 10 + (1 if rank == 0 else 0)

    def step(e):
        e[0].record()
        N.check(lib.mpskq_feature_map_coefficients_device(X_loc.data_ptr(), nloc, M, R, D, GAMMA, coef.data_ptr(),
                                                          bad.data_ptr(), sp))
        N.check(lib.mpskq_simulate(M, cap, ops.data_ptr(), prog.ops.shape[0], prog.n_gates, coef.data_ptr(),
                                   prog.n_params, nloc, BUDGET, 0, off_d.data_ptr(), stride, sites_loc.data_ptr(),
                                   chi_loc.data_ptr(), disc.data_ptr(), peak.data_ptr(), status.data_ptr(), None, sp))
        e[1].record()
        if nccl:  # the one exchange: all-gather of the packed MPS + bond dims
            pad_sites[:nloc].copy_(sites_loc)
            pad_chi[:nloc].copy_(chi_loc)
            dist.all_gather_into_tensor(g_sites, pad_sites)
            dist.all_gather_into_tensor(g_chi, pad_chi)
            o = 0
            for r, c in enumerate(counts):
                sites_all[o : o + c].copy_(g_sites[r * mx : r * mx + c])
                chi_all[o : o + c].copy_(g_chi[r * mx : r * mx + c])
                o += c
        elif world > 1:
            sites_all.copy_(allgather_rows(sites_loc, counts))
            chi_all.copy_(allgather_rows(chi_loc, counts))
        if world > 1:
            K.zero_()
        e[2].record()
        N.check(lib.mpskq_overlap(N.KIND_TRAIN, N.OUT_KERNEL, M, cap, off_d.data_ptr(), stride, sites_all.data_ptr(),
                                  chi_all.data_ptr(), n, sites_all.data_ptr(), chi_all.data_ptr(), n, rank, world,
                                  K.data_ptr(), n, sp))
        e[3].record()
        if nccl:
            dist.reduce(K, dst=0, op=dist.ReduceOp.SUM)
        elif world > 1:
            K.copy_(_reduce_sum_to0(K))
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
    spot = None
    if rank == 0:
        from oracle import mps_oracle as O

        sub = [O.simulate_row(x, M, R, D, GAMMA, BUDGET) for x in X[:6]]
        Ko = O.gram([s.sites for s in sub], [s.sites for s in sub], "train")
        spot = float(np.abs(K[:6, :6].cpu().numpy() - Ko).max())
        chi_ok = bool(np.array_equal(chi_all[:6].cpu().numpy(), np.array([s.bond_dims() for s in sub])))

    # e2e through the host-buffer entry points
    e2e = None
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
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        a.record()
        for _ in range(args.steps):
            host_call()
        b.record()
        b.synchronize()
        e2e_ms = a.elapsed_time(b) / args.steps
        wall_ms = 1e3 * (time.perf_counter() - w0) / args.steps
        e2e = {"value": n * (n - 1) / 2 / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": X.nbytes,
               "d2h_bytes_per_step": n * n * 8, "ms_per_step": e2e_ms, "host_wall_ms_per_step": wall_ms,
               "path": "C ABI mpskq_gram_host (pinned host rows -> pinned host K, row bands streamed "
                       "to host under the overlap)",
               "k_bitwise_equal_device_path": bool(torch.equal(Kp, K.cpu()))}
    else:
        sched = P.make_schedule(n, n, world, "round_robin", "train")
        for _ in range(max(1, args.warmup)):
            P.run_distributed(X, X, cfg, sched, budget=BUDGET)
        dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            P.run_distributed(X, X, cfg, sched, budget=BUDGET)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([(time.perf_counter() - w0) / args.steps], dtype=torch.float64, device=dev)
        e2e_ms = 1e3 * _all_reduce_max(t).item()
        e2e = {"value": n * (n - 1) / 2 / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": X.nbytes,
               "d2h_bytes_per_step": n * n * 8, "ms_per_step": e2e_ms,
               "path": "public API run_distributed (host rows -> host K on rank 0), max over ranks"}

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
        "config": {
            "workload": WORKLOAD,
            "m": M, "d": D, "layers": R, "gamma": GAMMA, "budget": BUDGET, "N": n,
            "computed_entries": int(entries),
            "parallelism": f"rows sharded x{world}, MPS all-gathered once, tiles block-cyclic",
            "l2": "working set (540 MB padded MPS + 328 MB K) larger than L2; no flush needed",
            "chi_cap": cap,
        },
        "train_wall_s": ms / 1e3,
        "mps_states_per_s": n / (sim_ms / 1e3),
        "phases_ms": {"simulate": sim_ms, "all_gather": comm_ms, "overlap": ov_ms, "reduce": red_ms},
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
        "gpu_launches": launches_per_step * args.steps,
        "parity_spot_check": {"max_abs_err_vs_oracle_6x6": spot, "bond_dims_equal": chi_ok},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ reference arm
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
        "config": {"workload": WORKLOAD, "m": M, "d": D, "layers": R, "gamma": GAMMA, "budget": BUDGET, "N": n,
                   "computed_entries": n * (n - 1) // 2},
        "train_wall_s": float(np.median(walls)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": s["cores"], "kind": "port", "sample": s["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference is pure Python/numpy (nothing to compile); timed through oracle/mps_oracle.py, "
                "which is bitwise identical to it (tests/test_oracle.py)",
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--rows", type=int, default=6400, help="N feature rows (train kernel N x N)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        reference_main(args)
    else:
        gpu_main(args)


if __name__ == "__main__":
    main()
