"""Kernel (Gram) matrices on the GPU — drop-in for ``mpskernel.kernel``.

Reference: /root/reference/pkg/src/mpskernel/kernel.py.  Same names,
signatures, defaults, result types and error messages.  Underneath:

* ``simulate_dataset`` (kernel.py:128-135) simulates every row at once with
  the batched GPU engine and returns a device-resident ``MpsBatch`` (a
  sequence of ``MpsState``).
* ``compute_gram`` (kernel.py:147-185) runs the tiled overlap kernel; train
  computes i<j once, mirrors bit-exactly and fixes the diagonal to 1.
* ``run_distributed`` (kernel.py:443-512) accepts the reference's tile
  schedules for API parity, simulates each state exactly once and computes
  the whole matrix on the GPU(s).  Under ``torch.distributed`` it shards the
  simulation by row, all-gathers the MPS once and splits tiles
  block-cyclically (``distributed.py``).
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .ansatz import FeatureMapConfig, feature_map_angles, feature_map_topology, half_angle_coefficients
from .mps import DEFAULT_TRUNC_BUDGET, MpsBatch, MpsState, compile_program, overlap_matrix_host, simulate_program

STRATEGIES = ("no_messaging", "round_robin")
KINDS = ("train", "test")


@dataclass
class GramMatrix:
    """``train``: square symmetric; ``test``: test rows x train columns (kernel.py:34-47)."""

    entries: np.ndarray
    kind: str

    @property
    def rows(self) -> int:
        return self.entries.shape[0]

    @property
    def cols(self) -> int:
        return self.entries.shape[1]


@dataclass(frozen=True)
class Tile:
    worker: int
    row_start: int
    row_stop: int
    col_start: int
    col_stop: int


@dataclass(frozen=True)
class Transfer:
    src: int
    dst: int
    which: str
    start: int
    stop: int


@dataclass
class ScheduleStep:
    tiles: list = field(default_factory=list)
    transfers: list = field(default_factory=list)


@dataclass
class TileSchedule:
    strategy: str
    kind: str
    k: int
    n_bras: int
    n_kets: int
    initial_states: dict
    steps: list


@dataclass
class RunReport:
    """Counters and phase seconds (kernel.py:94-110); GPU phases are CUDA-event times."""

    n_simulations: int = 0
    n_inner_products: int = 0
    seconds: dict = field(
        default_factory=lambda: {"simulation": 0.0, "inner_products": 0.0, "communication": 0.0, "merge": 0.0}
    )

    def _add(self, phase: str, dt: float) -> None:
        self.seconds[phase] = self.seconds.get(phase, 0.0) + dt


# ---------------------------------------------------------------- schedules
def _split(n: int, parts: int) -> list:
    """range(n) in `parts` contiguous blocks, the first n % parts one longer."""
    q, rem = divmod(n, parts)
    sizes = [q + (i < rem) for i in range(parts)]
    starts = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    return [(int(starts[i]), int(starts[i + 1])) for i in range(parts)]


def _train_round_robin(n: int, k: int) -> TileSchedule:
    """Circle-method tournament over 2k half-blocks (kernel.py:188-232): worker
    w starts with half-blocks in slots w and 2k-1-w; slot 2k-1 is fixed and the
    others rotate one slot per round, so every half-block pair meets once."""
    halves = []
    for a, b in _split(n, k):
        mid = a + (b - a + 1) // 2
        halves += [(a, mid), (mid, b)]
    slots = 2 * k
    start_slot = {}
    for w in range(k):
        start_slot[2 * w] = w
        start_slot[2 * w + 1] = slots - 1 - w

    def owner(u: int, t: int) -> int:
        s = start_slot[u]
        if s != slots - 1:
            s = (s + t) % (slots - 1)
        return s if s < k else slots - 1 - s

    rounds = slots - 1 if k > 1 else 1
    steps = []
    for t in range(rounds):
        step = ScheduleStep()
        if t:
            step.transfers = [
                Transfer(owner(u, t - 1), owner(u, t), "ket", a, b)
                for u, (a, b) in enumerate(halves)
                if a < b and owner(u, t - 1) != owner(u, t)
            ]
        held = {w: [] for w in range(k)}
        for u in range(len(halves)):
            held[owner(u, t)].append(halves[u])
        for w, (h1, h2) in held.items():
            if t == 0:
                step.tiles.append(Tile(w, h1[0], h2[1], h1[0], h2[1]))
            elif h1[0] < h1[1] and h2[0] < h2[1]:
                lo, hi = sorted([h1, h2])
                step.tiles.append(Tile(w, lo[0], lo[1], hi[0], hi[1]))
        steps.append(step)
    return TileSchedule("round_robin", "train", k, n, n, {w: [("ket", *blk)] for w, blk in enumerate(_split(n, k))}, steps)


def _test_round_robin(n_bras: int, n_kets: int, k: int) -> TileSchedule:
    """Each worker owns a train block; the test set is cut into ell blocks that
    rotate among the first ell workers while the rest receive copies
    (kernel.py:235-266)."""
    ell = min(max(1, round(k * n_bras / n_kets)), k, n_bras)
    kb = _split(n_kets, k)
    bb = _split(n_bras, ell)
    initial = {w: [("ket", *kb[w])] for w in range(k)}
    for b in range(ell):
        initial[b].append(("bra", *bb[b]))
    steps = []
    for t in range(ell):
        step = ScheduleStep()
        if t:
            for a in range(ell):
                dst = (a - 1) % ell
                if dst != a:
                    step.transfers.append(Transfer(a, dst, "bra", *bb[(a + t - 1) % ell]))
        for w in range(ell, k):
            a = w % ell
            src = (a + 1) % ell if t else a
            if src != w:
                step.transfers.append(Transfer(src, w, "bra", *bb[(a + t) % ell]))
        step.tiles = [Tile(w, *bb[(w % ell + t) % ell], *kb[w]) for w in range(k)]
        steps.append(step)
    return TileSchedule("round_robin", "test", k, n_bras, n_kets, initial, steps)


def _no_messaging(n_bras: int, n_kets: int, k: int, kind: str) -> TileSchedule:
    """Independent tiles; workers simulate what they touch (kernel.py:269-313)."""
    if kind == "train":
        g = 1
        while g * (g + 1) // 2 < k:
            g += 1
        blocks = _split(n_kets, min(g, n_kets))
        cells = [(i, j) for i in range(len(blocks)) for j in range(i, len(blocks))]
        tiles = [Tile(t % k, *blocks[i], *blocks[j]) for t, (i, j) in enumerate(cells)]
    else:
        best = None
        for gr in range(1, n_bras + 1):  # grid with >= k tiles closest to square tiles
            gc = min(max(1, -(-k // gr)), n_kets)
            key = (gr * gc < k, abs(np.log((n_bras / gr) / (n_kets / gc))), gr * gc, gr)
            if best is None or key < best[0]:
                best = (key, gr, gc)
        rb, cb = _split(n_bras, best[1]), _split(n_kets, best[2])
        cells = [(i, j) for i in range(len(rb)) for j in range(len(cb))]
        tiles = [Tile(t % k, *rb[i], *cb[j]) for t, (i, j) in enumerate(cells)]
    initial = {}
    for w in range(k):
        mine = [t for t in tiles if t.worker == w]
        cols = {(t.col_start, t.col_stop) for t in mine}
        rows = {(t.row_start, t.row_stop) for t in mine}
        if kind == "train":
            initial[w] = [("ket", a, b) for a, b in sorted(cols | rows)]
        else:
            initial[w] = [("bra", a, b) for a, b in sorted(rows)] + [("ket", a, b) for a, b in sorted(cols)]
    return TileSchedule("no_messaging", kind, k, n_bras, n_kets, initial, [ScheduleStep(tiles=tiles)])


def make_schedule(n_bras: int, n_kets: int, k: int, strategy: str, kind: str) -> TileSchedule:
    """Tile schedule covering every required entry once (kernel.py:316-333)."""
    if strategy not in STRATEGIES:
        raise ValueError(f"strategy must be one of {STRATEGIES}")
    if kind not in KINDS:
        raise ValueError(f"kind must be one of {KINDS}")
    if kind == "train" and n_bras != n_kets:
        raise ValueError("train kind requires equal bra and ket counts")
    if k < 1:
        raise ValueError("worker count must be at least 1")
    if n_kets < 1 or n_bras < 1:
        raise ValueError("state counts must be at least 1")
    k = min(k, n_kets)
    if strategy == "no_messaging":
        return _no_messaging(n_bras, n_kets, k, kind)
    return _train_round_robin(n_kets, k) if kind == "train" else _test_round_robin(n_bras, n_kets, k)


def validate_schedule(schedule: TileSchedule) -> None:
    """Exact single coverage plus per-strategy simulation invariants (kernel.py:336-367)."""
    cover = np.zeros((schedule.n_bras, schedule.n_kets), dtype=np.int64)
    train = schedule.kind == "train"
    for step in schedule.steps:
        for t in step.tiles:
            block = np.ones((t.row_stop - t.row_start, t.col_stop - t.col_start), dtype=np.int64)
            if train and (t.row_start, t.row_stop) == (t.col_start, t.col_stop):
                block = np.triu(block, k=1)
            cover[t.row_start : t.row_stop, t.col_start : t.col_stop] += block
    need = np.triu(np.ones_like(cover), k=1) if train else np.ones_like(cover)
    if not np.array_equal(cover * need, need):
        raise AssertionError("schedule does not cover every required entry exactly once")
    if np.any(cover * (1 - need)):
        raise AssertionError("schedule covers entries outside the required region")
    sims = np.zeros(schedule.n_bras + schedule.n_kets, dtype=np.int64)
    for ranges in schedule.initial_states.values():
        for which, a, b in ranges:
            base = 0 if which == "bra" else schedule.n_bras
            sims[base + a : base + b] += 1
    needed = sims if schedule.kind == "test" else sims[schedule.n_bras :]
    if schedule.strategy == "round_robin" and not np.all(needed == 1):
        raise AssertionError("round_robin must simulate each state exactly once")
    if np.any(needed < 1):
        raise AssertionError("some state is never simulated")


# ---------------------------------------------------------------- GPU path
def _check_rows(X, m: int) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.size == 0:
        return X.reshape(0, m)
    if X.ndim != 2 or X.shape[1] != m:
        raise ValueError(f"expected feature rows of length {m}, got shape {X.shape}")
    return X


def simulate_rows(X: np.ndarray, cfg: FeatureMapConfig, budget: float, chi_max: int = 0,
                  chi_cap: int | None = None) -> MpsBatch:
    """One feature-map MPS per row on the GPU (the engine behind simulate_dataset)."""
    from ._device import require_cuda

    require_cuda()
    topo = feature_map_topology(cfg.m, cfg.r, cfg.d)
    prog = compile_program(topo)
    X = np.ascontiguousarray(X, dtype=np.float64)
    if not np.all(np.isfinite(X)):
        raise ValueError("features must be finite")
    if np.any((X < 0.0) | (X > 2.0)):
        raise ValueError("features must lie in [0, 2]; rescale the data first")
    coef, _ = encode_device(torch.from_numpy(X).to("cuda"), cfg)
    return simulate_program(prog, coef, budget, chi_max=chi_max, chi_cap=chi_cap)


def encode_device(X_dev, cfg: FeatureMapConfig):
    """(n, n_params, 2) half-angle cos/sin table computed on the GPU from device rows."""
    from . import _native as N
    from ._device import dptr, require_cuda, stream_ptr

    require_cuda()
    topo = feature_map_topology(cfg.m, cfg.r, cfg.d)
    X_dev = X_dev.to(torch.float64).contiguous()
    n = X_dev.shape[0]
    coef = torch.empty((n, topo.n_params, 2), dtype=torch.float64, device=X_dev.device)
    bad = torch.zeros(1, dtype=torch.int32, device=X_dev.device)
    N.check(N.lib().mpskq_feature_map_coefficients_device(dptr(X_dev), n, cfg.m, cfg.r, cfg.d, float(cfg.gamma),
                                                          dptr(coef), dptr(bad), stream_ptr()))
    return coef, bad


def simulate_dataset(X, cfg: FeatureMapConfig, budget: float = DEFAULT_TRUNC_BUDGET):
    """Encode and simulate one MPS per data row (kernel.py:128-135)."""
    X = _check_rows(X, cfg.m)
    if not np.all(np.isfinite(X)):
        raise ValueError("features must be finite")
    if X.shape[0] == 0:
        return []
    return simulate_rows(X, cfg, budget)


def _to_batch(states) -> MpsBatch:
    return states if isinstance(states, MpsBatch) else MpsBatch.from_states(states)


def compute_gram(bras, kets, kind: str, report: RunReport | None = None) -> GramMatrix:
    """Gram matrix of |<bra_i|ket_j>|^2 (kernel.py:147-185)."""
    if kind not in KINDS:
        raise ValueError(f"kind must be one of {KINDS}")
    if kind == "train":
        same = bras is kets or (isinstance(bras, MpsBatch) and bras.same_states(kets)) or (
            not isinstance(bras, MpsBatch) and not isinstance(kets, MpsBatch) and len(bras) == len(kets)
            and all(a is b for a, b in zip(bras, kets))
        )
        if not same:
            raise ValueError("train kind requires bras and kets to be the same states")
    if len(bras) and len(kets) and _m_of(bras) != _m_of(kets):
        raise ValueError("qubit count mismatch between state lists")
    nb, nk = len(bras), len(kets)
    if nb == 0 or nk == 0:
        K = np.eye(nk) if kind == "train" else np.empty((nb, nk))
        return GramMatrix(K, kind)
    t0 = time.perf_counter()
    b = _to_batch(bras)
    k = b if kind == "train" else _to_batch(kets)
    K = overlap_matrix_host(b, k, kind)
    count = nk * (nk - 1) // 2 if kind == "train" else nb * nk
    if report is not None:
        report.n_inner_products += count
        report._add("inner_products", time.perf_counter() - t0)
    return GramMatrix(K, kind)


def _m_of(states) -> int:
    return states.m if isinstance(states, MpsBatch) else states[0].m


def run_distributed(X_bras, X_kets, cfg: FeatureMapConfig, schedule: TileSchedule,
                    budget: float = DEFAULT_TRUNC_BUDGET, report: RunReport | None = None) -> GramMatrix:
    """The reference's distributed executor (kernel.py:443-512) on the GPU.

    Every state is simulated exactly once (the schedule's coverage is
    validated; its worker count only sets how the reference would have
    split the work).  With torch.distributed initialised on several ranks the
    work is sharded across GPUs and rank 0 receives the matrix; other ranks
    get an empty GramMatrix of the right kind.
    """
    X_bras = _check_rows(X_bras, cfg.m)
    X_kets = _check_rows(X_kets, cfg.m)
    if (X_bras.shape[0], X_kets.shape[0]) != (schedule.n_bras, schedule.n_kets):
        raise ValueError("schedule was built for different state counts")
    same = X_bras is X_kets or (X_bras.shape == X_kets.shape and X_bras.ctypes.data == X_kets.ctypes.data
                                and X_bras.strides == X_kets.strides)
    if schedule.kind == "train" and not same and not np.array_equal(X_bras, X_kets):
        raise ValueError("train kind requires identical bra and ket rows")
    # finiteness and the [0, 2] range are checked where the rows are encoded
    # (the device encoder on one GPU, simulate_rows on several), with the
    # reference's messages (kernel.py:138-144, ansatz.py:121-124)
    from . import distributed

    try:
        K, rep = distributed.gram(X_bras, X_kets, cfg, schedule.kind, budget)
    except ValueError:
        raise
    except Exception as exc:  # surfaced like the reference's worker failure
        raise RuntimeError("worker failed during distributed run") from exc
    if report is not None:
        report.n_simulations += rep.n_simulations
        report.n_inner_products += rep.n_inner_products
        for phase, dt in rep.seconds.items():
            report._add(phase, dt)
    return GramMatrix(K, schedule.kind)


# ---------------------------------------------------------------- persistence
def save_gram(gram: GramMatrix, csv_path, sidecar: dict | None = None) -> None:
    """CSV with 17 significant digits plus an optional JSON sidecar (kernel.py:515-527)."""
    np.savetxt(csv_path, np.atleast_2d(gram.entries), delimiter=",", fmt="%.17g")
    if sidecar is not None:
        meta = {"kind": gram.kind, "rows": gram.rows, "cols": gram.cols, **sidecar}
        with open(str(csv_path) + ".json", "w", encoding="utf-8") as fh:
            json.dump(meta, fh, indent=2, sort_keys=True)
            fh.write("\n")


def load_gram(csv_path, kind: str) -> GramMatrix:
    return GramMatrix(np.loadtxt(csv_path, delimiter=",", dtype=np.float64, ndmin=2), kind)
