"""CPU oracle for the quantum-kernel hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline.  The product path (paper_2411_09336_b200) never imports it and
has no CPU fallback.

It restates, in numpy, the reference's algorithm for the path named by
BASELINE.json (paths relative to /root/reference/pkg/src/mpskernel/):

    feature map         ansatz.py:102-136 (edges, build), :139-184 (layer
                        scheduling), :187-215 (SWAP routing), :82-99 (gates)
    MPS simulation      mps.py:90-102 (init), :105-138 (QR canonicalisation),
                        :147-205 (1q / 2q gates), :224-257 (run/simulate)
    truncated SVD       tensor.py:87-123 (noise floor :17, budget tail rule)
    overlap             mps.py:260-268
    Gram                kernel.py:147-185

It calls the same LAPACK routines in the same order as the reference
(np.linalg.qr -> zgeqrf/zungqr, np.linalg.svd -> zgesdd, np.tensordot ->
zgemm), so on the same numpy build its outputs are bitwise identical to the
reference's; tests/test_oracle.py pins that against the golden fixtures in
tests/golden/ that tests/golden/make_golden.py produced by running the
reference itself.  Parity is therefore PINNED (not "unpinned").

Deviations by design: no per-gate unitary check (mps.py:141-144 is pure
validation overhead), no phase timers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NOISE_FLOOR = 10.0 * np.finfo(np.float64).eps  # tensor.py:17
H_GATE = np.array([[1.0, 1.0], [1.0, -1.0]], dtype=np.complex128) / math.sqrt(2.0)  # ansatz.py:76
SWAP_GATE = np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]  # ansatz.py:77-79


# --------------------------------------------------------------------------- circuit
def edges(m: int, d: int) -> list[tuple[int, int]]:
    """interaction_graph (ansatz.py:102-106): grouped by distance, then start."""
    return [(i, i + k) for k in range(1, d + 1) for i in range(m - k)]


def _greedy_layers(run):
    """layered_gates (ansatz.py:139-161): first layer whose qubits are free."""
    layers: list[list] = []
    busy: list[set] = []
    for g in run:
        a, b = g[1], g[2]
        for lay, used in zip(layers, busy):
            if a not in used and b not in used:
                lay.append(g)
                used |= {a, b}
                break
        else:
            layers.append([g])
            busy.append({a, b})
    return [g for lay in layers for g in lay]


def feature_map_gates(x, m: int, r: int, d: int, gamma: float):
    """encode_circuit (ansatz.py:218-220) as a list of (kind, a, b, angle).

    kind in {"H", "RZ", "RXX", "SWAP"}; b = -1 for one-qubit gates.
    """
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (m,):
        raise ValueError(f"expected {m} features, got shape {x.shape}")
    if not np.all(np.isfinite(x)):
        raise ValueError("features must be finite")
    if np.any(x < 0.0) or np.any(x > 2.0):
        raise ValueError("features must lie in [0, 2]; rescale the data first")
    E = edges(m, d)
    built = [("H", q, -1, None) for q in range(m)]
    for _ in range(r):
        built += [("RZ", q, -1, 2.0 * gamma * x[q]) for q in range(m)]  # ansatz.py:130
        built += [
            ("RXX", i, j, 2.0 * gamma**2 * (math.pi / 2.0) * (1.0 - x[i]) * (1.0 - x[j]))  # :132
            for i, j in E
        ]
    # schedule every maximal RXX run (ansatz.py:170-184)
    sched, run = [], []
    for g in built:
        if g[0] == "RXX":
            run.append(g)
            continue
        if run:
            sched += _greedy_layers(run)
            run = []
        sched.append(g)
    if run:
        sched += _greedy_layers(run)
    # route on the line with restoring SWAP ladders (ansatz.py:187-215)
    pos = list(range(m))
    occ = list(range(m))
    out = []

    def swap(p):
        out.append(("SWAP", p, p + 1, None))
        la, lb = occ[p], occ[p + 1]
        occ[p], occ[p + 1] = lb, la
        pos[la], pos[lb] = p + 1, p

    for kind, a, b, ang in sched:
        if b < 0:
            out.append((kind, pos[a], -1, ang))
            continue
        lo, hi = sorted((pos[a], pos[b]))
        for p in range(hi - 1, lo, -1):
            swap(p)
        out.append((kind, lo, lo + 1, ang))
        for p in range(lo + 1, hi):
            swap(p)
    return out


def gate_unitary(kind: str, angle) -> np.ndarray:
    """gate_matrix (ansatz.py:82-99)."""
    if kind == "H":
        return H_GATE
    if kind == "SWAP":
        return SWAP_GATE
    half = 0.5 * angle
    if kind == "RZ":
        return np.diag([np.exp(-1j * half), np.exp(1j * half)]).astype(np.complex128)
    c, s = math.cos(half), -1j * math.sin(half)
    return np.array([[c, 0, 0, s], [0, c, s, 0], [0, s, c, 0], [s, 0, 0, c]], dtype=np.complex128)


# --------------------------------------------------------------------------- SVD
def svd_truncated(mat: np.ndarray, budget: float, chi_max: int = 0):
    """(U, s, Vh, discarded) of tensor.svd_truncated on a matrix (tensor.py:87-123).

    chi_max > 0 is an EXTENSION with no reference counterpart (BASELINE
    config 2 names a chi_max): keep = min(keep, chi_max) after the budget
    rule, the cut weight is discarded and renormalised like any other
    (mps.py:189-192).  Unpinned by reference fixtures by construction."""
    if budget < 0:
        raise ValueError("budget must be non-negative")
    if not np.all(np.isfinite(mat)):
        raise ValueError("tensor has non-finite entries")
    u, s, vh = np.linalg.svd(mat, full_matrices=False)
    if s.size and s[0] > 0.0:
        s = np.where(s < NOISE_FLOOR * s[0], 0.0, s)
    sq = s * s
    tail = np.cumsum(sq[::-1])[::-1]
    cut = np.flatnonzero(tail <= budget)
    keep = max(int(cut[0]) if cut.size else s.size, 1)
    if chi_max > 0:
        keep = min(keep, chi_max)
    return u[:, :keep], s[:keep].copy(), vh[:keep], float(np.sum(sq[keep:]))


# --------------------------------------------------------------------------- MPS
@dataclass
class OracleState:
    sites: list
    discard: float = 0.0
    center: int = 0
    peak: int = 1
    g1: int = 0
    g2: int = 0
    memory: list = field(default_factory=list)

    def bond_dims(self):
        return [t.shape[0] for t in self.sites] + [self.sites[-1].shape[2]]


def _move_center(st: OracleState, target: int) -> None:
    """canonicalize (mps.py:123-138) from a known center."""
    while st.center < target:  # _left_isometrize step (mps.py:105-111)
        i = st.center
        cl, p, cr = st.sites[i].shape
        q, rr = np.linalg.qr(st.sites[i].reshape(cl * p, cr))
        st.sites[i] = q.reshape(cl, p, q.shape[1])
        st.sites[i + 1] = np.tensordot(rr, st.sites[i + 1], axes=(1, 0))
        st.center += 1
    while st.center > target:  # _right_isometrize step (mps.py:114-120)
        i = st.center
        cl, p, cr = st.sites[i].shape
        q, rr = np.linalg.qr(st.sites[i].reshape(cl, p * cr).conj().T)
        st.sites[i] = q.conj().T.reshape(q.shape[1], p, cr)
        st.sites[i - 1] = np.tensordot(st.sites[i - 1], rr.conj().T, axes=(2, 0))
        st.center -= 1


def simulate_gates(gates, m: int, budget: float, record_memory: bool = False, chi_max: int = 0) -> OracleState:
    """simulate_circuit (mps.py:250-257) over a (kind, a, b, angle) list."""
    st = OracleState([np.array([1.0, 0.0], dtype=np.complex128).reshape(1, 2, 1) for _ in range(m)])
    two = [b >= 0 for _, _, b, _ in gates]
    nxt = [None] * (len(gates) + 1)  # lower qubit of the next 2q gate (mps.py:233-236)
    for i in range(len(gates) - 1, -1, -1):
        nxt[i] = min(gates[i][1], gates[i][2]) if two[i] else nxt[i + 1]
    for i, (kind, a, b, ang) in enumerate(gates):
        u = gate_unitary(kind, ang)
        if b < 0:  # apply_one_qubit (mps.py:147-160)
            st.sites[a] = np.tensordot(u, st.sites[a], axes=(1, 1)).transpose(1, 0, 2)
            st.g1 += 1
        else:  # apply_two_qubit (mps.py:163-205)
            q = min(a, b)
            if abs(a - b) != 1:
                raise ValueError("two-qubit gate is not adjacent; route the circuit first")
            if a > b:
                u = u.reshape(2, 2, 2, 2).transpose(1, 0, 3, 2).reshape(4, 4)
            left = nxt[i + 1] is not None and nxt[i + 1] <= q
            _move_center(st, q)
            theta = np.tensordot(st.sites[q], st.sites[q + 1], axes=(2, 0))
            theta = np.tensordot(u.reshape(2, 2, 2, 2), theta, axes=((2, 3), (1, 2)))
            theta = theta.transpose(2, 0, 1, 3)
            cl, cr = theta.shape[0], theta.shape[3]
            U, s, Vh, disc = svd_truncated(theta.reshape(cl * 2, 2 * cr), budget, chi_max)
            k = s.size
            if disc > 0.0:
                kept = float(s @ s)
                s = s * np.sqrt((kept + disc) / kept)
            U = U.reshape(cl, 2, k)
            Vh = Vh.reshape(k, 2, cr)
            if left:
                st.sites[q], st.sites[q + 1], st.center = U * s, Vh, q
            else:
                st.sites[q], st.sites[q + 1], st.center = U, s[:, None, None] * Vh, q + 1
            st.discard += disc
            st.peak = max(st.peak, k)
            st.g2 += 1
        if record_memory:
            st.memory.append(16 * sum(t.size for t in st.sites))
    return st


def simulate_row(x, m: int, r: int, d: int, gamma: float, budget: float, chi_max: int = 0) -> OracleState:
    return simulate_gates(feature_map_gates(x, m, r, d, gamma), m, budget, chi_max=chi_max)


def overlap(bra_sites, ket_sites) -> complex:
    """inner_product (mps.py:260-268)."""
    env = np.ones((1, 1), dtype=np.complex128)
    for a, b in zip(bra_sites, ket_sites):
        env = np.tensordot(np.tensordot(env, a.conj(), axes=(0, 0)), b, axes=((0, 1), (0, 1)))
    return complex(env[0, 0])


def gram(bras, kets, kind: str) -> np.ndarray:
    """compute_gram (kernel.py:147-185) on lists of site lists."""
    if kind == "train":
        n = len(kets)
        K = np.eye(n)
        for i in range(n):
            for j in range(i + 1, n):
                K[i, j] = K[j, i] = abs(overlap(kets[i], kets[j])) ** 2
        return K
    return np.array([[abs(overlap(b, k)) ** 2 for k in kets] for b in bras]).reshape(len(bras), len(kets))


def overlap_flops(bra_chi, ket_chi) -> int:
    """Algorithmic FP64 flops of one inner_product in the reference contraction
    order: sum_s 16 chi^b_s chi^a_{s+1} (chi^a_s + chi^b_{s+1})."""
    a = np.asarray(bra_chi, dtype=np.int64)
    b = np.asarray(ket_chi, dtype=np.int64)
    return int(np.sum(16 * b[:-1] * a[1:] * (a[:-1] + b[1:])))
