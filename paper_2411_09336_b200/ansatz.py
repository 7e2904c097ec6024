"""Feature-map circuits: the host-side half of the drop-in API.

Mirrors the public names of the reference's ``mpskernel.ansatz``
(/root/reference/pkg/src/mpskernel/ansatz.py) so callers switch by import.
The data-independent topology of ``encode_circuit`` (gate kinds, qubits,
angle slots) and the per-row angle tables come from the native runtime
(libmpskq: mpskq_feature_map_topology / mpskq_feature_map_angles), which the
GPU simulator consumes directly; the Python objects here exist for API
parity and for arbitrary user circuits.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as N

GATE_KINDS = ("H", "RZ", "RXX", "SWAP")  # ansatz.py:15
TWO_QUBIT = frozenset({"RXX", "SWAP"})
PARAMETRIC = frozenset({"RZ", "RXX"})


@dataclass(frozen=True)
class FeatureMapConfig:
    """m qubits/features, r layer repetitions, d interaction distance, gamma
    bandwidth (ansatz.py:20-41)."""

    m: int
    r: int
    d: int
    gamma: float

    def __post_init__(self):
        if self.m < 1:
            raise ValueError("m must be at least 1")
        if self.r < 1:
            raise ValueError("r must be at least 1")
        if not 1 <= self.d <= self.m - 1:
            raise ValueError(f"d must satisfy 1 <= d <= m-1, got d={self.d} for m={self.m}")
        if not self.gamma > 0:
            raise ValueError("gamma must be positive")


@dataclass(frozen=True)
class Gate:
    """One gate; ``angle`` only for RZ/RXX (ansatz.py:44-62)."""

    kind: str
    qubits: tuple
    angle: float | None = None

    def __post_init__(self):
        if self.kind not in GATE_KINDS:
            raise ValueError(f"unknown gate kind {self.kind!r}")
        want = 2 if self.kind in TWO_QUBIT else 1
        if len(self.qubits) != want:
            raise ValueError(f"{self.kind} acts on exactly {want} qubit(s)")
        needs = self.kind in PARAMETRIC
        if needs and self.angle is None:
            raise ValueError(f"{self.kind} requires an angle")
        if not needs and self.angle is not None:
            raise ValueError(f"{self.kind} takes no angle")
        object.__setattr__(self, "qubits", tuple(int(q) for q in self.qubits))
        if self.angle is not None:
            object.__setattr__(self, "angle", float(self.angle))


@dataclass
class Circuit:
    m: int
    gates: list = field(default_factory=list)

    def __post_init__(self):
        for g in self.gates:
            if any(q < 0 or q >= self.m for q in g.qubits):
                raise ValueError(f"gate {g} addresses a qubit outside 0..{self.m - 1}")


def gate_matrix(gate: Gate) -> np.ndarray:
    """Unitary of a gate in the |q0 q1> basis (ansatz.py:82-99):
    H, RZ(t) = exp(-i t Z/2), RXX(t) = exp(-i t XX/2), SWAP."""
    if gate.kind == "H":
        return np.array([[1.0, 1.0], [1.0, -1.0]], dtype=np.complex128) / math.sqrt(2.0)
    if gate.kind == "SWAP":
        return np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]
    h = 0.5 * gate.angle
    if gate.kind == "RZ":
        return np.diag([np.exp(-1j * h), np.exp(1j * h)]).astype(np.complex128)
    c, s = math.cos(h), -1j * math.sin(h)
    out = np.zeros((4, 4), dtype=np.complex128)
    out[[0, 1, 2, 3], [0, 1, 2, 3]] = c
    out[[0, 1, 2, 3], [3, 2, 1, 0]] = s
    return out


def interaction_graph(m: int, d: int) -> list:
    """Chain edges (i, i+k), 1 <= k <= d, grouped by k (ansatz.py:102-106)."""
    if not 1 <= d <= m - 1:
        raise ValueError(f"d must satisfy 1 <= d <= m-1, got d={d} for m={m}")
    return [(i, i + k) for k in range(1, d + 1) for i in range(m - k)]


def _check_row(x, m: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1 or x.size != m:
        raise ValueError(f"expected {m} features, got shape {x.shape}")
    if not np.all(np.isfinite(x)):
        raise ValueError("features must be finite")
    if np.any((x < 0.0) | (x > 2.0)):
        raise ValueError("features must lie in [0, 2]; rescale the data first")
    return x


def build_circuit(x, cfg: FeatureMapConfig, drop_zero_rxx: bool = False) -> Circuit:
    """H on every qubit, then r x (RZ layer + one RXX per edge) (ansatz.py:109-136)."""
    x = _check_row(x, cfg.m)
    angles = feature_map_angles(x[None, :], cfg)[0]
    E = interaction_graph(cfg.m, cfg.d)
    gates = [Gate("H", (q,)) for q in range(cfg.m)]
    per = cfg.m + len(E)
    for layer in range(cfg.r):
        a = angles[layer * per : (layer + 1) * per]
        gates += [Gate("RZ", (q,), a[q]) for q in range(cfg.m)]
        gates += [
            Gate("RXX", e, a[cfg.m + k])
            for k, e in enumerate(E)
            if not (drop_zero_rxx and a[cfg.m + k] == 0.0)
        ]
    return Circuit(cfg.m, gates)


def layered_gates(c: Circuit, d: int) -> list:
    """Greedy first-fit packing of a commuting RXX run into <= 2d layers
    (ansatz.py:139-161)."""
    layers: list = []
    for g in c.gates:
        if g.kind != "RXX":
            raise ValueError(f"layer scheduling expects RXX gates only, got {g.kind}")
        slot = next((lay for lay in layers if not (lay[0] & set(g.qubits))), None)
        if slot is None:
            layers.append([set(g.qubits), [g]])
        else:
            slot[0].update(g.qubits)
            slot[1].append(g)
    if len(layers) > 2 * d:
        raise AssertionError(f"greedy scheduling used {len(layers)} > 2d = {2 * d} layers")
    return [lay[1] for lay in layers]


def schedule_layers(c: Circuit, d: int) -> Circuit:
    return Circuit(c.m, [g for lay in layered_gates(c, d) for g in lay])


def schedule_circuit(c: Circuit, d: int) -> Circuit:
    """Layer-schedule every maximal run of RXX gates (ansatz.py:170-184)."""
    out, run = [], []
    for g in c.gates + [None]:
        if g is not None and g.kind == "RXX":
            run.append(g)
            continue
        if run:
            out += schedule_layers(Circuit(c.m, run), d).gates
            run = []
        if g is not None:
            out.append(g)
    return Circuit(c.m, out)


def route_linear(c: Circuit) -> Circuit:
    """Bring every 2q gate onto neighbours with a SWAP ladder and undo it
    right after, tracking the logical->physical map (ansatz.py:187-215)."""
    where = list(range(c.m))  # logical -> physical
    who = list(range(c.m))  # physical -> logical
    out: list = []

    def ladder(ps):
        for p in ps:
            out.append(Gate("SWAP", (p, p + 1)))
            a, b = who[p], who[p + 1]
            who[p], who[p + 1] = b, a
            where[a], where[b] = p + 1, p

    for g in c.gates:
        if len(g.qubits) == 1:
            out.append(replace(g, qubits=(where[g.qubits[0]],)))
            continue
        lo, hi = sorted(where[q] for q in g.qubits)
        ladder(range(hi - 1, lo, -1))
        out.append(replace(g, qubits=(lo, lo + 1)))
        ladder(range(lo + 1, hi))
    return Circuit(c.m, out)


# ---------------------------------------------------------------- native topology
@dataclass(frozen=True)
class Topology:
    """Row-independent gate sequence of encode_circuit for one config."""

    m: int
    kinds: np.ndarray  # int32 (GATE_KINDS index)
    q0: np.ndarray
    q1: np.ndarray  # -1 for 1q gates
    param_slot: np.ndarray  # -1 for unparametrised gates
    n_params: int


@functools.lru_cache(maxsize=64)
def feature_map_topology(m: int, r: int, d: int) -> Topology:
    lib = N.lib()
    ng, npar = N.C.c_int64(0), N.C.c_int64(0)
    N.check(lib.mpskq_feature_map_topology(m, r, d, None, None, None, None, 0, N.C.byref(ng), N.C.byref(npar)))
    arr = [np.zeros(ng.value, dtype=np.int32) for _ in range(4)]
    N.check(
        lib.mpskq_feature_map_topology(
            m, r, d, *(N.ptr(a, N.C.c_int32) for a in arr), ng.value, N.C.byref(ng), N.C.byref(npar)
        )
    )
    for a in arr:
        a.setflags(write=False)
    return Topology(m, arr[0], arr[1], arr[2], arr[3], int(npar.value))


def feature_map_angles(X, cfg: FeatureMapConfig) -> np.ndarray:
    """Angle table (n_rows x n_params) in the reference's expression order."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    topo = feature_map_topology(cfg.m, cfg.r, cfg.d)
    out = np.empty((X.shape[0], topo.n_params), dtype=np.float64)
    N.check(
        N.lib().mpskq_feature_map_angles(
            N.ptr(X, N.C.c_double), X.shape[0], cfg.m, cfg.r, cfg.d, float(cfg.gamma), N.ptr(out, N.C.c_double)
        )
    )
    return out


def half_angle_coefficients(angles: np.ndarray) -> np.ndarray:
    """(cos(a/2), sin(a/2)) pairs for every angle, host libm."""
    a = np.ascontiguousarray(angles, dtype=np.float64)
    out = np.empty(a.shape + (2,), dtype=np.float64)
    N.check(N.lib().mpskq_half_angle_coefficients(N.ptr(a, N.C.c_double), a.size, N.ptr(out, N.C.c_double)))
    return out


def encode_circuit(x, cfg: FeatureMapConfig) -> Circuit:
    """route_linear(schedule_circuit(build_circuit(x, cfg), cfg.d)) (ansatz.py:218-220),
    materialised from the native topology and angle table."""
    x = _check_row(x, cfg.m)
    topo = feature_map_topology(cfg.m, cfg.r, cfg.d)
    ang = feature_map_angles(x[None, :], cfg)[0]
    gates = []
    for k, a, b, s in zip(topo.kinds, topo.q0, topo.q1, topo.param_slot):
        kind = GATE_KINDS[k]
        qubits = (int(a),) if b < 0 else (int(a), int(b))
        gates.append(Gate(kind, qubits, float(ang[s]) if s >= 0 else None))
    return Circuit(cfg.m, gates)


def circuit_topology(circuit: Circuit) -> tuple:
    """(Topology, angle vector) of an arbitrary circuit for the GPU simulator."""
    n = len(circuit.gates)
    kinds = np.empty(n, dtype=np.int32)
    q0 = np.empty(n, dtype=np.int32)
    q1 = np.full(n, -1, dtype=np.int32)
    slot = np.full(n, -1, dtype=np.int32)
    angles = []
    for i, g in enumerate(circuit.gates):
        kinds[i] = GATE_KINDS.index(g.kind)
        q0[i] = g.qubits[0]
        if len(g.qubits) == 2:
            q1[i] = g.qubits[1]
        if g.angle is not None:
            slot[i] = len(angles)
            angles.append(g.angle)
    topo = Topology(circuit.m, kinds, q0, q1, slot, len(angles))
    return topo, np.array(angles, dtype=np.float64)
