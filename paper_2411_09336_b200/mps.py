"""MPS states and the GPU simulation / overlap entry points.

Drop-in for the hot-path names of the reference's ``mpskernel.mps``
(/root/reference/pkg/src/mpskernel/mps.py):

* ``MpsState`` / ``SimStats`` / ``stats`` / ``init_state`` / ``to_statevector``
  are host-side containers and helpers with the reference's fields.
* ``simulate_circuit`` (mps.py:250-257) and ``inner_product`` (mps.py:260-268)
  run on the GPU through libmpskq.
* ``MpsBatch`` is the device-resident batch the GPU path produces: a
  sequence whose items are ``MpsState`` views (copied to the host on access)
  with site arrays in the reference layout.
"""

from __future__ import annotations

import functools
import struct
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._device import Timer, dptr, require_cuda, stream_ptr
from .ansatz import Circuit, Topology, circuit_topology, half_angle_coefficients

DEFAULT_TRUNC_BUDGET = 1e-24  # mps.py:25
_MAX_DENSE_QUBITS = 20


@dataclass
class MpsState:
    """Chain of (chi_l, 2, chi_r) site tensors plus truncation bookkeeping (mps.py:31-77)."""

    sites: list
    trunc_budget_per_gate: float = DEFAULT_TRUNC_BUDGET
    accumulated_discard: float = 0.0
    ortho_center: int | None = None
    peak_chi: int = 1
    gate_count_1q: int = 0
    gate_count_2q: int = 0
    timings: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return len(self.sites)

    def bond_dims(self) -> list:
        return [t.shape[0] for t in self.sites] + [self.sites[-1].shape[2]]

    def max_bond(self) -> int:
        return max(self.bond_dims())

    def entry_count(self) -> int:
        return sum(t.size for t in self.sites)

    def copy(self) -> "MpsState":
        return MpsState(
            [t.copy() for t in self.sites], self.trunc_budget_per_gate, self.accumulated_discard,
            self.ortho_center, self.peak_chi, self.gate_count_1q, self.gate_count_2q, dict(self.timings),
        )


@dataclass(frozen=True)
class SimStats:
    max_chi: int
    entry_count: int
    memory_bytes: int
    gate_count_1q: int
    gate_count_2q: int
    wall_time_per_phase: dict


def init_state(m: int, basis: str = "zero", trunc_budget_per_gate: float = DEFAULT_TRUNC_BUDGET) -> MpsState:
    """|0...0> or |+>^m product state (mps.py:90-102)."""
    if m < 1:
        raise ValueError("qubit count must be at least 1")
    vecs = {"zero": [1.0, 0.0], "plus": [2**-0.5, 2**-0.5]}
    if basis not in vecs:
        raise ValueError(f"unknown basis {basis!r}; use 'zero' or 'plus'")
    v = np.array(vecs[basis], dtype=np.complex128).reshape(1, 2, 1)
    return MpsState([v.copy() for _ in range(m)], trunc_budget_per_gate=trunc_budget_per_gate, ortho_center=0)


def stats(state: MpsState) -> SimStats:
    """Resource counters (mps.py:281-291); memory is 16 bytes per entry."""
    n = state.entry_count()
    return SimStats(
        max(state.peak_chi, state.max_bond()), n, 16 * n, state.gate_count_1q, state.gate_count_2q,
        dict(state.timings),
    )


def to_statevector(state: MpsState) -> np.ndarray:
    """Dense amplitudes, qubit 0 most significant (host test aid, mps.py:271-278)."""
    if state.m > _MAX_DENSE_QUBITS:
        raise ValueError(f"refusing dense conversion beyond {_MAX_DENSE_QUBITS} qubits")
    psi = np.ones((1, 1), dtype=np.complex128)
    for t in state.sites:
        psi = np.einsum("xa,apb->xpb", psi, t).reshape(-1, t.shape[2])
    return psi.reshape(-1)


# ---------------------------------------------------------------- wire format
_MAGIC = b"MPS1"
_HEADER = struct.Struct("<IddiIQQ")  # m, budget, discard, center, peak_chi, g1, g2


def serialize_state(state: MpsState) -> bytes:
    """MPS1 bytes (mps.py:294-314): header, then per site (chi_l, chi_r) as
    <II and the little-endian complex128 entries."""
    center = -1 if state.ortho_center is None else state.ortho_center
    out = [_MAGIC, _HEADER.pack(state.m, state.trunc_budget_per_gate, state.accumulated_discard, center,
                                state.peak_chi, state.gate_count_1q, state.gate_count_2q)]
    for t in state.sites:
        out.append(struct.pack("<II", t.shape[0], t.shape[2]))
        out.append(np.ascontiguousarray(t, dtype="<c16").tobytes())
    return b"".join(out)


def deserialize_state(buf: bytes) -> MpsState:
    """Inverse of serialize_state (mps.py:317-340)."""
    if bytes(buf[:4]) != _MAGIC:
        raise ValueError("not a serialized MPS state")
    m, budget, disc, center, peak, g1, g2 = _HEADER.unpack_from(buf, 4)
    off = 4 + _HEADER.size
    sites = []
    for _ in range(m):
        cl, cr = struct.unpack_from("<II", buf, off)
        off += 8
        n = cl * 2 * cr
        sites.append(np.frombuffer(buf, dtype="<c16", count=n, offset=off).astype(np.complex128).reshape(cl, 2, cr))
        off += 16 * n
    return MpsState(sites, budget, disc, None if center < 0 else center, peak, g1, g2)


# ---------------------------------------------------------------- programs
@dataclass(frozen=True)
class Program:
    """A gate topology compiled into the op list replayed by the GPU."""

    m: int
    ops: np.ndarray  # (n_ops, 4) int32
    n_gates: int
    n_params: int
    n_qr_left: int
    n_qr_right: int
    final_center: int
    gate_count_1q: int
    gate_count_2q: int

    @functools.cached_property
    def device_ops(self) -> torch.Tensor:
        return torch.from_numpy(self.ops).to("cuda")


def _topology_key(topo: Topology):
    return (topo.m, topo.kinds.tobytes(), topo.q0.tobytes(), topo.q1.tobytes(), topo.param_slot.tobytes())


_PROGRAMS: dict = {}
_CAP_HINT: dict = {}


def compile_program(topo: Topology) -> Program:
    key = _topology_key(topo)
    prog = _PROGRAMS.get(key)
    if prog is not None:
        return prog
    lib = N.lib()
    kinds = np.ascontiguousarray(topo.kinds, dtype=np.int32)
    q0 = np.ascontiguousarray(topo.q0, dtype=np.int32)
    q1 = np.ascontiguousarray(topo.q1, dtype=np.int32)
    slot = np.ascontiguousarray(topo.param_slot, dtype=np.int32)
    args = [N.ptr(a, N.C.c_int32) for a in (kinds, q0, q1, slot)]
    n_ops, nl, nr = N.C.c_int64(0), N.C.c_int64(0), N.C.c_int64(0)
    N.check(lib.mpskq_program_compile(topo.m, kinds.size, *args, None, 0, N.C.byref(n_ops), None, None))
    ops = np.zeros((n_ops.value, 4), dtype=np.int32)
    N.check(
        lib.mpskq_program_compile(
            topo.m, kinds.size, *args, N.ptr(ops, N.C.c_int32), n_ops.value, N.C.byref(n_ops),
            N.C.byref(nl), N.C.byref(nr),
        )
    )
    center = 0
    for code, site, _, _ in ops:
        c = code & 0xFF
        if c in (3, 4):  # two-qubit ops: center ends on the absorbing side
            center = site if (code >> 8) & 1 else site + 1
    two = np.isin(kinds, (N.GATE_RXX, N.GATE_SWAP))
    prog = Program(topo.m, ops, int(kinds.size), int(topo.n_params), int(nl.value), int(nr.value), center,
                   int((~two).sum()), int(two.sum()))
    _PROGRAMS[key] = prog
    return prog


def batch_layout(m: int, chi_cap: int) -> tuple:
    off = np.zeros(m + 1, dtype=np.int64)
    stride = N.C.c_int64(0)
    N.check(N.lib().mpskq_batch_layout(m, chi_cap, N.ptr(off, N.C.c_int64), N.C.byref(stride)))
    return off, int(stride.value)


# ---------------------------------------------------------------- device batch
class MpsBatch(Sequence):
    """Device-resident batch of MPS produced by the GPU simulator.

    Storage (see include/mpskq.h): one complex128 slab with per-site slots,
    ``chi`` bond dims (n, m+1).  Indexing returns host ``MpsState`` copies in
    the reference layout.
    """

    def __init__(self, m, chi_cap, site_off, stride, sites, chi, discard, peak, budget,
                 gate_count_1q, gate_count_2q, ortho_center, entry_log=None, seconds=0.0):
        self.m = m
        self.chi_cap = chi_cap
        self.site_off = site_off
        self.site_off_dev = torch.from_numpy(site_off).to(sites.device)
        self.stride = stride
        self.sites = sites  # float64 (n, 2*stride)
        self.chi = chi  # int32 (n, m+1)
        self.discard = discard  # float64 (n,)
        self.peak = peak  # int32 (n,)
        self.budget = budget
        self.gate_count_1q = gate_count_1q
        self.gate_count_2q = gate_count_2q
        self.ortho_center = ortho_center
        self.entry_log = entry_log
        self.seconds = seconds
        self._root, self._base, self._items = self, 0, {}  # row views share the root's item cache
        self.phase_cycles = None  # int64 (n, 3) device clocks per phase (simulate_program)
        self.nominal_flops = None  # float64 (n,) nominal simulation flops
        self._phase_host = None
        self._host = None

    def __len__(self) -> int:
        return self.chi.shape[0]

    def _host_arrays(self):
        if self._host is None:
            self._host = (
                self.sites.cpu().numpy().view(np.complex128),
                self.chi.cpu().numpy(),
                self.discard.cpu().numpy(),
                self.peak.cpu().numpy(),
            )
        return self._host

    def bond_dims(self) -> np.ndarray:
        return self._host_arrays()[1]

    def __getitem__(self, i):
        if isinstance(i, slice):
            a, b, step = i.indices(len(self))
            if step == 1:  # a device view, like slicing the reference's list of states
                return self.rows(a, max(a, b))
            return [self[k] for k in range(a, b, step)]
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        # one host MpsState object per state (list semantics: batch[i] is batch[i],
        # which compute_gram's train check relies on, kernel.py:161-164).  The
        # object is a host copy: mutating it does not change the device batch.
        key = self._base + i
        hit = self._root._items.get(key)
        if hit is not None:
            return hit
        sites, chi, disc, peak = self._host_arrays()
        row, c = sites[i], chi[i]
        ts = [
            row[self.site_off[s] : self.site_off[s] + c[s] * 2 * c[s + 1]].reshape(c[s], 2, c[s + 1]).copy()
            for s in range(self.m)
        ]
        st = MpsState(ts, self.budget, float(disc[i]), self.ortho_center, int(peak[i]), self.gate_count_1q,
                      self.gate_count_2q, self.timings(i))
        self._root._items[key] = st
        return st

    def same_states(self, other) -> bool:
        """True when `other` views exactly the same states (the batch analogue
        of the reference's element-wise `is` check)."""
        return (isinstance(other, MpsBatch) and other._root is self._root and other._base == self._base
                and len(other) == len(self))

    def timings(self, i: int) -> dict:
        """Per-phase device seconds of state i (MpsState.timings keys,
        mps.py:137 / :159 / :204), from the simulator's per-state clocks."""
        if self.phase_cycles is None:
            return {}
        if self._phase_host is None:
            self._phase_host = self.phase_cycles.cpu().numpy() / _sm_hz()
        c, o, t = (float(x) for x in self._phase_host[i])
        return {k: v for k, v in (("canonicalize", c), ("one_qubit", o), ("two_qubit", t)) if v > 0.0}

    def rows(self, a: int, b: int) -> "MpsBatch":
        """Device view of states a..b-1 (no copy)."""
        log = None if self.entry_log is None else self.entry_log[a:b]
        out = MpsBatch(self.m, self.chi_cap, self.site_off, self.stride, self.sites[a:b], self.chi[a:b],
                       self.discard[a:b], self.peak[a:b], self.budget, self.gate_count_1q,
                       self.gate_count_2q, self.ortho_center, log, self.seconds * (b - a) / max(len(self), 1))
        out.phase_cycles = None if self.phase_cycles is None else self.phase_cycles[a:b]
        out.nominal_flops = None if self.nominal_flops is None else self.nominal_flops[a:b]
        out._root, out._base = self._root, self._base + a
        return out

    def to_states(self) -> list:
        return [self[i] for i in range(len(self))]

    def memory_log(self, i: int) -> list:
        if self.entry_log is None:
            raise ValueError("batch was simulated without a memory log")
        return [16 * int(x) for x in self.entry_log[i].cpu().numpy()]

    @classmethod
    def from_states(cls, states, chi_cap: int | None = None) -> "MpsBatch":
        """Upload host MpsState objects (e.g. produced by the reference) into a batch."""
        require_cuda()
        states = list(states)
        if not states:
            raise ValueError("no states")
        m = states[0].m
        if any(s.m != m for s in states):
            raise ValueError("qubit count mismatch between state lists")
        need = max(max(s.bond_dims()) for s in states)
        phys = np.minimum(np.arange(m + 1), m - np.arange(m + 1))
        for s in states:  # the layout's slot of bond b holds at most 2^min(b, m-b)
            if np.any(np.array(s.bond_dims(), dtype=np.float64) > np.exp2(phys)):
                raise ValueError("bond dimension exceeds the exact-state bound 2^min(b, m-b)")
        caps = N.supported_chi_caps()
        if chi_cap is None:
            chi_cap = next((c for c in caps if c >= need), None)
            if chi_cap is None:
                raise ValueError(f"bond dimension {need} exceeds the largest compiled capacity {caps[-1]}")
        elif chi_cap < need:
            raise ValueError(f"bond dimension {need} exceeds chi capacity {chi_cap}")
        off, stride = batch_layout(m, chi_cap)
        host = np.zeros((len(states), stride), dtype=np.complex128)
        chi = np.zeros((len(states), m + 1), dtype=np.int32)
        for n, s in enumerate(states):
            chi[n] = s.bond_dims()
            for k, t in enumerate(s.sites):
                host[n, off[k] : off[k] + t.size] = np.asarray(t, dtype=np.complex128).reshape(-1)
        dev = torch.device("cuda")
        return cls(
            m, chi_cap, off, stride, torch.from_numpy(host.view(np.float64)).to(dev), torch.from_numpy(chi).to(dev),
            torch.tensor([s.accumulated_discard for s in states], dtype=torch.float64, device=dev),
            torch.tensor([s.peak_chi for s in states], dtype=torch.int32, device=dev),
            states[0].trunc_budget_per_gate, states[0].gate_count_1q, states[0].gate_count_2q,
            states[0].ortho_center,
        )


def _sm_hz() -> float:
    khz = N.lib().mpskq_sm_clock_khz()
    return 1e3 * khz if khz > 0 else 1.9e9


def _check_states(status: np.ndarray) -> np.ndarray:
    """Raise like the reference for failed states; returns the overflow rows."""
    if np.any(status == N.STATE_NONFINITE):
        raise ValueError("tensor has non-finite entries")
    if np.any(status == N.STATE_NOCONV):
        raise np.linalg.LinAlgError("SVD did not converge")
    return np.nonzero(status == N.STATE_CAPACITY)[0]


def simulate_program(prog: Program, coef, budget: float, chi_max: int = 0,
                     chi_cap: int | None = None, memory_log: bool = False) -> MpsBatch:
    """Run the compiled program from |0..0> for every row of the coefficient
    table ``coef`` ((n, n_params, 2) half-angle cos/sin, numpy or a CUDA
    tensor).  Every state starts at the hinted chi capacity; only the states
    that outgrow it are re-simulated at the next capacity (per-state
    escalation), and the levels are gathered into the final capacity's
    layout (mpskq_relayout)."""
    require_cuda()
    if budget < 0:
        raise ValueError("budget must be non-negative")
    dev = torch.device("cuda")
    if not isinstance(coef, torch.Tensor):
        coef = torch.from_numpy(np.ascontiguousarray(coef, dtype=np.float64))
    coef = coef.to(dev, torch.float64).contiguous()
    if coef.ndim != 3 or tuple(coef.shape[1:]) != (prog.n_params, 2):
        raise ValueError(f"coefficient table must be (n, {prog.n_params}, 2), got {tuple(coef.shape)}")
    n = coef.shape[0]
    ops_d = prog.device_ops
    caps = N.supported_chi_caps()
    key = (id(prog), float(budget), int(chi_max))
    if chi_cap is not None:
        if chi_cap not in caps:
            raise ValueError(f"chi capacity {chi_cap} is not compiled in (have {caps})")
        order = [chi_cap]
    else:
        order = [c for c in caps if c >= _CAP_HINT.get(key, caps[0])]
        if chi_max > 0:  # the kept rank never exceeds chi_max
            order = [c for c in order if c < chi_max] + [c for c in order if c >= chi_max][:1]
    m = prog.m
    levels = []
    rows = None  # device int64 global row ids of this level (None: all rows)
    seconds = 0.0
    for cap in order:
        nl = n if rows is None else int(rows.numel())
        coef_l = coef if rows is None else coef.index_select(0, rows)
        if coef_l.numel() == 0:
            coef_l = torch.zeros((max(nl, 1), max(prog.n_params, 1), 2), dtype=torch.float64, device=dev)
        off, stride = batch_layout(m, cap)
        off_d = torch.from_numpy(off).to(dev)
        lv = dict(
            cap=cap, rows=rows, off=off, stride=stride, off_d=off_d,
            sites=torch.empty((nl, 2 * stride), dtype=torch.float64, device=dev),
            chi=torch.empty((nl, m + 1), dtype=torch.int32, device=dev),
            disc=torch.empty(nl, dtype=torch.float64, device=dev),
            peak=torch.empty(nl, dtype=torch.int32, device=dev),
            status=torch.zeros(nl, dtype=torch.int32, device=dev),
            elog=torch.zeros((nl, prog.n_gates), dtype=torch.int64, device=dev) if memory_log else None,
            phase=torch.zeros((nl, 3), dtype=torch.int64, device=dev),
            flops=torch.zeros(nl, dtype=torch.float64, device=dev),
        )
        def run():
            return N.lib().mpskq_run_program(
                m, cap, dptr(ops_d), prog.ops.shape[0], prog.n_gates, dptr(coef_l), prog.n_params, nl,
                float(budget), int(chi_max), dptr(off_d), stride, 0, dptr(lv["sites"]), dptr(lv["chi"]),
                dptr(lv["disc"]), dptr(lv["peak"]), dptr(lv["status"]), dptr(lv["elog"]),
                dptr(lv["phase"]), dptr(lv["flops"]), stream_ptr(),
            )

        with Timer() as tm:
            st_code = run()
            if st_code == N.ERR_CUDA and b"out of memory" in (N.lib().mpskq_last_error() or b""):
                # the simulator's per-CTA workspaces come from the stream-ordered
                # pool; blocks torch's caching allocator keeps for reuse are not
                # visible to it: hand them back and retry once
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
                st_code = run()
            N.check(st_code)
        seconds += tm.seconds()
        over = _check_states(lv["status"].cpu().numpy())
        levels.append(lv)
        if over.size == 0:
            break
        if chi_cap is not None:
            raise RuntimeError(f"bond dimension exceeds the largest usable chi capacity {order[-1]}")
        # keep this level's states exactly packed (their own bond dims, no
        # capacity padding) until the final layout is known: at large
        # capacities the padded levels would otherwise stack up in HBM
        ent = (2 * lv["chi"][:, :-1].long() * lv["chi"][:, 1:].long()).sum(1)
        lv["state_off"] = torch.cumsum(ent, 0) - ent
        lv["packed"] = torch.empty(max(2 * int(ent.sum().item()), 2), dtype=torch.float64, device=dev)
        N.check(N.lib().mpskq_pack_exact(m, nl, dptr(lv["sites"]), dptr(off_d), stride, dptr(lv["chi"]),
                                         dptr(lv["state_off"]), dptr(lv["packed"]), stream_ptr()))
        lv["sites"] = None
        ov = torch.from_numpy(over).to(dev)
        rows = ov if rows is None else rows.index_select(0, ov)
    else:
        raise RuntimeError(f"bond dimension exceeds the largest usable chi capacity {order[-1]}")
    if chi_cap is None:
        # the next call of this program starts at the capacity the whole batch
        # needed: a level below it costs a full replay of every state that
        # later overflows (measured at config 5 d=8: starting two levels lower
        # was 1.6x slower overall), so escalation only pays on the first call
        _CAP_HINT[key] = levels[-1]["cap"]
    fin = levels[-1]
    if len(levels) == 1:
        sites, chi, disc, peak, elog, phase = (fin[k] for k in ("sites", "chi", "disc", "peak", "elog", "phase"))
        flops = fin["flops"]
    else:
        sites = torch.empty((n, 2 * fin["stride"]), dtype=torch.float64, device=dev)
        chi = torch.empty((n, m + 1), dtype=torch.int32, device=dev)
        disc = torch.empty(n, dtype=torch.float64, device=dev)
        peak = torch.empty(n, dtype=torch.int32, device=dev)
        phase = torch.empty((n, 3), dtype=torch.int64, device=dev)
        flops = torch.zeros(n, dtype=torch.float64, device=dev)
        elog = torch.empty((n, prog.n_gates), dtype=torch.int64, device=dev) if memory_log else None
        for lv in levels:  # later levels overwrite the rows that overflowed earlier ones
            r32 = None if lv["rows"] is None else lv["rows"].to(torch.int32)
            nl = lv["chi"].shape[0]
            if lv.get("packed") is not None:
                N.check(N.lib().mpskq_unpack_exact(m, nl, dptr(lv["packed"]), dptr(lv["state_off"]), dptr(lv["chi"]),
                                                   dptr(sites), dptr(fin["off_d"]), fin["stride"], dptr(r32),
                                                   stream_ptr()))
            else:
                N.check(N.lib().mpskq_relayout(m, nl, dptr(lv["sites"]), dptr(lv["off_d"]), lv["stride"],
                                               dptr(lv["chi"]), dptr(sites), dptr(fin["off_d"]), fin["stride"],
                                               dptr(r32), stream_ptr()))
            idx = lv["rows"] if lv["rows"] is not None else torch.arange(n, device=dev)
            chi.index_copy_(0, idx, lv["chi"])
            disc.index_copy_(0, idx, lv["disc"])
            peak.index_copy_(0, idx, lv["peak"])
            phase.index_copy_(0, idx, lv["phase"])
            flops.index_add_(0, idx, lv["flops"])  # nominal work of every level a state ran at
            if elog is not None:
                elog.index_copy_(0, idx, lv["elog"])
    batch = MpsBatch(m, fin["cap"], fin["off"], fin["stride"], sites, chi, disc, peak, budget, prog.gate_count_1q,
                     prog.gate_count_2q, prog.final_center, elog, seconds)
    batch.phase_cycles = phase
    batch.nominal_flops = flops
    return batch


def simulate_circuit(circuit: Circuit, budget: float = DEFAULT_TRUNC_BUDGET, memory_log: list | None = None) -> MpsState:
    """Simulate ``circuit`` from |0...0> on the GPU (mps.py:250-257)."""
    topo, angles = circuit_topology(circuit)
    prog = compile_program(topo)
    coef = half_angle_coefficients(angles).reshape(1, -1, 2)
    batch = simulate_program(prog, coef, budget, memory_log=memory_log is not None)
    if memory_log is not None:
        memory_log.extend(batch.memory_log(0))
    return batch[0]


# ---------------------------------------------------------------- gates on given states
_UNITARY_ATOL = 1e-10  # mps.py:26


def _check_unitary(u: np.ndarray) -> None:
    """mps.py:141-144 (input validation of a 2x2 / 4x4 host matrix)."""
    if not np.allclose(u.conj().T @ u, np.eye(u.shape[0]), atol=_UNITARY_ATOL):
        raise ValueError("gate matrix is not unitary")


def _moves(m: int, center, target: int) -> list:
    """canonicalize(state, target) as QR-move ops (mps.py:123-138): left
    steps (_left_isometrize, :105-111) below the target, right steps
    (_right_isometrize, :114-120) above it."""
    if center is None:
        return [(N.OP_QRL, s) for s in range(0, target)] + [(N.OP_QRR, s) for s in range(m - 1, target, -1)]
    if center < target:
        return [(N.OP_QRL, s) for s in range(center, target)]
    return [(N.OP_QRR, s) for s in range(center, target, -1)]


def _evolve(state: MpsState, ops: list, coef: np.ndarray, n_gates: int = 0, memory_log: bool = False):
    """Replay `ops` ((code, site[, slot, gate index, left])) on `state` on the
    GPU (mpskq_run_program with from_input=1) and write the result back into
    `state` (the reference mutates the state in place).  Escalates the chi
    capacity when a bond outgrows it.  Returns the per-gate entry counts."""
    require_cuda()
    if not ops:
        return []
    dev = torch.device("cuda")
    arr = np.zeros((len(ops), 4), dtype=np.int32)
    for k, op in enumerate(ops):
        code, site = op[0], op[1]
        slot = op[2] if len(op) > 2 else -1
        gidx = op[3] if len(op) > 3 else -1
        left = op[4] if len(op) > 4 else False
        arr[k] = (code | ((N.ABSORB_LEFT if left else 0) << 8), site, slot, gidx)
    ops_d = torch.from_numpy(arr).to(dev)
    cf = np.ascontiguousarray(coef, dtype=np.complex128).reshape(-1)
    n_params = max(cf.size, 1)
    coef_d = torch.from_numpy(np.concatenate([cf, np.zeros(1, np.complex128)])[:n_params].view(np.float64)).to(dev)
    caps = N.supported_chi_caps()
    start = next((c for c in caps if c >= state.max_bond()), None)
    if start is None:
        raise ValueError(f"bond dimension {state.max_bond()} exceeds the largest compiled capacity {caps[-1]}")
    for cap in [c for c in caps if c >= start]:
        b = MpsBatch.from_states([state], cap)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        elog = torch.zeros((1, max(n_gates, 1)), dtype=torch.int64, device=dev) if memory_log else None
        phase = torch.zeros((1, 3), dtype=torch.int64, device=dev)
        N.check(N.lib().mpskq_run_program(
            state.m, cap, dptr(ops_d), len(ops), max(n_gates, 1), dptr(coef_d), n_params, 1,
            float(state.trunc_budget_per_gate), 0, dptr(b.site_off_dev), b.stride, 1, dptr(b.sites), dptr(b.chi),
            dptr(b.discard), dptr(b.peak), dptr(status), dptr(elog), dptr(phase), None, stream_ptr()))
        if _check_states(status.cpu().numpy()).size:
            continue
        b.phase_cycles = phase
        out = b[0]
        state.sites[:] = out.sites
        state.accumulated_discard = out.accumulated_discard
        state.peak_chi = out.peak_chi
        for k, v in b.timings(0).items():
            state.timings[k] = state.timings.get(k, 0.0) + v
        return [16 * int(x) for x in elog[0, :n_gates].cpu().numpy()] if memory_log else []
    raise RuntimeError(f"bond dimension exceeds the largest usable chi capacity {caps[-1]}")


def canonicalize(state: MpsState, center: int) -> MpsState:
    """Move the orthogonality center to ``center`` (mps.py:123-138) with QR
    moves on the GPU."""
    if not 0 <= center < state.m:
        raise ValueError(f"center {center} out of range for {state.m} sites")
    _evolve(state, _moves(state.m, state.ortho_center, center), np.zeros(0))
    state.ortho_center = center
    return state


def apply_one_qubit(state: MpsState, q: int, matrix) -> MpsState:
    """Contract a 2x2 unitary with site q on the GPU (mps.py:147-160)."""
    if not 0 <= q < state.m:
        raise ValueError(f"qubit {q} out of range")
    matrix = np.asarray(matrix, dtype=np.complex128)
    if matrix.shape != (2, 2):
        raise ValueError("single-qubit gate must be a 2x2 matrix")
    _check_unitary(matrix)
    _evolve(state, [(N.OP_U1, q, 0)], matrix)
    state.gate_count_1q += 1
    return state


def apply_two_qubit(state: MpsState, q: int, matrix, absorb: str = "right") -> MpsState:
    """4x4 unitary on (q, q+1): canonicalize, theta, truncated SVD, renorm,
    absorb (mps.py:163-205), all on the GPU."""
    if not 0 <= q < state.m - 1:
        raise ValueError(f"site pair ({q}, {q + 1}) out of range")
    if absorb not in ("left", "right"):
        raise ValueError("absorb must be 'left' or 'right'")
    matrix = np.asarray(matrix, dtype=np.complex128)
    if matrix.shape != (4, 4):
        raise ValueError("two-qubit gate must be a 4x4 matrix")
    _check_unitary(matrix)
    left = absorb == "left"
    _evolve(state, _moves(state.m, state.ortho_center, q) + [(N.OP_U2, q, 0, -1, left)], matrix)
    state.ortho_center = q if left else q + 1
    state.gate_count_2q += 1
    return state


def apply_gate(state: MpsState, gate, absorb: str = "right") -> MpsState:
    """Apply one circuit gate (mps.py:208-221); two-qubit gates must act on
    adjacent qubits."""
    from .ansatz import gate_matrix

    for q in gate.qubits:
        if not 0 <= q < state.m:
            raise ValueError(f"qubit {q} out of range for {state.m} sites")
    u = gate_matrix(gate)
    if len(gate.qubits) == 1:
        return apply_one_qubit(state, gate.qubits[0], u)
    a, b = gate.qubits
    if abs(a - b) != 1:
        raise ValueError(f"two-qubit gate on ({a}, {b}) is not adjacent; route the circuit first")
    if a > b:
        u = u.reshape(2, 2, 2, 2).transpose(1, 0, 3, 2).reshape(4, 4)
    return apply_two_qubit(state, min(a, b), u, absorb=absorb)


def run_circuit(state: MpsState, circuit: Circuit, memory_log: list | None = None) -> MpsState:
    """Apply every gate of ``circuit`` in order with run_circuit's absorb rule
    (mps.py:224-247) as ONE GPU program: the canonicalize moves start from the
    state's own orthogonality center; H/RZ/RXX/SWAP use the simulator's gate
    ops (the ones simulate_circuit replays)."""
    if circuit.m != state.m:
        raise ValueError(f"circuit has {circuit.m} qubits, state has {state.m}")
    gates = circuit.gates
    next_2q = [None] * (len(gates) + 1)
    for i in range(len(gates) - 1, -1, -1):
        next_2q[i] = min(gates[i].qubits) if len(gates[i].qubits) == 2 else next_2q[i + 1]
    codes = {"H": N.OP_H, "RZ": N.OP_RZ, "RXX": N.OP_RXX, "SWAP": N.OP_SWAP}
    ops, angles = [], []
    center = state.ortho_center
    g1 = g2 = 0
    for i, g in enumerate(gates):
        for q in g.qubits:
            if not 0 <= q < state.m:
                raise ValueError(f"qubit {q} out of range for {state.m} sites")
        slot = -1
        if g.angle is not None:
            slot = len(angles)
            angles.append(g.angle)
        if len(g.qubits) == 1:
            ops.append((codes[g.kind], g.qubits[0], slot, i))
            g1 += 1
            continue
        a, b = g.qubits
        if abs(a - b) != 1:
            raise ValueError(f"two-qubit gate on ({a}, {b}) is not adjacent; route the circuit first")
        q = min(a, b)  # H/RZ/RXX/SWAP are symmetric under exchanging the qubits
        nxt = next_2q[i + 1]
        left = nxt is not None and nxt <= q
        ops += _moves(state.m, center, q)
        ops.append((codes[g.kind], q, slot, i, left))
        center = q if left else q + 1
        g2 += 1
    from .ansatz import half_angle_coefficients

    hc = half_angle_coefficients(np.array(angles, dtype=np.float64)) if angles else np.zeros((0, 2))
    coef = hc[:, 0] + 1j * hc[:, 1]
    log = _evolve(state, ops, coef, n_gates=len(gates), memory_log=memory_log is not None)
    if memory_log is not None:
        memory_log.extend(log)
    state.ortho_center = center
    state.gate_count_1q += g1
    state.gate_count_2q += g2
    return state


def _as_batch(x) -> tuple:
    if isinstance(x, MpsBatch):
        return x, None
    if isinstance(x, MpsState):
        return MpsBatch.from_states([x]), None
    raise TypeError(f"expected MpsState or MpsBatch, got {type(x).__name__}")


def _common_cap(bras: MpsBatch, kets: MpsBatch) -> tuple:
    if bras.m != kets.m:
        raise ValueError("qubit count mismatch between state lists")
    if bras.chi_cap != kets.chi_cap:
        cap = max(bras.chi_cap, kets.chi_cap)
        bras = bras if bras.chi_cap == cap else MpsBatch.from_states(bras.to_states(), cap)
        kets = kets if kets.chi_cap == cap else MpsBatch.from_states(kets.to_states(), cap)
    return bras, kets


def pinned_matrix(rows: int, cols: int) -> torch.Tensor:
    """Page-locked host float64 matrix (torch's caching host allocator: the
    block returns to the cache when the numpy view handed out is dropped)."""
    return torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)


def overlap_matrix_host(bras: MpsBatch, kets: MpsBatch, kind: str) -> np.ndarray:
    """Host matrix of |<bra_i|ket_j>|^2 in page-locked memory: at chi <= 4 the
    overlap streams finished row bands into it under the computation
    (mpskq_overlap_host), otherwise one device-to-host copy."""
    require_cuda()
    bras, kets = _common_cap(bras, kets)
    nb, nk = len(bras), len(kets)
    K = pinned_matrix(nb, nk)
    kind_id = N.KIND_TRAIN if kind == "train" else N.KIND_TEST
    N.check(N.lib().mpskq_overlap_host(
        kind_id, bras.m, bras.chi_cap, dptr(bras.site_off_dev), bras.stride, dptr(bras.sites), dptr(bras.chi), nb,
        dptr(kets.sites), dptr(kets.chi), nk, K.data_ptr(), stream_ptr()))
    return K.numpy()


def overlap_matrix(bras: MpsBatch, kets: MpsBatch, kind: str, amplitude: bool = False,
                   rank: int = 0, world: int = 1, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device matrix of |<bra_i|ket_j>|^2 (or the complex amplitudes)."""
    require_cuda()
    bras, kets = _common_cap(bras, kets)
    kind_id = N.KIND_TRAIN if kind == "train" else N.KIND_TEST
    nb, nk = len(bras), len(kets)
    if out is None:
        shape = (nb, nk, 2) if amplitude else (nb, nk)
        out = torch.zeros(shape, dtype=torch.float64, device=bras.sites.device)
    N.check(
        N.lib().mpskq_overlap(
            kind_id, N.OUT_AMPLITUDE if amplitude else N.OUT_KERNEL, bras.m, bras.chi_cap,
            dptr(bras.site_off_dev), bras.stride, dptr(bras.sites), dptr(bras.chi), nb,
            dptr(kets.sites), dptr(kets.chi), nk, rank, world, dptr(out), nk, stream_ptr(),
        )
    )
    return out


def inner_product(bra, ket) -> complex:
    """<bra|ket> with the bra conjugated, contracted site by site (mps.py:260-268)."""
    if bra.m != ket.m:
        raise ValueError(f"qubit count mismatch: {bra.m} vs {ket.m}")
    b, _ = _as_batch(bra)
    k, _ = _as_batch(ket)
    if len(b) != 1 or len(k) != 1:
        raise ValueError("inner_product takes single states")
    amp = overlap_matrix(b, k, "test", amplitude=True).cpu().numpy()
    return complex(amp[0, 0, 0], amp[0, 0, 1])
