"""Host-side logic of the drop-in (no GPU needed): the C ABI loads and exports
every symbol include/mpskq.h declares; topology / angles / coefficients /
program compiler / layout / tiles / schedules agree with the reference."""

import math
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import mps_oracle as O


def test_library_exports_every_header_symbol(native):
    header = (ROOT / "include" / "mpskq.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(mpskq_\w+)\s*\(", header, re.M))
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(native, name), name
    from paper_2411_09336_b200 import _native

    assert declared == set(_native.exported_symbols())


def test_abi_version_and_caps(native):
    from paper_2411_09336_b200 import _native

    assert native.mpskq_abi_version() == 1
    assert _native.supported_chi_caps() == [4, 8, 12, 16, 24, 32, 48, 64, 80, 96, 128]
    assert native.mpskq_device_count() >= 0


@pytest.mark.parametrize("name", ["config1_m8_d1.npz", "headline_m165_d1.npz", "config2_m50_d2.npz", "config3_m100_d4.npz"])
def test_native_topology_and_angles_match_reference(name):
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.ansatz import feature_map_topology

    g = golden(name)
    m, r, d, gamma = int(g["m"]), int(g["r"]), int(g["d"]), float(g["gamma"])
    t = feature_map_topology(m, r, d)
    assert np.array_equal(t.kinds, g["kinds"]) and np.array_equal(t.q0, g["q0"]) and np.array_equal(t.q1, g["q1"])
    c = P.encode_circuit(g["X"][0], P.FeatureMapConfig(m, r, d, gamma))
    ang = np.array([np.nan if x.angle is None else x.angle for x in c.gates])
    assert np.array_equal(ang, g["angles0"], equal_nan=True)  # bitwise


def test_half_angle_coefficients_reproduce_gate_matrix_bitwise():
    from paper_2411_09336_b200.ansatz import half_angle_coefficients

    ang = np.concatenate([np.random.default_rng(0).uniform(-4, 4, 500), [0.0, -math.pi, 1e-300]])
    cs = half_angle_coefficients(ang)
    for a, (c, s) in zip(ang, cs):
        rz = O.gate_unitary("RZ", a)
        assert rz[0, 0] == complex(c, -s) and rz[1, 1] == complex(c, s)
        rxx = O.gate_unitary("RXX", a)
        assert rxx[0, 0].real == c and rxx[0, 3].imag == -s


def test_program_counts_match_survey():
    from paper_2411_09336_b200.ansatz import feature_map_topology
    from paper_2411_09336_b200.mps import compile_program

    # QR step counts per state
    for (m, r, d), (gates, nl, nr) in {
        (165, 2, 1): (823, 324, 485),
        (50, 2, 2): (536, 182, 416),
        (100, 2, 4): (3400, 744, 2570),
    }.items():
        p = compile_program(feature_map_topology(m, r, d))
        assert (p.n_gates, p.n_qr_left, p.n_qr_right) == (gates, nl, nr)


def test_program_matches_oracle_center_moves():
    """Replaying the ops' QR moves and absorb sides reproduces the reference's
    canonical-center trajectory (mps.py:181, :193-200, :235-241)."""
    from paper_2411_09336_b200.ansatz import feature_map_topology
    from paper_2411_09336_b200.mps import compile_program

    p = compile_program(feature_map_topology(12, 2, 3))
    center = 0
    for code, site, _, _ in p.ops:
        c = code & 0xFF
        if c == 5:
            assert site == center
            center += 1
        elif c == 6:
            assert site == center
            center -= 1
        elif c in (3, 4):
            assert center == site
            center = site if (code >> 8) & 1 else site + 1
    assert center == p.final_center


def test_program_rejects_non_adjacent_and_bad_qubits():
    from paper_2411_09336_b200.ansatz import Circuit, Gate, circuit_topology
    from paper_2411_09336_b200.mps import compile_program

    topo, _ = circuit_topology(Circuit(4, [Gate("RXX", (0, 2), 0.3)]))
    with pytest.raises(ValueError, match="adjacent"):
        compile_program(topo)


def test_feature_rows_validated():
    import paper_2411_09336_b200 as P

    cfg = P.FeatureMapConfig(4, 1, 1, 0.5)
    with pytest.raises(ValueError, match="range|\\[0, 2\\]"):
        P.encode_circuit(np.array([0.0, 2.5, 1.0, 1.0]), cfg)
    with pytest.raises(ValueError, match="finite"):
        P.encode_circuit(np.array([0.0, np.nan, 1.0, 1.0]), cfg)
    with pytest.raises(ValueError, match="features"):
        P.encode_circuit(np.zeros(3), cfg)
    with pytest.raises(ValueError):
        P.FeatureMapConfig(4, 1, 4, 0.5)


def test_generic_circuit_helpers_match_oracle_routing():
    import paper_2411_09336_b200 as P

    rng = np.random.default_rng(3)
    for m in range(2, 9):
        for d in range(1, m):
            cfg = P.FeatureMapConfig(m, 2, d, 0.7)
            x = rng.uniform(0, 2, m)
            routed = P.route_linear(P.schedule_circuit(P.build_circuit(x, cfg), d))
            ref = O.feature_map_gates(x, m, 2, d, 0.7)
            got = [(g.kind, g.qubits[0], g.qubits[1] if len(g.qubits) > 1 else -1, g.angle) for g in routed.gates]
            assert got == ref
            assert routed.gates == P.encode_circuit(x, cfg).gates
            swaps = sum(g.kind == "SWAP" for g in routed.gates)
            assert swaps == 2 * 2 * sum((k - 1) * (m - k) for k in range(2, d + 1))


def test_gate_matrix_matches_reference_definition():
    import paper_2411_09336_b200 as P

    for kind, ang in [("H", None), ("SWAP", None), ("RZ", 0.37), ("RXX", -1.3)]:
        g = P.Gate(kind, (0,) if kind in ("H", "RZ") else (0, 1), ang)
        assert np.array_equal(P.gate_matrix(g), O.gate_unitary(kind, ang))


def test_batch_layout():
    from paper_2411_09336_b200.mps import batch_layout

    off, stride = batch_layout(6, 4)
    caps = [min(4, 2 ** min(b, 6 - b)) for b in range(7)]
    sizes = [2 * caps[s] * caps[s + 1] for s in range(6)]
    assert list(off[:6]) == list(np.cumsum([0] + sizes[:-1]))
    assert stride >= sum(sizes) and stride % 2 == 0


@pytest.mark.parametrize("kind,nb,nk", [("train", 70, 70), ("train", 33, 33), ("test", 17, 70), ("test", 5, 3)])
@pytest.mark.parametrize("cap", [4, 8, 32])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_overlap_tiles_cover_exactly_once(kind, nb, nk, cap, world):
    from paper_2411_09336_b200.distributed import tiles_of

    cover = np.zeros((nb, nk), dtype=int)
    for rank in range(world):
        tiles, rb, cb = tiles_of(kind, cap, nb, nk, rank, world)
        for I, J in tiles:
            for i in range(I * rb, min(nb, (I + 1) * rb)):
                for j in range(J * cb, min(nk, (J + 1) * cb)):
                    if kind == "test" or i < j:
                        cover[i, j] += 1
    need = np.triu(np.ones((nb, nk), dtype=int), 1) if kind == "train" else np.ones((nb, nk), dtype=int)
    assert np.array_equal(cover, need)


def test_schedules_match_reference():
    import paper_2411_09336_b200 as P

    for row in golden("schedules.json"):
        s = P.make_schedule(row["nb"], row["nk"], row["k"], row["strategy"], row["kind"])
        assert s.k == row["kk"]
        tiles = [[si, t.worker, t.row_start, t.row_stop, t.col_start, t.col_stop] for si, st in enumerate(s.steps) for t in st.tiles]
        transfers = [[si, t.src, t.dst, t.which, t.start, t.stop] for si, st in enumerate(s.steps) for t in st.transfers]
        assert tiles == row["tiles"]
        assert transfers == row["transfers"]
        assert {str(w): [list(x) for x in v] for w, v in s.initial_states.items()} == row["initial"]
        P.validate_schedule(s)


def test_schedule_errors():
    import paper_2411_09336_b200 as P

    with pytest.raises(ValueError):
        P.make_schedule(4, 5, 2, "round_robin", "train")
    with pytest.raises(ValueError):
        P.make_schedule(4, 4, 0, "round_robin", "train")
    with pytest.raises(ValueError):
        P.make_schedule(4, 4, 2, "broadcast", "train")
    with pytest.raises(ValueError):
        P.make_schedule(4, 4, 2, "round_robin", "validation")
    assert P.make_schedule(3, 3, 10, "round_robin", "train").k == 3


def test_gram_persistence_round_trip(tmp_path):
    import json

    import paper_2411_09336_b200 as P

    K = golden("config1_m8_d1.npz")["K_train"]
    g = P.GramMatrix(K, "train")
    P.save_gram(g, tmp_path / "g.csv", sidecar={"k": 1})
    assert np.array_equal(P.load_gram(tmp_path / "g.csv", "train").entries, K)
    meta = json.loads((tmp_path / "g.csv.json").read_text())
    assert meta["rows"] == 64 and meta["kind"] == "train" and meta["k"] == 1


def test_gpu_entry_points_fail_loudly_without_cuda():
    import torch

    import paper_2411_09336_b200 as P

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        P.simulate_dataset(np.ones((2, 4)), P.FeatureMapConfig(4, 1, 1, 0.5))


def test_mps1_wire_format_round_trip_is_byte_exact():
    """serialize/deserialize (mps.py:294-340) on the reference's own bytes."""
    import paper_2411_09336_b200 as P

    g = golden("wire_mps1.npz")
    for key in ("blob0", "blob1"):
        blob = g[key].tobytes()
        st = P.deserialize_state(blob)
        assert P.serialize_state(st) == blob
        assert st.m == 6 and st.ortho_center is not None
    with pytest.raises(ValueError, match="serialized"):
        P.deserialize_state(b"XXXX" + bytes(40))
