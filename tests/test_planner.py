"""CPU tests of the host planner + device-op encoding (no GPU).

The detailed plan (qt_plan_probe_ex) is replayed by tests/emulator.py, an
independent numpy interpretation of every encoded op, and compared with the
dense oracle (oracle/, the restatement of oracle.cpp:15-50)."""
import json
import math

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import plan_probe, workloads as W
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array, lower_to_reference
from tests.emulator import apply_plan, logical_view

ALL = list(K)


def random_circuit(rng, n, count, kinds=ALL):
    rows = []
    for _ in range(count):
        kind = kinds[int(rng.integers(len(kinds)))]
        if n < 2 and kind in (K.Cnot, K.Swap, K.Cz):
            kind = K.H
        t = int(rng.integers(n))
        c = -1
        if kind in (K.Cnot, K.Swap, K.Cz):
            c = t
            while c == t:
                c = int(rng.integers(n))
        th, ph, la = (float(x) for x in rng.uniform(-7, 7, 3))
        rows.append(gate(kind, t, c, th, ph, la))
    return gate_array(rows)


def random_state(rng, n):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


@pytest.mark.parametrize("seed", range(12))
def test_plan_replay_matches_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 11))
    g = random_circuit(rng, n, int(rng.integers(1, 120)))
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, g, state=psi0.copy(), threads=1)
    for tile in (0, 3, 5):
        plan = json.loads(plan_probe(n, g, tile_qubits=tile, detail=True))
        got = apply_plan(psi0, plan)
        assert np.abs(got - want).max() < 1e-12, (tile, n)


@pytest.mark.parametrize("seed", range(8))
def test_plan_with_global_qubits_inserts_exchanges(seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(6, 11))
    ng = int(rng.integers(1, 4))
    g = random_circuit(rng, n, 80)
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, g, state=psi0.copy(), threads=1)
    plan = json.loads(plan_probe(n, g, global_qubits=ng, tile_qubits=4, detail=True))
    # tiles never contain global physical bits
    for ps in plan["passes"]:
        if ps["kind"] == "tile":
            assert max(ps["tile"]) < n - ng
    got = logical_view(apply_plan(psi0, plan), plan["perm_after"])
    assert np.abs(got - want).max() < 1e-12


def test_every_op_scheduled_once_and_tiles_bounded():
    w = W.config3(n=20, layers=6)
    plan = json.loads(plan_probe(20, w.gates, tile_qubits=10, detail=True))
    seen = []
    for ps in plan["passes"]:
        assert ps["kind"] == "tile"
        assert len(ps["tile"]) == 10 and ps["tile"][:4] == [0, 1, 2, 3]
        for rd in ps["round_detail"]:
            assert len(rd["reg"]) == 3  # kDefaultRegBits
        seen.extend(ps["gates"])
    # every op lands in exactly one pass (an op is listed under the first
    # gate of its fused run: odd layers leave q0 / q19 without a CZ, so their
    # consecutive U3s fuse); the output phases carried forward by phase
    # pushing are flushed once per qubit at the end as diagonal ops listed
    # under the last gate
    fused = len(w.gates) - 2 * 2
    assert len(set(seen)) == fused
    assert sum(ps["ops"] for ps in plan["passes"]) == plan["ops"]
    assert fused < plan["ops"] <= fused + 20


def test_fusion_merges_single_qubit_runs():
    g = gate_array([gate(K.Rz, 0, theta=0.3), gate(K.Ry, 0, theta=0.2),
                    gate(K.Rz, 0, theta=0.1), gate(K.H, 1)])
    plan = json.loads(plan_probe(4, g))
    # the three rotations on q0 are one 2x2, whose output phase is carried
    # forward (phase pushing) and flushed as one diagonal at the end; H's
    # factorisation has no output phase
    assert plan["ops"] == 3


def test_deep_fusion_of_layered_circuit():
    """C3 at full size: far fewer passes than gates (each pass streams the
    state once)."""
    w = W.config3()
    plan = json.loads(plan_probe(30, w.gates))
    tiles = [p for p in plan["passes"] if p["kind"] == "tile"]
    assert len(tiles) < len(w.gates) / 20
    assert sum(p["ops"] for p in tiles) == plan["ops"]


@pytest.mark.parametrize("eps", [1e-3, 1e-7, 1e-12])
def test_near_diagonal_and_antidiagonal_factorisation(eps):
    """U3s within eps of diagonal / anti-diagonal (|u10| or |u00| ~ eps) go
    through the diag . rotation . diag split and phase pushing; the split
    takes q1 from the larger column entry, so the replay stays at rounding
    level for any eps (qt_plan.cpp zyz_split)."""
    rng = np.random.default_rng(7)
    n = 6
    rows = []
    for layer in range(8):
        for q in range(n):
            th = eps if (q + layer) % 2 else math.pi - eps
            rows.append(gate(K.U3, q, -1, th, *rng.uniform(0, 2 * math.pi, 2)))
        for a in range(layer % 2, n - 1, 2):
            rows.append(gate(K.Cz, a + 1, a))
    g = gate_array(rows)
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, lower_to_reference(g), state=psi0.copy())
    for tq in (0, 4):
        plan = json.loads(plan_probe(n, g, tile_qubits=tq, detail=True))
        got = apply_plan(psi0, plan)
        assert np.abs(got - want).max() < 1e-13
