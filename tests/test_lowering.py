"""Host-only parity of the lowered layer words (csrc/qt_micro.cpp) -- the
instruction stream both device kernels execute: shear-form diagonal tables
centred by a common phase (the removed scalars carried through the plan and
folded into its last table), tile-uniform sign terms as slot flips, sign-only
tables as integer flips, rotations as shears, X / CX permutations. The words
of every pass are replayed by tests/emulator_lowered.py (an independent
decoder of the documented layout) and compared with the dense oracle
(oracle/, pinned to the reference oracle.cpp:15-50)."""
import json

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import jit_probe, workloads as W
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array, lower_to_reference
from tests.emulator_lowered import apply_lowered
from tests.test_planner import random_circuit, random_state

# kinds whose passes lower completely (SWAP and off-register diagonal
# variants keep generic passes)
LEAN = [K.H, K.X, K.Y, K.Z, K.S, K.Sdg, K.T, K.Tdg, K.Rx, K.Ry, K.Rz, K.Cnot, K.Cz, K.U3]
GEOMETRIES = [dict(), dict(tile_qubits=6, reg_bits=3, low_bits=2),
              dict(tile_qubits=7, reg_bits=4, low_bits=3), dict(tile_qubits=5, reg_bits=2, low_bits=1)]


def replay(n, gates, psi0=None, **geom):
    plan = json.loads(jit_probe(n, gates, source_pass=-2, **geom))
    if any(p["kind"] != "lowered" for p in plan["passes"]):
        pytest.skip("plan has generic passes")
    if psi0 is None:
        psi0 = np.zeros(1 << n, dtype=np.complex128)
        psi0[0] = 1.0
    return apply_lowered(psi0, plan)


@pytest.mark.parametrize("geom", range(len(GEOMETRIES)))
def test_layered_u3_cz(geom):
    w = W.config3(n=11, layers=6)
    got = replay(w.n, w.gates, **GEOMETRIES[geom])
    want = oracle.simulate(w.n, lower_to_reference(w.gates))
    assert np.abs(got - want).max() <= 1e-12


@pytest.mark.parametrize("geom", range(len(GEOMETRIES)))
def test_config5_family(geom):
    w = W.config5(n=11, ngates=250, nmods=0)
    got = replay(w.n, w.gates, **GEOMETRIES[geom])
    want = oracle.simulate(w.n, lower_to_reference(w.gates))
    assert np.abs(got - want).max() <= 1e-12


@pytest.mark.parametrize("seed", range(10))
def test_random_lean_circuits(seed):
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.integers(3, 11))
    g = random_circuit(rng, n, int(rng.integers(20, 200)), kinds=LEAN)
    psi0 = random_state(rng, n)
    geom = GEOMETRIES[seed % len(GEOMETRIES)]
    if geom and geom["tile_qubits"] > n:
        geom = dict(geom, tile_qubits=n)
    plan = json.loads(jit_probe(n, g, source_pass=-2, **geom))
    if any(p["kind"] != "lowered" for p in plan["passes"]):
        pytest.skip("plan has generic passes")
    got = apply_lowered(psi0, plan)
    want = oracle.simulate(n, g, state=psi0.copy())
    assert np.abs(got - want).max() <= 1e-12


def test_sign_only_tables_are_flips_and_scalars_fold():
    """RY with cos(theta/2) < 0 makes -1 factors (sign terms / tables of
    +-1): they lower to integer flips, and a plan whose only table factors
    are scalars still leaves the exact global phase (the carried scalar)."""
    n = 6
    rows = [gate(K.Ry, q, -1, 4.0 + q) for q in range(n)]
    rows += [gate(K.Rz, q, -1, 0.7 * q) for q in range(n)]
    g = gate_array(rows)
    got = replay(n, g)
    want = oracle.simulate(n, lower_to_reference(g))
    assert np.abs(got - want).max() <= 1e-12
    plan = json.loads(jit_probe(n, g, source_pass=-2))
    assert all(p["kind"] == "lowered" for p in plan["passes"])


def test_scaled_rotations_renormalise_long_plans():
    """Rotations lower to two-FMA scaled forms (c[[1,-t],[t,1]] or
    s[[u,-1],[1,u]]) whose scales the plan carries; H / RY(pi/2) grow the
    stored state by sqrt(2) each, so a 2400-rotation plan would overflow FP64
    without the power-of-two renormalising words (qt_micro.cpp
    kRescaleBelow). The replay must still match the oracle exactly."""
    n = 6
    rows = []
    for layer in range(400):
        for q in range(n):
            rows.append(gate(K.H, q, -1) if (layer + q) % 2 else gate(K.Ry, q, -1, 1.5707963267948966))
        for q in range(layer % 2, n - 1, 2):      # brick-wall CZ: no fusion
            rows.append(gate(K.Cz, q, q + 1))
    g = gate_array(rows)
    plan = json.loads(jit_probe(n, g, source_pass=-2))
    assert all(p["kind"] == "lowered" for p in plan["passes"])
    from tests.emulator_lowered import _f
    tiny = [v for ps in plan["passes"] for v in map(_f, ps["pool"]) if 0.0 < abs(v) < 2.0 ** -200]
    assert tiny, "no renormalising scale word was emitted"

    got = replay(n, g)
    want = oracle.simulate(n, lower_to_reference(g))
    assert np.isfinite(got).all()
    assert np.abs(got - want).max() <= 1e-10
    assert abs(float(np.vdot(got, got).real) - 1.0) <= 1e-12


PLANNER_ENVS = [
    {"QTB_WINDOW_SEARCH": "1"},
    {"QTB_WINDOW_SEARCH": "1", "QTB_WINDOW_BEAM": "8"},
    {"QTB_WINDOW_SEARCH": "1", "QTB_WINDOW_BEAM": "8", "QTB_PASS_FP64": "40"},
    {"QTB_SHRINK_MIN": "5", "QTB_SHRINK_RUN": "1"},
    {"QTB_WINDOW_SEARCH": "1", "QTB_SHRINK_MIN": "5"},
]


@pytest.mark.parametrize("env", range(len(PLANNER_ENVS)))
@pytest.mark.parametrize("workload", ["c3", "c5"])
def test_planner_options_keep_the_state(env, workload, monkeypatch):
    """Window search (tiles seeded with every window of consecutive bits), its
    beam search and tile shrinking only move pass boundaries / tile bits: the
    replayed plan must still match the oracle, and on the layered circuit the
    window search must not need more passes than the first-need greedy."""
    w = W.config3(n=12, layers=8) if workload == "c3" else W.config5(n=11, ngates=250, nmods=0)
    geom = dict(tile_qubits=7, reg_bits=3, low_bits=2)
    base = json.loads(jit_probe(w.n, w.gates, source_pass=-2, **geom))
    for k, v in PLANNER_ENVS[env].items():
        monkeypatch.setenv(k, v)
    plan = json.loads(jit_probe(w.n, w.gates, source_pass=-2, **geom))
    if any(p["kind"] != "lowered" for p in plan["passes"]):
        pytest.skip("plan has generic passes")
    psi0 = np.zeros(1 << w.n, dtype=np.complex128)
    psi0[0] = 1.0
    got = apply_lowered(psi0, plan)
    want = oracle.simulate(w.n, lower_to_reference(w.gates))
    assert np.abs(got - want).max() <= 1e-12
    if workload == "c3" and "QTB_WINDOW_SEARCH" in PLANNER_ENVS[env] and "QTB_PASS_FP64" not in PLANNER_ENVS[env] \
            and "QTB_SHRINK_MIN" not in PLANNER_ENVS[env]:
        assert len(plan["passes"]) <= len(base["passes"])
