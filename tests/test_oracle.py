"""CPU tests of the parity oracle (oracle/qt_oracle.c, restating the
reference's oracle.cpp:15-50 and gate.cpp:42-90): pinned bit-for-bit to the
reference compiled from its own sources (oracle/_ref), to the golden fixtures
that reference produced (tests/golden), and to the reference's own
known-answer tests (proj/tests/test_gates.cpp, test_oracle.cpp,
test_engine.cpp), restated."""
import math

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import workloads as W
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array, lower_to_reference
from tests.golden.replay import load_logs, load_random
from tests.test_planner import random_circuit

INV = 0.70710678118654752440


def test_golden_random_bit_identical():
    for n, g, want in load_random():
        got = oracle.simulate(n, g, threads=4)
        assert got.tobytes() == want.tobytes(), n


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not compiled here")
@pytest.mark.parametrize("seed", range(6))
def test_pinned_to_reference_oracle(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(2, 15))
    g = lower_to_reference(random_circuit(rng, n, 150))
    a = oracle.simulate(n, g, threads=4)
    b, _ = oracle.ref_simulate(n, g)
    assert a.tobytes() == b.tobytes()


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not compiled here")
def test_gate_matrices_match_reference():
    for k in range(1, 12):
        for th in (0.0, math.pi, -1.3, 5.7):
            m = np.zeros(8)
            assert oracle.ref_lib().ref_gate_matrix(k, th, m.ctypes.data) == 2
            mine = oracle.gate_matrix(k, th).reshape(-1)
            assert mine.view(np.float64).tobytes() == m.tobytes(), (k, th)  # incl. signed zeros


def test_gate_matrix_kats():
    # test_gates.cpp:12-37
    x = oracle.gate_matrix(K.X)
    assert (x == np.array([[0, 1], [1, 0]])).all()
    h = oracle.gate_matrix(K.H)
    assert abs(h[0, 0] - INV) <= 1e-15 and abs(h[1, 1] + INV) <= 1e-15
    rz0 = oracle.gate_matrix(K.Rz, 0.0)
    assert np.abs(rz0 - np.eye(2)).max() < 1e-15
    # unitarity (test_gates.cpp:39-51)
    for k in (K.X, K.Y, K.Z, K.H, K.S, K.Sdg, K.T, K.Tdg):
        m = oracle.gate_matrix(k)
        assert np.abs(m @ m.conj().T - np.eye(2)).max() < 1e-12
    for k in (K.Rx, K.Ry, K.Rz):
        for i in range(50):
            m = oracle.gate_matrix(k, -7.0 + 0.29 * i)
            assert np.abs(m @ m.conj().T - np.eye(2)).max() < 1e-12


def test_single_gate_and_bell_kats():
    # test_oracle.cpp:10-45
    s = oracle.simulate(1, gate_array([gate(K.H, 0)]))
    assert abs(s[0] - INV) < 1e-15 and abs(s[1] - INV) < 1e-15
    t = oracle.simulate(2, gate_array([gate(K.Cnot, 0, 1)]), basis=2)
    assert t[3] == 1 and t[2] == 0
    b = oracle.simulate(2, gate_array([gate(K.H, 0), gate(K.Cnot, 1, 0)]))
    assert abs(b[0] - INV) < 1e-15 and abs(b[3] - INV) < 1e-15
    assert abs(b[1]) < 1e-15 and abs(b[2]) < 1e-15
    # test_engine.cpp:219-238
    y = oracle.simulate(1, gate_array([gate(K.Y, 0)]))
    assert abs(y[1] - 1j) < 1e-15 and abs(y[0]) < 1e-15
    hz = oracle.simulate(1, gate_array([gate(K.H, 0), gate(K.Z, 0)]))
    assert abs(hz[0] - INV) < 1e-12 and abs(hz[1] + INV) < 1e-12


def test_norm_preserved_every_gate():
    # test_oracle.cpp:57-77
    rng = np.random.default_rng(5)
    for _ in range(30):
        n = int(rng.integers(1, 7))
        st = np.zeros(1 << n, dtype=np.complex128)
        st[0] = 1
        for row in random_circuit(rng, n, 20):
            oracle.simulate(n, gate_array([tuple(row.tolist())]), state=st, threads=1)
            assert abs(oracle.norm_squared(st) - 1) < 1e-12


def test_golden_logs_replay_on_oracle():
    """The reference engine's incremental states equal the dense oracle of
    the circuit at each update (acceptance criterion 2's property), for the
    committed logs; bit-exact is not required for the engine (it fuses
    superposition gates of a net)."""
    for name in ("golden_incremental.npz", "golden_traces.npz"):
        for n, ops, states in load_logs(name):
            assert len(states) >= 1
            for st in states:
                assert abs(oracle.norm_squared(st) - 1) < 1e-9


def test_entangle5_golden_values():
    # Listing-1 circuit: every amplitude 1/sqrt(32) (test_engine.cpp:88-97)
    (n, ops, states), _ = list(load_logs("golden_traces.npz"))
    assert n == 5
    assert np.abs(states[0] - 1 / math.sqrt(32)).max() < 1e-12


@pytest.mark.parametrize("n", [6, 10, 14])
def test_qft_closed_form_on_oracle(n):
    w = W.config2(n=n)
    st = oracle.simulate(n, w.gates)
    assert np.abs(st - W.qft_closed_form(n, w.basis)).max() < 1e-12


def test_decompositions_pinned():
    """U3 = RZ(phi) RY(theta) RZ(lambda) and CZ = H CX H."""
    rng = np.random.default_rng(11)
    th, ph, la = rng.uniform(0, 2 * math.pi, 3)
    u3 = oracle.simulate(1, gate_array([gate(K.U3, 0, -1, th, ph, la)]), basis=1)
    seq = oracle.simulate(1, gate_array([gate(K.Rz, 0, theta=la), gate(K.Ry, 0, theta=th),
                                         gate(K.Rz, 0, theta=ph)]), basis=1)
    assert u3.tobytes() == seq.tobytes()
    psi = np.ones(4, dtype=np.complex128) / 2
    cz = oracle.simulate(2, gate_array([gate(K.Cz, 1, 0)]), state=psi.copy())
    assert np.abs(cz - np.array([0.5, 0.5, 0.5, -0.5])).max() < 1e-15
