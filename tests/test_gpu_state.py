"""GPU parity of the fused sm_100a gate path (qt_state_* C ABI) against the
dense oracle (oracle/, bit-pinned to the reference oracle.cpp:15-50).

Bar (BASELINE.json north_star): per-amplitude max |diff| <= 1e-10 and
|norm^2 - 1| <= 1e-12 for complex128."""
import math

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import StateVector, workloads as W
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array, lower_to_reference
from tests.test_planner import random_circuit, random_state

pytestmark = pytest.mark.gpu
TOL = 1e-10
NORM_TOL = 1e-12


def run_gpu(n, gates, psi0=None, **kw):
    st = StateVector(n, **kw)
    if psi0 is not None:
        st.write(psi0)
    st.apply(gates)
    out = st.read()
    nrm = st.norm_squared()
    st.close()
    return out, nrm


def test_single_gate_kats(gpu):
    inv = 1 / math.sqrt(2)
    out, _ = run_gpu(1, gate_array([gate(K.H, 0)]))
    assert abs(out[0] - inv) < 1e-15 and abs(out[1] - inv) < 1e-15
    # CNOT(control=q1, target=q0) maps |10> to |11>
    st = StateVector(2)
    st.set_basis(2)
    st.apply(gate_array([gate(K.Cnot, 0, 1)]))
    out = st.read()
    assert out[3] == 1 and out[2] == 0
    # Y|0> = i|1>; H then Z = (1/sqrt2, -1/sqrt2)
    out, _ = run_gpu(1, gate_array([gate(K.Y, 0)]))
    assert abs(out[1] - 1j) < 1e-15 and abs(out[0]) < 1e-15
    out, _ = run_gpu(1, gate_array([gate(K.H, 0), gate(K.Z, 0)]))
    assert abs(out[0] - inv) < 1e-12 and abs(out[1] + inv) < 1e-12
    # Bell
    out, _ = run_gpu(2, gate_array([gate(K.H, 0), gate(K.Cnot, 1, 0)]))
    assert abs(out[0] - inv) < 1e-15 and abs(out[3] - inv) < 1e-15
    assert abs(out[1]) < 1e-15 and abs(out[2]) < 1e-15


def test_entangle5_uniform(gpu):
    # Listing-1 circuit (test_engine.cpp:88-97): every amplitude 1/sqrt(32)
    rows = [gate(K.H, q) for q in range(4, -1, -1)]
    rows += [gate(K.Cnot, 3, 4), gate(K.Cnot, 1, 4), gate(K.Cnot, 2, 3), gate(K.Cnot, 0, 2)]
    out, nrm = run_gpu(5, gate_array(rows))
    assert np.abs(out - 1 / math.sqrt(32)).max() < 1e-12
    assert abs(nrm - 1) < NORM_TOL


@pytest.mark.parametrize("seed", range(40))
def test_random_circuits_vs_oracle(gpu, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 17))
    g = random_circuit(rng, n, int(rng.integers(1, 300)))
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, g, state=psi0.copy())
    for tile in (0, 5):
        got, nrm = run_gpu(n, g, psi0, tile_qubits=tile)
        assert np.abs(got - want).max() <= TOL
        assert abs(nrm - 1) <= NORM_TOL


def test_reference_gate_lowering_equivalence(gpu):
    """Native U3 / CZ == their reference decompositions."""
    w = W.config3(n=12, layers=6)
    got, _ = run_gpu(12, w.gates)
    want = oracle.simulate(12, lower_to_reference(w.gates))
    assert np.abs(got - want).max() <= TOL


def test_config1_full_vs_reference_oracle(gpu):
    w = W.config1()
    got, nrm = run_gpu(w.n, w.gates)
    want = oracle.simulate(w.n, lower_to_reference(w.gates))
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL


@pytest.mark.parametrize("n", [20, 24])
def test_config2_qft_closed_form(gpu, n):
    w = W.config2(n=n)
    got, nrm = run_gpu(n, w.gates)
    want = W.qft_closed_form(n, w.basis)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL


def test_config3_reduced_vs_oracle(gpu):
    w = W.config3(n=22, layers=20)
    got, nrm = run_gpu(22, w.gates)
    want = oracle.simulate(22, w.gates)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL


def inverse(gates):
    """C^dagger: reversed order, each gate inverted (SURVEY 8(c) mirror)."""
    rows = []
    for g in gates[::-1].tolist():
        kind, t, c, _, th, ph, la = g
        kind = K(kind)
        if kind in (K.Rx, K.Ry, K.Rz):
            rows.append(gate(kind, t, c, -th))
        elif kind == K.U3:  # (RZ(p) RY(t) RZ(l))^-1 = RZ(-l) RY(-t) RZ(-p)
            rows.append(gate(K.U3, t, -1, -th, -la, -ph))
        elif kind == K.S:
            rows.append(gate(K.Sdg, t))
        elif kind == K.Sdg:
            rows.append(gate(K.S, t))
        elif kind == K.T:
            rows.append(gate(K.Tdg, t))
        elif kind == K.Tdg:
            rows.append(gate(K.T, t))
        else:
            rows.append(gate(kind, t, c))
    return gate_array(rows)


def test_config3_full_size_mirror(gpu):
    """n=30 headline config: C then C^dagger returns |0...0> (no CPU state
    needed at 16 GiB), plus the norm after C."""
    w = W.config3()
    st = StateVector(30)
    st.apply(w.gates)
    nrm = st.norm_squared()
    st.apply(inverse(w.gates))
    head = st.read(0, 1 << 12)
    nrm2 = st.norm_squared()
    st.close()
    assert abs(nrm - 1) <= NORM_TOL and abs(nrm2 - 1) <= NORM_TOL
    assert abs(head[0] - 1) <= TOL and np.abs(head[1:]).max() <= TOL


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_loopback_sharding_matches_single(gpu, shards):
    """The sharded scheduler (global qubits, exchanges) on one GPU equals the
    unsharded run bit for bit up to reassociation (<= 1e-12)."""
    rng = np.random.default_rng(7 + shards)
    n = 14
    g = random_circuit(rng, n, 200)
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, g, state=psi0.copy())
    got, nrm = run_gpu(n, g, psi0, mode="loopback", shards=shards, tile_qubits=6)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL


def test_config4_shape_loopback(gpu):
    w = W.config4(n=20, ngates=300)
    want = oracle.simulate(20, w.gates)
    for shards in (2, 4, 8):
        got, _ = run_gpu(20, w.gates, mode="loopback", shards=shards)
        assert np.abs(got - want).max() <= TOL


def test_numeric_error_on_nonfinite(gpu):
    from paper_2210_01076_b200.errors import NumericError
    st = StateVector(4)
    psi = np.zeros(16, dtype=np.complex128)
    psi[3] = np.inf
    st.write(psi)
    st.apply(gate_array([gate(K.H, 0)]))
    with pytest.raises(NumericError):
        st.sync()
    st.close()


def test_deterministic_bits(gpu):
    rng = np.random.default_rng(5)
    g = random_circuit(rng, 18, 400)
    a, _ = run_gpu(18, g)
    b, _ = run_gpu(18, g)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("eps", [1e-3, 1e-9])
def test_near_diagonal_u3_layers(gpu, eps):
    """Near-diagonal / near-anti-diagonal U3 layers (the ZYZ split's hard
    cases) at 12 qubits on the GPU vs the oracle."""
    rng = np.random.default_rng(11)
    n = 12
    rows = []
    for layer in range(10):
        for q in range(n):
            th = eps if (q + layer) % 2 else math.pi - eps
            rows.append(gate(K.U3, q, -1, th, *rng.uniform(0, 2 * math.pi, 2)))
        for a in range(layer % 2, n - 1, 2):
            rows.append(gate(K.Cz, a + 1, a))
    g = gate_array(rows)
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, lower_to_reference(g), state=psi0.copy())
    got, nrm = run_gpu(n, g, psi0)
    assert np.abs(got - want).max() < TOL
    assert abs(nrm - 1.0) < NORM_TOL
