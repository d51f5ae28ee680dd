"""Device-side top-K readout: the reference's amplitude
report (tools/qtask_cli.cpp:53-86) -- std::partial_sort of the indices by
std::norm descending, index ascending -- restated in numpy as the checker
(norm = re*re + im*im without FMA, exactly like libstdc++'s std::norm)."""
import numpy as np
import pytest

from paper_2210_01076_b200 import Config, Simulator, StateVector
from paper_2210_01076_b200.errors import StaleStateError
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array
from tests.test_planner import random_circuit, random_state

pytestmark = pytest.mark.gpu


def expected(psi, k):
    nrm = psi.real * psi.real + psi.imag * psi.imag
    order = np.lexsort((np.arange(len(psi)), -nrm))[:k]
    return order.astype(np.uint64), psi[order]


def check(st, psi, k):
    idx, amps = st.top_k(k)
    want_i, want_a = expected(psi, k)
    assert len(idx) == min(k, len(psi))
    assert (idx == want_i).all()
    assert (amps == want_a).all()  # the stored amplitudes themselves


@pytest.mark.parametrize("k", [1, 7, 1000, 1 << 14])
def test_random_state(gpu, k):
    rng = np.random.default_rng(k)
    n = 16
    psi = random_state(rng, n)
    st = StateVector(n)
    st.write(psi)
    check(st, psi, k)
    st.close()


def test_uniform_superposition_ties(gpu):
    """Every |a|^2 equal: the exact threshold path ranks the ties by index."""
    n = 20
    st = StateVector(n)
    st.apply(gate_array([gate(K.H, q) for q in range(n)]))
    psi = st.read()
    for k in (1, 100, 5000):
        check(st, psi, k)
    st.close()


def test_near_ties_across_a_binade(gpu):
    """Keys one or two ulps apart on both sides of a power of two (a nearly
    uniform state): the radix digits split high up and the last, narrower
    digit must still be read below the chosen prefix."""
    rng = np.random.default_rng(11)
    n = 20
    base = 2.0 ** -10
    lo = np.nextafter(base, 0.0)
    hi = np.nextafter(base, 1.0)
    vals = rng.choice([lo, base, hi, np.nextafter(hi, 1.0)], size=1 << n, p=[0.45, 0.45, 0.0998, 0.0002])
    psi = vals.astype(np.complex128)
    st = StateVector(n)
    st.write(psi)
    for k in (1, 100, 5000, 300000):
        check(st, psi, k)
    st.close()


def test_quantised_amplitudes_many_ties(gpu):
    rng = np.random.default_rng(5)
    n = 18
    vals = rng.integers(-3, 4, size=(1 << n)) + 1j * rng.integers(-3, 4, size=(1 << n))
    psi = (vals / np.linalg.norm(vals)).astype(np.complex128)
    st = StateVector(n)
    st.write(psi)
    for k in (3, 777, 20000, 1 << n):
        check(st, psi, k)
    st.close()


def test_circuit_state_large(gpu):
    rng = np.random.default_rng(9)
    n = 24
    st = StateVector(n)
    st.apply(random_circuit(rng, n, 300))
    psi = st.read()
    check(st, psi, 2048)
    st.close()


def test_loopback_permuted_state(gpu):
    """Loopback shards end with a permuted qubit map: the report is in
    logical indices (chunks gathered in logical order)."""
    rng = np.random.default_rng(3)
    n = 14
    g = random_circuit(rng, n, 150)
    st = StateVector(n, mode="loopback", shards=4)
    st.apply(g)
    psi = st.read()
    assert st.stats()["swaps"] > 0
    check(st, psi, 300)
    st.close()


def test_simulator_top_k_and_stale(gpu):
    sim = Simulator(3, Config())
    net = sim.insert_net_back()
    sim.insert_gate(K.H, net, 0)
    sim.insert_gate(K.Cnot, sim.insert_net_back(), 1, 0)
    with pytest.raises(StaleStateError):
        sim.top_k(2)
    sim.update_state()
    idx, amps = sim.top_k(4)
    # |00> and |11> (equal up to rounding: their order follows the computed norms)
    assert sorted(idx.tolist()[:2]) == [0, 3] and abs(abs(amps[0]) - 2 ** -0.5) < 1e-15
    nrm = np.abs(amps) ** 2
    assert (np.diff(nrm) <= 0).all()
    sim.close()
