"""GPU parity against the golden fixtures produced by the reference itself
(tests/golden/make_golden.py): dense-oracle states of random circuits, and
the reference qtask::Simulator's states after every update_state of random
modifier logs, replayed through the GPU drop-in (qt_sim_* C ABI)."""
import numpy as np
import pytest

from paper_2210_01076_b200 import Config, Simulator, StateVector
from tests.golden.replay import load_logs, load_random, replay

pytestmark = pytest.mark.gpu


def test_golden_random_circuits(gpu):
    for n, g, want in load_random():
        st = StateVector(n)
        st.apply(g)
        got = st.read()
        st.close()
        assert np.abs(got - want).max() <= 1e-10, n


@pytest.mark.parametrize("name", ["golden_incremental.npz", "golden_traces.npz"])
@pytest.mark.parametrize("segment", [0, 1, 3])
def test_golden_modifier_logs(gpu, name, segment):
    for n, ops, states in load_logs(name):
        sim = Simulator(n, Config(4, 1, max_checkpoints=3, segment_gates=segment))

        def check(i):
            got = sim.amplitudes(0, (1 << n) - 1)
            assert np.abs(got - states[i]).max() <= 1e-10, (name, i)
            assert abs(sim.norm_squared() - 1) <= 1e-12

        replay(sim, ops, check)
        sim.close()
