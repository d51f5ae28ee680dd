"""Full-size parity on the driver's GPU run (slow: ~6 min of host oracle
time on the GPU box's 16 cores): BASELINE config 5 at its full 28 qubits
through the incremental Simulator API, after the base simulation and its
first modifier (an incremental update), against the multithreaded oracle
(oracle/qt_oracle.c, memcmp-pinned to the reference oracle.cpp:15-50) on the
modified 5001-gate circuit. Named to run last."""
import time

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import Config, Simulator, workloads as W
from paper_2210_01076_b200.gates import lower_to_reference

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c5_full_size_after_one_modifier(gpu):
    w = W.config5()
    sim = Simulator(w.n, Config())
    drv = W.NetDriver(sim)
    drv.build(w.gates)
    sim.update_state()
    drv.modify(w.modifiers[0])
    sim.update_state()
    after = sim.amplitudes(0, (1 << w.n) - 1)
    nrm = sim.norm_squared()
    sim.close()
    t0 = time.perf_counter()
    want1 = oracle.simulate(w.n, lower_to_reference(W.apply_modifier(w.gates, w.modifiers[0])))
    d1 = float(np.abs(after - want1).max())
    print(f"c5 n=28 after modifier 1: max|d|={d1:.3e} |norm-1|={abs(nrm - 1):.3e} "
          f"oracle {time.perf_counter() - t0:.0f} s")
    assert d1 <= 1e-10
    assert abs(nrm - 1.0) <= 1e-12
