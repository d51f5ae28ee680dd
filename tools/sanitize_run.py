"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
both tile-pass kernel families (the layer-word interpreter and the compiled
ring kernel, with enough tiles per CTA that the ring reaches its steady
state), the incremental engine with modifiers, top-K, the norm, and a
sharded in-process rank group with exchanges. Checks results against the
oracle so a silent corruption also fails.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2210_01076_b200 import (Config, RankGroup, Simulator, StateVector,  # noqa: E402
                                   lower_to_reference, workloads as W)

n = int(os.environ.get("QTB_SAN_N", "21"))
w = W.config3(n=n, layers=3)
want = oracle.simulate(n, lower_to_reference(w.gates))
for compiled in (False, True):
    st = StateVector(n, compiled=compiled)
    st.apply(w.gates)
    got = st.read()
    idx, _ = st.top_k(8)
    nrm = st.norm_squared()
    st.close()
    assert np.abs(got - want).max() < 1e-10 and abs(nrm - 1) < 1e-12, compiled
    print("tile passes ok, compiled =", compiled, flush=True)

w4 = W.config4(n=14, ngates=120)
g = RankGroup(14, 4)
g.apply(w4.gates)
got = g.read()
g.close()
assert np.abs(got - oracle.simulate(14, lower_to_reference(w4.gates))).max() < 1e-10
print("rank group ok", flush=True)

w5 = W.config5(n=12, ngates=300, nmods=6)
sim = Simulator(12, Config())
drv = W.NetDriver(sim)
drv.build(w5.gates)
sim.update_state()
gates = w5.gates
for mod in w5.modifiers:
    drv.modify(mod)
    sim.update_state()
    gates = W.apply_modifier(gates, mod)
got = sim.amplitudes(0, (1 << 12) - 1)
sim.close()
assert np.abs(got - oracle.simulate(12, lower_to_reference(gates))).max() < 1e-10
print("incremental engine ok", flush=True)
print("sanitize workload done")
