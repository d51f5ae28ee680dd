import sys, time
sys.path.insert(0, '.')
from paper_2210_01076_b200 import Config, Simulator, workloads as W
from paper_2210_01076_b200.gates import GateKind as K, gate
g = W.qft_gates(16, 12345)
sim = Simulator(16, Config())
drv = W.NetDriver(sim)
drv.build(g)
sim.update_state()
ts = []
for i in range(8):
    t0 = time.perf_counter()
    drv.modify(("insert", 40 * i + 5, gate(K.H, i % 16)))
    sim.update_state()
    ts.append((time.perf_counter() - t0) * 1e3)
print("ms per update", [round(t, 3) for t in ts])
