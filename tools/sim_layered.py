"""The layered headline circuit (C3) through the drop-in Simulator API: full
update cold, then a modifier in the first net (everything downstream is
re-simulated: a warm full pass over the cached segment plans) and one in the
last net. python tools/sim_layered.py [--n 30]"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_01076_b200 import Config, Simulator, jit_wait, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--seg", type=int, default=0)
args = ap.parse_args()
w = W.config3(n=args.n, layers=20)
sim = Simulator(w.n, Config(segment_gates=args.seg))
drv = W.NetDriver(sim)
drv.build(w.gates)
t0 = time.perf_counter(); sim.update_state(); cold = (time.perf_counter() - t0) * 1e3
st = sim.last_update()
jit_wait(300)
out = {"seg": args.seg, "n": w.n, "gates": len(w.gates), "cold_full_ms": cold, "passes": st.passes, "segments": st.segments}
from paper_2210_01076_b200.gates import GateKind as K
lat = []
for rep in range(4):
    # insert an RZ on qubit 0 in a new net at the front, update, remove it, update
    net = sim.insert_net_front()
    sim.insert_gate(K.Rz, 0.3 + rep, net, 0)
    t0 = time.perf_counter(); sim.update_state(); a = (time.perf_counter() - t0) * 1e3
    sim.remove_net(net)
    t0 = time.perf_counter(); sim.update_state(); b = (time.perf_counter() - t0) * 1e3
    lat += [a, b]
    jit_wait(300)
out["warm_full_update_ms"] = [round(x, 1) for x in lat]
out["last_passes"] = sim.last_update().passes
out["norm_error"] = abs(sim.norm_squared() - 1)
sim.close()
print(json.dumps(out))
