for tb in 10 11 12 13; do
QTB_TILE_BITS=$tb python - <<'PY'
import sys, time, os, statistics
sys.path.insert(0,'/root/repo')
from paper_2210_01076_b200 import Config, Simulator, workloads as W
w=W.config1()
sim=Simulator(w.n, Config()); drv=W.NetDriver(sim); drv.build(w.gates); sim.update_state()
lat=[]; ps=[]
for rep in range(3):
  for m,mod in enumerate(w.modifiers[:20]):
    t0=time.perf_counter(); drv.modify(mod); sim.update_state(); lat.append((time.perf_counter()-t0)*1e3); ps.append(sim.last_update().passes)
print('tile', os.environ['QTB_TILE_BITS'], 'mean ms', round(statistics.mean(lat),4), 'median', round(statistics.median(lat),4), 'mean passes', statistics.mean(ps), 'norm', sim.norm_squared())
PY
done
