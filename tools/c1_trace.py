import sys, time
sys.path.insert(0,'/root/repo')
from paper_2210_01076_b200 import Config, Simulator, workloads as W
w=W.config1()
sim=Simulator(w.n, Config()); drv=W.NetDriver(sim); drv.build(w.gates); sim.update_state()
for m,mod in enumerate(w.modifiers[:8]):
    t0=time.perf_counter(); drv.modify(mod); t1=time.perf_counter(); sim.update_state(); t2=time.perf_counter()
    st=sim.last_update()
    print(f"mod {m}: modify {1e3*(t1-t0):.3f} ms update {1e3*(t2-t1):.3f} ms passes {st.passes} segments {st.segments} plan_ms {getattr(st,'plan_ms',0)}", file=sys.stderr)
