"""C5 incremental latency: interpreter vs hybrid compiled passes (cached
segments compiled; the engine warmed by one full update + background
compiles). python tools/c5_hybrid.py [--mods 24] [--n 28]"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import latency_stats  # noqa: E402
from paper_2210_01076_b200 import Config, Simulator, jit_stats, jit_wait, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mods", type=int, default=24)
ap.add_argument("--n", type=int, default=28)
ap.add_argument("--seg", type=int, default=0)
ap.add_argument("--modes", default="-1,0")
args = ap.parse_args()
w = W.config5(n=args.n, nmods=max(args.mods, 2))
for compiled in [int(x) for x in args.modes.split(',')]:
    sim = Simulator(w.n, Config(compiled=compiled, segment_gates=args.seg))
    drv = W.NetDriver(sim)
    drv.build(w.gates)
    t0 = time.perf_counter(); sim.update_state(); full = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter(); ok = jit_wait(300) if compiled >= 0 else True; wait = time.perf_counter() - t0
    lat = {"uniform": [], "tail": []}
    passes = []
    plan_ms = []
    from paper_2210_01076_b200 import _ffi, lib
    import ctypes
    for m, mod in enumerate(w.modifiers[:args.mods]):
        cls = "tail" if (m // 2) % 2 == 1 else "uniform"
        t0 = time.perf_counter(); drv.modify(mod); sim.update_state()
        lat[cls].append((time.perf_counter() - t0) * 1e3)
        passes.append(sim.last_update().passes)
        rs = _ffi.QtRunStats()
        lib().qt_sim_last_update(sim._h, ctypes.byref(rs))
        plan_ms.append(rs.plan_ms)
    nrm = sim.norm_squared()
    amps = sim.amplitudes(0, 1 << 10)
    sim.close()
    print(json.dumps({"compiled": compiled, "seg": args.seg, "mean_passes": sum(passes) / len(passes), "mean_plan_ms": sum(plan_ms) / len(plan_ms), "full_ms": full, "bg_wait_s": wait, "bg_done": ok,
                      "uniform": latency_stats(lat["uniform"]), "tail": latency_stats(lat["tail"]),
                      "norm_error": abs(nrm - 1), "amp0": [amps[0].real, amps[0].imag],
                      "jit": jit_stats()}), flush=True)
