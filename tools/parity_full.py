"""Full-size parity of the GPU path against the CPU oracle:
the multithreaded restatement of oracle.cpp:15-50 (oracle/qt_oracle.c, pair
loop split across all host threads, per-pair arithmetic as written) runs the
SAME lowered gate list at the configs' full sizes. Too slow for pytest (tens
of minutes of host time); run on the GPU box, results go to profiles/.

  python tools/parity_full.py c3            # 30 qubits, 890 gates (2670 reference gates)
  python tools/parity_full.py c5 --mods 1000  # 28 qubits: base + after modifiers 1/250/500/1000
  python tools/parity_full.py c4            # C4 family at 30 qubits, loopback 8 shards

Prints one JSON object per config: max |delta| over all 2^n amplitudes, the
oracle's pairwise norm of the GPU state, timings, host threads.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (the checker)
from paper_2210_01076_b200 import Config, Simulator, StateVector  # noqa: E402
from paper_2210_01076_b200 import workloads as W  # noqa: E402
from paper_2210_01076_b200.gates import lower_to_reference  # noqa: E402

CHUNK = 1 << 24


def max_abs_diff(a, b):
    d = 0.0
    for i in range(0, len(a), CHUNK):
        d = max(d, float(np.abs(a[i:i + CHUNK] - b[i:i + CHUNK]).max()))
    return d


def host_info():
    mem = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    mem = int(line.split()[1]) * 1024 / 2**30
    except OSError:
        pass
    return {"threads": os.cpu_count(), "host_mem_gib": mem}


def oracle_state(n, gates):
    ref = lower_to_reference(gates)
    t0 = time.perf_counter()
    st = oracle.simulate(n, ref, threads=os.cpu_count())
    return st, time.perf_counter() - t0, len(ref)


def compare(n, got, gates, label, want=None):
    """got: one GPU state or a dict {mode: state} checked against ONE oracle run."""
    sec, nref = 0.0, len(lower_to_reference(gates))
    if want is None:
        want, sec, nref = oracle_state(n, gates)
    states = got if isinstance(got, dict) else {"": got}
    rows = []
    for mode, g in states.items():
        out = {"case": label + (f" [{mode}]" if mode else ""), "qubits": n,
               "logical_gates": len(gates), "reference_gates": nref,
               "oracle_seconds": sec, "max_abs_diff": max_abs_diff(g, want),
               "norm_error_gpu_state": abs(oracle.norm_squared(g) - 1.0),
               "norm_error_oracle_state": abs(oracle.norm_squared(want) - 1.0)}
        out["pass"] = out["max_abs_diff"] <= 1e-10 and out["norm_error_gpu_state"] <= 1e-12
        rows.append(out)
    del want
    return rows if isinstance(got, dict) else rows[0]


def run_modes(n, gates, **kw):
    """The circuit on a fresh state per device path: the interpreter kernel
    and the compiled passes (second apply: every pass from the cache)."""
    got, secs = {}, {}
    for mode in ("interpreted", "compiled"):
        st = StateVector(n, compiled=mode == "compiled", **kw)
        if mode == "compiled":
            st.apply(gates)        # builds the passes
        st.set_basis(0)
        t0 = time.perf_counter()
        st.apply(gates)
        st.sync()
        secs[mode] = time.perf_counter() - t0
        got[mode] = st.read()
        st.close()
    return got, secs


def c3(args):
    w = W.config3(n=args.n) if args.n else W.config3()
    got, secs = run_modes(w.n, w.gates)
    rows = compare(w.n, got, w.gates, w.name)
    for r, mode in zip(rows, got):
        r["gpu_seconds"] = secs[mode]
    return rows


def c5(args):
    """Base state, then after modifiers 1, 250, 500 and 1000."""
    w = W.config5(n=args.n, nmods=args.mods) if args.n else W.config5(nmods=args.mods)
    sim = Simulator(w.n, Config())   # hybrid compiled passes (the engine's default)
    drv = W.NetDriver(sim)
    drv.build(w.gates)
    sim.update_state()
    res = [compare(w.n, sim.amplitudes(0, (1 << w.n) - 1), w.gates, f"{w.name} base")]
    marks = sorted({m for m in (1, 250, 500, args.mods) if m <= args.mods})
    gates = w.gates
    mod_s = 0.0
    for m, mod in enumerate(w.modifiers[:args.mods], start=1):
        t0 = time.perf_counter()
        drv.modify(mod)
        sim.update_state()
        mod_s += time.perf_counter() - t0
        gates = W.apply_modifier(gates, mod)
        if m in marks:
            out = compare(w.n, sim.amplitudes(0, (1 << w.n) - 1), gates,
                          f"{w.name} after {m} modifiers")
            out["gpu_modifier_seconds_so_far"] = mod_s
            res.append(out)
    sim.close()
    return res


def c4(args):
    """The config-4 circuit family at 30 qubits on a LOOPBACK 8-shard state
    (the sharded scheduler: top 3 qubits global, exchanges) vs the oracle
    (SURVEY.md 8(c), C4 parity chain item 3)."""
    n = args.n or 30
    w = W.config4(n=n, ngates=1500)
    got, secs = run_modes(n, w.gates, mode="loopback", shards=8)
    rows = compare(n, got, w.gates, f"{w.name} loopback 8 shards")
    for r, mode in zip(rows, got):
        r["gpu_seconds"] = secs[mode]
    return rows


ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+", choices=["c3", "c4", "c5"])
ap.add_argument("--mods", type=int, default=1000)
ap.add_argument("--n", type=int, default=0, help="override the qubit count (quick check)")
args = ap.parse_args()
print(json.dumps({"host": host_info()}), flush=True)
for name in args.configs:
    for row in {"c3": c3, "c4": c4, "c5": c5}[name](args):
        print(json.dumps(row), flush=True)
