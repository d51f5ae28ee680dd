"""Supplementary measurements of the other BASELINE.json configs on one B200
(the headline config 3 is bench.py). Prints one JSON object.

  python tools/bench_configs.py [--c5-mods 1000] [--skip c4]

* c2: 24-qubit QFT of a seeded basis state; parity vs the exact closed form.
* c4: 33-qubit random circuit (128 GiB state, fits one B200), full simulation,
      then the mirror circuit C^dagger back to |0...0> (parity without CPU state);
      plus the same circuit family at 30 qubits as a LOOPBACK 8-shard state
      (the sharded scheduler: exchanges for non-diagonal targets on the top 3
      qubits) vs the unsharded run.
* c5: 28 qubits, 5000 gates, 1000 alternating insert/remove modifiers through
      the Simulator API: per-modifier latency by position class.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2210_01076_b200 import StateVector, workloads as W  # noqa: E402
from paper_2210_01076_b200.gates import GateKind as K  # noqa: E402
from paper_2210_01076_b200.gates import gate, gate_array  # noqa: E402


def timed_apply(st, gates, reps=2):
    best = None
    for _ in range(reps):
        st.set_basis(0)
        st.sync()
        t0 = time.perf_counter()
        st.apply(gates)
        st.sync()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


def inverse(gates):
    rows = []
    for g in gates[::-1].tolist():
        kind, t, c, _, th, ph, la = g
        kind = K(kind)
        if kind in (K.Rx, K.Ry, K.Rz):
            rows.append(gate(kind, t, c, -th))
        elif kind == K.U3:
            rows.append(gate(K.U3, t, -1, -th, -la, -ph))
        else:
            rows.append(gate(kind, t, c))
    return gate_array(rows)


def c2():
    w = W.config2()
    out = {"workload": w.name, "gates": w.metric_gates}
    for mode in ("interpreted", "compiled"):
        st = StateVector(w.n, compiled=mode == "compiled")
        st.set_basis(0)
        st.apply(w.gates)          # compiled: builds the passes (process cache)
        st.sync()
        t0 = time.perf_counter()
        st.set_basis(0)
        st.apply(w.gates)
        st.sync()
        sec = time.perf_counter() - t0
        got = st.read()
        dev = float(np.abs(got - W.qft_closed_form(w.n, w.basis)).max())
        out[mode] = {"seconds": sec, "amp_gate_per_s": w.metric_gates * (1 << w.n) / sec,
                     "passes": st.stats()["passes"], "max_abs_diff_vs_closed_form": dev,
                     "norm_error": abs(st.norm_squared() - 1.0)}
        st.close()
    return out


def c4():
    w = W.config4()
    out = {"workload": w.name, "qubits": w.n, "state_gib": 16 * (1 << w.n) / 2**30,
           "gates": w.metric_gates}
    for mode in ("interpreted", "compiled"):
        st = StateVector(w.n, compiled=mode == "compiled")
        if mode == "compiled":
            st.apply(w.gates)      # build the passes (outside the timing)
            st.sync()
        sec = timed_apply(st, w.gates, reps=1)
        passes = st.stats()["passes"]
        nrm = st.norm_squared()
        st.apply(inverse(w.gates))
        head = st.read(0, 1 << 10)
        mirror = max(abs(head[0] - 1.0), float(np.abs(head[1:]).max()))
        st.close()
        out[mode] = {"seconds": sec, "passes": passes,
                     "amp_gate_per_s": w.metric_gates * (1 << w.n) / sec,
                     "norm_error": abs(nrm - 1.0), "mirror_max_abs_diff": mirror}
    # the sharded scheduler at 30 qubits: loopback 8 shards vs unsharded
    w30 = W.config4(n=30, ngates=1500)
    single = StateVector(30)
    t_single = timed_apply(single, w30.gates, reps=1)
    a = single.read(0, 1 << 20)
    single.close()
    lb = StateVector(30, mode="loopback", shards=8)
    t_lb = timed_apply(lb, w30.gates, reps=1)
    s = lb.stats()
    b = lb.read(0, 1 << 20)
    lb.close()
    out["loopback8_n30"] = {"seconds_unsharded": t_single, "seconds_loopback8": t_lb,
                            "exchanges": s["swaps"], "exchanged_bytes": s["exchanged_bytes"],
                            "max_abs_diff_vs_unsharded_first_2^20": float(np.abs(a - b).max())}
    return out


def c5(nmods):
    from bench import measure_incremental
    from paper_2210_01076_b200 import Config, Simulator
    w = W.config5(nmods=nmods)
    return dict(measure_incremental(lambda n: Simulator(n, Config()), w, nmods),
                workload=w.name, modifiers=nmods)


def topk():
    """Device top-K readout (qt_top_k) of the C3 final state at 30 qubits vs
    the full-state D2H copy it replaces."""
    w = W.config3()
    st = StateVector(w.n)
    st.apply(w.gates)
    st.sync()
    out = {"qubits": w.n}
    for k in (16, 4096):
        st.top_k(k)
        t0 = time.perf_counter()
        idx, amps = st.top_k(k)
        dt = time.perf_counter() - t0
        out[f"k{k}_seconds"] = dt
        out[f"k{k}_first"] = [int(idx[0]), abs(complex(amps[0])) ** 2]
    half = np.empty(1 << (w.n - 1), dtype=np.complex128)
    t0 = time.perf_counter()
    st.read(0, 1 << (w.n - 1), out=half)
    out["d2h_full_state_seconds_est"] = 2 * (time.perf_counter() - t0)
    st.close()
    return out


ap = argparse.ArgumentParser()
ap.add_argument("--c5-mods", type=int, default=1000)
ap.add_argument("--skip", nargs="*", default=[])
args = ap.parse_args()
res = {}
for name, fn in (("c2", c2), ("c4", c4), ("c5", lambda: c5(args.c5_mods)), ("topk", topk)):
    if name in args.skip:
        continue
    try:
        res[name] = fn()
    except Exception as e:
        res[name] = {"error": f"{type(e).__name__}: {e}"}
    print(json.dumps({name: res[name]}), flush=True)
print(json.dumps(res))
