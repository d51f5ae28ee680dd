"""Profiling driver: one warm-up + one timed full simulation of a workload
(default: config 3 at 30 qubits) through StateVector, for ncu captures.

  python tools/prof_pass.py [--workload c3] [--n 30] [--layers 20]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_01076_b200 import StateVector, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--layers", type=int, default=20)
ap.add_argument("--tile-qubits", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()

if args.workload == "c3":
    w = W.config3(n=args.n, layers=args.layers)
elif args.workload == "c2":
    w = W.config2(n=args.n)
elif args.workload == "c5":
    w = W.config5(n=args.n, nmods=0)
else:
    w = W.config4(n=args.n)
st = StateVector(w.n, tile_qubits=args.tile_qubits)
st.set_timing(True)
for r in range(args.reps):
    st.set_basis(w.basis)
    t0 = time.perf_counter()
    st.apply(w.gates)
    st.sync()
    dt = time.perf_counter() - t0
    tim = st.last_timings()
    print(json.dumps({"rep": r, "wall_ms": dt * 1e3, "passes": len(tim),
                      "pass_ms": [round(x[1], 3) for x in tim]}))
print("norm", st.norm_squared())
