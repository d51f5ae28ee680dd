"""Kernel microbenchmarks: FP64 efficiency of the tile pass on synthetic
single-pass circuits (all gates on the low qubits, so the whole circuit is one
pass; R=QTB_REG_BITS register rounds of max_round_ops ops).

  python tools/microbench.py [--n 26] [--layers 200]
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

from paper_2210_01076_b200 import StateVector, plan_probe, probe_fp64  # noqa: E402
from paper_2210_01076_b200.gates import GateKind as K  # noqa: E402
from paper_2210_01076_b200.gates import gate, gate_array  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=26)
ap.add_argument("--layers", type=int, default=200)
args = ap.parse_args()
rng = np.random.default_rng(0)
R = int(os.environ.get("QTB_REG_BITS", "4"))


def circuit(kind):
    rows = []
    for _ in range(args.layers):
        for q in range(R):
            if kind == "ry":
                rows.append(gate(K.Ry, q, theta=float(rng.uniform(0, 6.28))))
            elif kind == "u3":
                rows.append(gate(K.U3, q, -1, *rng.uniform(0, 6.28, 3)))
            elif kind == "h":
                rows.append(gate(K.H, q))
        for a in range(0, R - 1, 2):
            rows.append(gate(K.Cz, a + 1, a))
        for a in range(1, R - 1, 2):
            rows.append(gate(K.Cz, a + 1, a))
    return gate_array(rows)


peak = probe_fp64(0)
st = StateVector(args.n)
st.set_timing(True)
for kind in ("ry", "u3", "h"):
    g = circuit(kind)
    plan = json.loads(st.plan_json(g))
    tiles = [p for p in plan["passes"] if p["kind"] == "tile"]
    fp = sum(p["fp64_per_amp"] for p in tiles)
    st.apply(g)
    st.sync()
    st.last_timings()
    t0 = time.perf_counter()
    st.apply(g)
    st.sync()
    ms = sum(x[1] for x in st.last_timings())
    eff = fp * (1 << args.n) / (ms * 1e-3) / peak
    print(json.dumps({"kind": kind, "R": R, "passes": len(tiles),
                      "rounds": sum(p["rounds"] for p in tiles),
                      "device_ops": sum(p["device_ops"] for p in tiles),
                      "fp64_per_amp": fp, "ms": round(ms, 3),
                      "fp64_eff": round(eff, 3),
                      "hbm_ms": round(len(tiles) * 32 * (1 << args.n) / 6556e9 * 1e3, 3)}))
