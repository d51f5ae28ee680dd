"""Streaming-efficiency probe of the tile pass: one cheap pass (a single
RY on qubit q) over a 30-qubit state, per tile shape, interpreter and
compiled modes. Prints GB/s of the pass (algorithmic 32 B / amplitude).

  python tools/membench.py [--n 30] [--reps 5]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--child", default="")
args = ap.parse_args()

if args.child:
    from paper_2210_01076_b200 import StateVector
    from paper_2210_01076_b200.gates import GateKind as K, gate, gate_array
    q = int(args.child)
    gs = gate_array([gate(K.Ry, q, -1, 0.3)])
    st = StateVector(args.n)
    st.set_timing(True)
    best = 1e9
    for _ in range(args.reps):
        st.apply(gs)
        st.sync()
        ms = sum(t[1] for t in st.last_timings())
        best = min(best, ms)
    gbs = 32.0 * 2 ** args.n / (best * 1e-3) / 1e9
    print(json.dumps({"q": q, "ms": round(best, 3), "gbs": round(gbs, 1)}))
    sys.exit(0)

cfgs = [
    {}, {"QTB_LOW_BITS": "3"}, {"QTB_TILE_BITS": "12", "QTB_LOW_BITS": "3"},
    {"QTB_TILE_BITS": "12", "QTB_LOW_BITS": "4"}, {"QTB_TILE_BITS": "12", "QTB_LOW_BITS": "6"},
    {"QTB_TILE_BITS": "12", "QTB_LOW_BITS": "3", "QTB_REG_BITS": "4"},
    {"QTB_TILE_BITS": "11", "QTB_LOW_BITS": "3", "QTB_PIPE": "1"},
]
for jit in ("0", "1"):
    for c in cfgs:
        for q in (20, 29):
            env = dict(os.environ, QTB_JIT=jit, **c)
            out = subprocess.run([sys.executable, __file__, "--n", str(args.n), "--reps",
                                  str(args.reps), "--child", str(q)], env=env,
                                 capture_output=True, text=True, timeout=600)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"jit={jit} {c} {line}", flush=True)
