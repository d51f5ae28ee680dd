"""HBM streaming efficiency of one compiled pass vs the tile's bit set: RY
on each qubit of a set (one pass, 1-2 rounds) over a 2^n state; prints the
pass time and the algorithmic GB/s (32 B per amplitude).

  python tools/tilebits_bench.py [--n 30]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_01076_b200 import StateVector  # noqa: E402
from paper_2210_01076_b200.gates import GateKind as K, gate, gate_array  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
SETS = {
    "contig4-11": [4, 5, 6, 7, 8, 9, 10, 11],
    "pass11": [6, 8, 10, 12, 13, 16, 26, 28],
    "pass16": [5, 7, 11, 14, 16, 18, 20, 21],
    "pass19": [13, 16, 18, 20, 21, 24, 26, 28],
    "high22-29": [22, 23, 24, 25, 26, 27, 28, 29],
    "odd5-19": [5, 7, 9, 11, 13, 15, 17, 19],
    "even4-18": [4, 6, 8, 10, 12, 14, 16, 18],
    "mid12-19": [12, 13, 14, 15, 16, 17, 18, 19],
}
st = StateVector(args.n, compiled=True)
st.set_timing(True)
for name, qs in SETS.items():
    gs = gate_array([gate(K.Ry, q, -1, 0.3 + 0.1 * q) for q in qs])
    best = 1e9
    for _ in range(args.reps):
        st.apply(gs)
        st.sync()
        t = st.last_timings()
        best = min(best, sum(x[1] for x in t))
    print(json.dumps({"set": name, "qubits": qs, "passes": len(t), "ms": round(best, 3),
                      "gbs": round(32.0 * 2 ** args.n / (best * 1e-3) / 1e9, 1)}), flush=True)
