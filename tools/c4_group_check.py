"""BASELINE config 4 at full size (33 qubits, 128 GiB) through the sharded
code path on ONE B200: an in-process group of 2 / 4 / 8 emulated ranks
(RankGroup: per-rank kernels with rank offsets, State::exchange's step loop,
two-buffer exchanges where a second shard fits) vs the same circuit on one
unsharded 128 GiB state. Compares the norm and the first 2^22 amplitudes
(bitwise and max |diff|), and reports exchange statistics.

  python tools/c4_group_check.py [--worlds 2 4 8] [--n 33]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_01076_b200 import RankGroup, StateVector, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=33)
ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--compiled", type=int, default=0)
ap.add_argument("--sample-bits", type=int, default=22)
args = ap.parse_args()
w = W.config4(n=args.n)
S = 1 << args.sample_bits

st = StateVector(w.n, compiled=bool(args.compiled))
st.apply(w.gates)
st.sync()
t0 = time.perf_counter()
st.set_basis(0)
st.apply(w.gates)
st.sync()
single_s = time.perf_counter() - t0
ref_norm = st.norm_squared()
ref = st.read(0, S)
st.close()
print(json.dumps({"n": w.n, "mode": "single", "apply_s": round(single_s, 3), "norm": ref_norm}), flush=True)

for world in args.worlds:
    g = RankGroup(w.n, world, compiled=bool(args.compiled))
    for r in g.ranks:
        r.set_timing(True)
    t0 = time.perf_counter()
    g.apply(w.gates)
    g.run(lambda s: s.sync())
    apply_s = time.perf_counter() - t0
    tim = g.run(lambda s: s.last_timings())
    stats = g.stats()
    nrm = g.norm_squared()
    got = g.read(0, S)
    g.close()
    ex_ms = max(sum(ms for k, ms in t if k == 1) for t in tim)
    print(json.dumps({
        "n": w.n, "mode": f"group{world}", "apply_s": round(apply_s, 3), "norm": nrm,
        "norm_diff_vs_single": abs(nrm - ref_norm),
        "sample_max_abs_diff": float(np.abs(got - ref).max()),
        "sample_bitwise_equal": bool(np.array_equal(got, ref)),
        "swaps": stats[0]["swaps"], "sent_bytes_per_rank": stats[0]["exchanged_bytes"],
        "local_copy_bytes_per_rank": stats[0]["exchange_local_bytes"],
        "exchange_device_ms_max_rank": round(ex_ms, 2),
        "note": "emulated ranks share one GPU: exchanges are device copies, so exchange "
                "time is HBM-bound here, not NVLink"}), flush=True)
