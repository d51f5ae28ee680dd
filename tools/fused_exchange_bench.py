"""Fused exchange vs the send/recv path on one GPU: BASELINE config 4's circuit
family on an in-process group of emulated ranks (compiled mode), warm second
apply (plans and kernels cached). python tools/fused_exchange_bench.py [--n 30] [--world 8]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_01076_b200 import RankGroup, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--world", type=int, default=8)
args = ap.parse_args()
w = W.config4(n=args.n)
for fuse in ("1", "0"):
    os.environ["QTB_FUSE_EXCHANGE"] = fuse
    g = RankGroup(w.n, args.world, compiled=True)
    times = []
    for rep in range(3):
        g.set_basis(0)
        g.run(lambda st: st.sync())
        t0 = time.perf_counter()
        g.apply(w.gates)
        g.run(lambda st: st.sync())
        times.append(time.perf_counter() - t0)
    st = g.stats()[0]
    nrm = g.norm_squared()
    g.close()
    print(json.dumps({"n": w.n, "world": args.world, "fused": fuse == "1", "apply_s": [round(t, 4) for t in times],
                      "passes": st["passes"], "swaps": st["swaps"], "fused_exchanges": st["fused_exchanges"],
                      "sent_bytes_per_rank": st["exchanged_bytes"],
                      "local_copy_bytes_per_rank": st["exchange_local_bytes"], "norm_error": abs(nrm - 1)}), flush=True)
