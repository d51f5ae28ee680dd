"""Incremental-update latency of the GPU engine (bench.measure_incremental):
C1 (16 q, 400 gates, 20 modifiers) and C5 (28 q, 5000 gates, --mods
alternating insert / remove, uniform / last-10% positions).
  python tools/inc_latency.py [--mods 16] [--skip-c1] [--skip-c5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import measure_incremental  # noqa: E402
from paper_2210_01076_b200 import Config, Simulator, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mods", type=int, default=16)
ap.add_argument("--skip-c1", action="store_true")
ap.add_argument("--skip-c5", action="store_true")
args = ap.parse_args()
if not args.skip_c1:
    w1 = W.config1()
    r = measure_incremental(lambda n: Simulator(n, Config()), w1, 20, tail_split=False)
    print(json.dumps({"c1": r}), flush=True)
if not args.skip_c5:
    w5 = W.config5(nmods=max(2, args.mods))
    r = measure_incremental(lambda n: Simulator(n, Config()), w5, args.mods)
    print(json.dumps({"c5": r}), flush=True)
