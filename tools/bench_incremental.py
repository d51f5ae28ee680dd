"""The paper's incremental-iteration benchmark (PAPER.md "Performance of
Incremental Simulation"; the reference harness tools/qtask_cli.cpp:365-502)
through paper_2210_01076_b200.trace.run_iterations: a QASM program's ASAP
levels inserted (insert-sweep) / removed (remove-sweep) / both (mix) a few
levels per iteration, one update_state each. The B200 engine vs the reference
engine (oracle/_ref, all host threads) on the same level plan and RNG seed.
QASMBench is not available: a decomposed QFT and a random layered circuit
(QASM text generated here) stand in. Prints one JSON object.

  python tools/bench_incremental.py [--qubits 16] [--per-iter 4] [--iters 30]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (the reference arm)
from paper_2210_01076_b200 import Config, Simulator, qasm, trace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qubits", type=int, default=16)
ap.add_argument("--per-iter", type=int, default=4)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--no-reference", action="store_true")
args = ap.parse_args()


def qft_text(n):
    out = ["OPENQASM 2.0;", f"qreg q[{n}];"]
    for j in range(n - 1, -1, -1):
        out.append(f"h q[{j}];")
        for k in range(j - 1, -1, -1):
            lam = math.pi / 2 ** (j - k)
            out += [f"rz({lam / 2!r}) q[{k}];", f"cx q[{k}],q[{j}];",
                    f"rz({-lam / 2!r}) q[{j}];", f"cx q[{k}],q[{j}];", f"rz({lam / 2!r}) q[{j}];"]
    for i in range(n // 2):
        out.append(f"swap q[{i}],q[{n - 1 - i}];")
    return "\n".join(out) + "\n"


def layered_text(n, layers, seed=4):
    rng = np.random.default_rng(seed)
    out = ["OPENQASM 2.0;", f"qreg q[{n}];"]
    for lv in range(layers):
        for q in range(n):
            out.append(f"r{'xyz'[int(rng.integers(3))]}({rng.uniform(-3.1, 3.1):.12f}) q[{q}];")
        for a in range(lv % 2, n - 1, 2):
            out.append(f"cx q[{a}],q[{a + 1}];")
    return "\n".join(out) + "\n"


def ref_insert(s, kind, theta, net, target, control):
    return s.insert_gate(int(kind), net, target, control, 0.0 if theta is None else theta)


res = {"qubits": args.qubits, "per_iter": args.per_iter, "iters": args.iters,
       "reference_threads": os.cpu_count(), "circuits": {}}
for name, text in (("qft", qft_text(args.qubits)), ("layered", layered_text(args.qubits, 24))):
    plan = trace.level_plan(qasm.parse(text))
    entry = {"levels": len(plan), "gates": sum(len(lv) for lv in plan)}
    for mode in ("insert-sweep", "remove-sweep", "mix"):
        finals = {}
        row = {}
        arms = [("b200", lambda q: Simulator(q, Config()), None)]
        if not args.no_reference and oracle.ref_available():
            arms.append(("reference", lambda q: oracle.RefSimulator(q, 256, 0), ref_insert))
        for arm, make, ins in arms:
            def fin(sim, arm=arm):
                n = args.qubits
                finals[arm] = (sim.amplitudes(0, (1 << n) - 1) if arm == "b200"
                               else sim.amplitudes())
            rows, _ = trace.run_iterations(make, args.qubits, plan, mode, seed=11,
                                           per_iter=args.per_iter, iters=args.iters,
                                           insert_gate=ins, finish=fin)
            ms = [r["wall_time_ms"] for r in rows]
            row[arm] = {"iterations": len(rows), "cumulative_ms": float(np.sum(ms)),
                        "mean_ms": float(np.mean(ms)), "median_ms": float(np.median(ms))}
        if "reference" in finals:
            row["max_abs_diff_final_state"] = float(np.abs(finals["b200"] - finals["reference"]).max())
            row["speedup_cumulative"] = row["reference"]["cumulative_ms"] / row["b200"]["cumulative_ms"]
        entry[mode] = row
    res["circuits"][name] = entry
print(json.dumps(res))
