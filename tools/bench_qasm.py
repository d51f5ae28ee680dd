"""OpenQASM front end measurement: parse + levelize
throughput of ours (library qt_qasm_parse, C++ header qtask/qasm.hpp) vs the
reference parser (oracle/_ref: qasm.cpp compiled from its sources) on the same
synthetic program, and (with a GPU) QASM text -> state through the Simulator
API vs the reference engine. Prints one JSON object.

  python tools/bench_qasm.py [--statements 200000] [--e2e-qubits 16]
"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (the reference side of the comparison)
from paper_2210_01076_b200 import _ffi, qasm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--statements", type=int, default=200000)
ap.add_argument("--qubits", type=int, default=30)
ap.add_argument("--e2e-qubits", type=int, default=16)
ap.add_argument("--e2e-statements", type=int, default=400)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()


def program(rng, n, count):
    words = ["h", "x", "y", "z", "s", "sdg", "t", "tdg"]
    out = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{n}];"]
    for i in range(count):
        r = rng.random()
        if r < 0.3 and n > 1:
            a, b = rng.choice(n, 2, replace=False)
            out.append(f"cx q[{a}],q[{b}];")
        elif r < 0.6:
            out.append(f"r{'xyz'[int(rng.integers(3))]}({rng.uniform(-6.3, 6.3):.15g}) "
                       f"q[{int(rng.integers(n))}];")
        elif r < 0.61:
            out.append("barrier q;")
        else:
            out.append(f"{words[int(rng.integers(8))]} q[{int(rng.integers(n))}];")
    return "\n".join(out) + "\n"


def best(fn):
    t = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return min(t)


rng = np.random.default_rng(8)
text = program(rng, args.qubits, args.statements).encode()
L = _ffi.lib()
cnt, nq = ctypes.c_size_t(0), ctypes.c_uint32(0)
el, ec = ctypes.c_int(0), ctypes.c_int(0)
buf = (qasm._Stmt * (args.statements + 1))()


def ours_parse():
    rc = L.qt_qasm_parse(text, len(text), buf, len(buf), ctypes.byref(cnt), ctypes.byref(nq),
                         ctypes.byref(el), ctypes.byref(ec))
    assert rc == 0


res = {"statements": args.statements, "qubits": args.qubits, "bytes": len(text)}
t_ours = best(ours_parse)
res["ours_parse_levelize_s"] = t_ours
res["ours_statements_per_s"] = args.statements / t_ours
if oracle.ref_available():
    lib = oracle.ref_lib()
    rows = np.zeros((args.statements + 1, 8))
    lv = np.zeros(args.statements + 1, dtype=np.int32)

    def ref_parse():
        n = lib.ref_qasm_parse(text, len(text), rows.ctypes.data, lv.ctypes.data, len(lv),
                               ctypes.byref(nq), ctypes.byref(el), ctypes.byref(ec))
        assert n == args.statements

    t_ref = best(ref_parse)
    res["reference_parse_levelize_s"] = t_ref
    res["reference_statements_per_s"] = args.statements / t_ref
    res["speedup"] = t_ref / t_ours

if _ffi.device_count() > 0:
    from paper_2210_01076_b200 import Config, Simulator
    small = program(np.random.default_rng(9), args.e2e_qubits, args.e2e_statements)
    e2e = {"qubits": args.e2e_qubits, "statements": args.e2e_statements}

    def ours_e2e():
        sim = Simulator(args.e2e_qubits, Config())
        qasm.build_text(sim, small)
        sim.update_state()
        e2e["ours_norm"] = sim.norm_squared()
        sim.close()

    ours_e2e()
    e2e["ours_text_to_state_s"] = best(ours_e2e)
    if oracle.ref_available():
        def ref_e2e():
            r = oracle.RefSimulator(args.e2e_qubits, 256, 0)
            r.qasm_build(small)
            r.update_state()
            e2e["reference_norm"] = r.norm_squared()
            r.close()

        e2e["reference_text_to_state_s"] = best(ref_e2e)
        e2e["reference_threads"] = os.cpu_count()
    res["text_to_state"] = e2e
print(json.dumps(res))
