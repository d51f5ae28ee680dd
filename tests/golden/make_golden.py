"""Generates the golden fixtures in tests/golden/ by running the REFERENCE
(oracle/_ref/libqtask_ref.so = /root/reference/proj/src compiled from its
own sources) in this container. The GPU box has no /root/reference, so the
outputs are committed as small .npz files; this script is how they were made.

  python tests/golden/make_golden.py

* golden_random.npz      -- 40 random circuits (all 13 reference kinds, n<=10)
                            and the reference dense oracle's final states
                            (oracle.cpp:15-50).
* golden_incremental.npz -- 24 random modifier logs replayed through the
                            reference qtask::Simulator (engine.cpp), with the
                            amplitudes after every update_state.
* golden_traces.npz      -- the reference's Listing-1 / entangle5 edit and an
                            8-qubit interleaved construction/removal sequence,
                            restated as modifier logs, with reference states.
* golden_fixture_traces.npz -- the reference's own trace fixtures
                            (proj/tests/data/entangle5.trace, mixed8.trace)
                            parsed by paper_2210_01076_b200.trace and replayed
                            on the reference engine: parsed statements (as
                            arrays) and the amplitudes after every update.

  python tests/golden/make_golden.py [random incremental traces fixture_traces]
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

KINDS = list(range(13))  # reference GateKind order
TWO = {0, 12}
ROT = {9, 10, 11}


def rand_gate(rng, n):
    k = int(rng.integers(13 if n >= 2 else 12))
    if n < 2 and k in TWO:
        k = 4
    t = int(rng.integers(n))
    c = -1
    if k in TWO:
        c = t
        while c == t:
            c = int(rng.integers(n))
    th = 0.0
    if k in ROT:
        th = [math.pi, math.pi / 2, 0.0, float(rng.uniform(-2 * math.pi, 2 * math.pi))][
            int(rng.integers(4))]
    return k, t, c, th


def gates_array(rows):
    g = np.zeros(len(rows), dtype=oracle.GATE_DTYPE)
    for i, (k, t, c, th) in enumerate(rows):
        g[i] = (k, t, c, 0, th, 0.0, 0.0)
    return g


def make_random():
    rng = np.random.default_rng(7771)
    ns, offs, all_gates, states, soffs = [], [0], [], [], [0]
    for _ in range(40):
        n = int(rng.integers(1, 11))
        rows = [rand_gate(rng, n) for _ in range(int(rng.integers(1, 80)))]
        g = gates_array(rows)
        st, _ = oracle.ref_simulate(n, g)
        ns.append(n)
        all_gates.append(g)
        offs.append(offs[-1] + len(g))
        states.append(st)
        soffs.append(soffs[-1] + len(st))
    np.savez_compressed(os.path.join(HERE, "golden_random.npz"), n=np.array(ns),
                        gate_offsets=np.array(offs), gates=np.concatenate(all_gates),
                        state_offsets=np.array(soffs), states=np.concatenate(states))


class Log:
    """Modifier log: list of [op, args...] replayable on either engine."""

    def __init__(self, sim, n):
        self.sim, self.n, self.ops, self.states = sim, n, [], []
        self.nets, self.gates = [], []

    def net_back(self):
        self.nets.append(self.sim.insert_net_back())
        self.ops.append(["net_back"])

    def net_after(self, i):
        self.nets.append(self.sim.insert_net_after(self.nets[i]))
        self.ops.append(["net_after", i])

    def gate(self, i, k, t, c, th):
        try:
            gid = self.sim.insert_gate(k, self.nets[i], t, c, th)
        except RuntimeError:
            return  # net conflict (reference NetConflictError): not logged
        self.gates.append(gid)
        self.ops.append(["gate", i, k, t, c, th])

    def remove_gate(self, j):
        self.sim.remove_gate(self.gates.pop(j))
        self.ops.append(["remove_gate", j])

    def remove_net(self, i):
        self.sim.remove_net(self.nets.pop(i))
        self.ops.append(["remove_net", i])

    def update(self):
        self.sim.update_state()
        self.states.append(self.sim.amplitudes())
        self.ops.append(["update", len(self.states) - 1])


def random_log(rng):
    n = int(rng.integers(1, 9))
    sim = oracle.RefSimulator(n, 1 << int(rng.integers(1, 7)), 1)
    lg = Log(sim, n)
    for _ in range(8 + int(rng.integers(30))):
        roll = int(rng.integers(12))
        if roll < 3 or not lg.nets:
            if not lg.nets or rng.integers(2) == 0:
                lg.net_back()
            else:
                lg.net_after(int(rng.integers(len(lg.nets))))
        elif roll < 9:
            lg.gate(int(rng.integers(len(lg.nets))), *rand_gate(rng, n))
        elif roll < 10 and lg.gates:
            lg.remove_gate(int(rng.integers(len(lg.gates))))
        else:
            lg.update()
    lg.update()
    sim.close()
    return lg


def save_logs(name, logs):
    meta = [{"n": lg.n, "ops": lg.ops} for lg in logs]
    states = [s for lg in logs for s in lg.states]
    lens = [len(s) for s in states]
    np.savez_compressed(os.path.join(HERE, name), meta=json.dumps(meta),
                        state_offsets=np.concatenate([[0], np.cumsum(lens)]),
                        states=np.concatenate(states))


def make_incremental():
    rng = np.random.default_rng(4242)
    save_logs("golden_incremental.npz", [random_log(rng) for _ in range(24)])


def make_traces():
    logs = []
    # Listing 1 (five qubits, Hadamard wall + four CNOTs), then replace the
    # third CNOT: CNOT(t=2, c=3) -> CNOT(t=1, c=2)  (entangle5)
    sim = oracle.RefSimulator(5, 4, 1)
    lg = Log(sim, 5)
    for _ in range(5):
        lg.net_back()
    for q in range(4, -1, -1):
        lg.gate(0, 4, q, -1, 0.0)
    lg.gate(1, 0, 3, 4, 0.0)
    lg.gate(2, 0, 1, 4, 0.0)
    lg.gate(3, 0, 2, 3, 0.0)
    lg.gate(4, 0, 0, 2, 0.0)
    lg.update()
    lg.remove_gate(7)
    lg.gate(3, 0, 1, 2, 0.0)
    lg.update()
    logs.append(lg)
    sim.close()
    # eight qubits: interleaved construction, removal and update
    sim = oracle.RefSimulator(8, 4, 2)
    lg = Log(sim, 8)
    lg.net_back()
    for q in range(3):
        lg.gate(0, 4, q, -1, 0.0)
    lg.update()
    lg.net_back()
    lg.gate(1, 0, 4, 0, 0.0)
    lg.gate(1, 0, 5, 1, 0.0)
    lg.update()
    lg.net_after(1)
    lg.gate(2, 11, 0, -1, math.pi / 4)
    lg.gate(2, 0, 6, 2, 0.0)
    lg.update()
    lg.remove_gate(4)
    lg.gate(1, 12, 5, 6, 0.0)
    lg.update()
    lg.remove_net(2)
    lg.update()
    lg.gate(0, 2, 3, -1, 0.0)
    lg.gate(0, 9, 7, -1, math.pi)
    lg.update()
    lg.net_back()
    lg.gate(2, 9, 4, -1, -math.pi / 2)
    lg.update()
    logs.append(lg)
    sim.close()
    save_logs("golden_traces.npz", logs)


def make_fixture_traces():
    from paper_2210_01076_b200 import trace
    from tests.test_trace import ref_insert, trace_to_arrays
    out = {}
    for name in ("entangle5", "mixed8"):
        path = os.path.join("/root/reference/proj/tests/data", name + ".trace")
        tr = trace.parse(open(path).read())
        states = []
        sim = oracle.RefSimulator(tr.num_qubits, 16, 1)
        trace.replay(sim, tr, verify=lambda s: states.append(s.amplitudes()) or 0.0,
                     insert_gate=ref_insert)
        sim.close()
        rows, ids = trace_to_arrays(tr)
        out[name] = np.stack(states)
        out[name + "_stmts"] = rows
        out[name + "_ids"] = ids
        out[name + "_n"] = np.array(tr.num_qubits)
    np.savez_compressed(os.path.join(HERE, "golden_fixture_traces.npz"), **out)


if __name__ == "__main__":
    oracle.build()
    which = sys.argv[1:] or ["random", "incremental", "traces", "fixture_traces"]
    if "random" in which:
        make_random()
    if "incremental" in which:
        make_incremental()
    if "traces" in which:
        make_traces()
    if "fixture_traces" in which:
        make_fixture_traces()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
