"""Modifier traces + incremental-iteration harness:
paper_2210_01076_b200/trace.py restating the reference's trace format and
bench protocol (tools/qtask_cli.cpp:118-502).

CPU: parser known answers / errors; the reference's own fixture traces
(read from /root/reference when present) replayed on the reference engine
must match the dense oracle and the committed goldens; the harness modes on
the reference engine match the dense oracle of the surviving circuit.
GPU: random traces and the harness on the B200 engine vs the reference engine
after every update; the fixture goldens replayed on the B200 engine.
"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import qasm, trace
from paper_2210_01076_b200.errors import Error
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = "/root/reference/proj/tests/data"


def ref_insert(s, kind, theta, net, target, control):
    return s.insert_gate(int(kind), net, target, control, 0.0 if theta is None else theta)


def test_parse_statements():
    tr = trace.parse("# comment\nqubits 3\nnet a\nnet b after a\nnet c front\n"
                     "gate g1 H a 0\ngate g2 RZ(pi/4) b 1\ngate g3 CNOT b 2 0\n"
                     "gate g4 RX(-pi) c 2\ngate g5 RY(0.25) c 1\nupdate\nremove_gate g3\n"
                     "remove_net c\nupdate\ndump /tmp/x.txt\n")
    assert tr.num_qubits == 3
    kinds = [s.kind for s in tr.stmts]
    assert kinds == ["net"] * 3 + ["gate"] * 5 + ["update", "remove_gate", "remove_net",
                                                   "update", "dump"]
    assert tr.stmts[1].anchor == "a" and tr.stmts[2].front
    g = tr.stmts[3:8]
    assert g[1].theta == math.pi / 4 and g[2].control == 0 and g[2].gate == K.Cnot
    assert g[3].theta == -math.pi and g[4].theta == 0.25 and g[0].control == -1


@pytest.mark.parametrize("text", ["net a\n", "qubits 0\n", "qubits 2\nfrob x\n",
                                  "qubits 2\nnet a\ngate g H a\n",
                                  "qubits 2\nnet a\ngate g RZ(pi/0) a 0\n",
                                  "qubits 2\nnet a\ngate g RZ(abc) a 0\n",
                                  "qubits 2\nnet a\ngate g U3 a 0\n", "qubits 2\nnet a sideways\n",
                                  "qubits 2\ndump\n"])
def test_parse_errors(text):
    with pytest.raises(Error):
        trace.parse(text)


def dense_of(view_gates, n):
    return oracle.simulate(n, view_gates)


def random_trace(rng, n, steps):
    """A random modifier trace in the wire format (reference gate kinds)."""
    lines = [f"qubits {n}"]
    nets, gates, nid, gid = [], {}, 0, 0
    kinds = ["H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "CNOT", "SWAP"]
    for _ in range(steps):
        r = rng.random()
        if r < 0.25 or not nets:
            nid += 1
            name = f"n{nid}"
            if nets and rng.random() < 0.5:
                lines.append(f"net {name} after {nets[int(rng.integers(len(nets)))]}")
            elif rng.random() < 0.2:
                lines.append(f"net {name} front")
            else:
                lines.append(f"net {name}")
            nets.append(name)
            gates[name] = set()
        elif r < 0.75:
            net = nets[int(rng.integers(len(nets)))]
            k = kinds[int(rng.integers(len(kinds) if n > 1 else 11))]
            free = [q for q in range(n) if all(q not in qs for qs in gates[net])]
            need = 2 if k in ("CNOT", "SWAP") else 1
            if len(free) < need:
                continue
            qs = [int(x) for x in rng.choice(free, need, replace=False)]
            gid += 1
            ang = ""
            if k in ("RX", "RY", "RZ"):
                ang = ["(pi/4)", "(-pi/2)", "(pi)", f"({rng.uniform(-3, 3):.6f})"][int(rng.integers(4))]
            lines.append(f"gate g{gid} {k}{ang} {net} " + " ".join(map(str, qs)))
            gates[net].add(tuple(qs))
        elif r < 0.85 and nets:
            victim = nets.pop(int(rng.integers(len(nets))))
            del gates[victim]
            lines.append(f"remove_net {victim}")
        else:
            lines.append("update")
    lines.append("update")
    return "\n".join(lines) + "\n"


@needs_ref
@pytest.mark.skipif(not os.path.isdir(FIXTURES), reason="reference fixtures not present")
@pytest.mark.parametrize("name", ["entangle5.trace", "mixed8.trace"])
def test_reference_fixture_traces_on_reference_engine(name):
    """The reference's own traces, parsed by trace.parse and replayed on the
    reference engine: every update matches the committed golden (made by
    tests/golden/make_golden.py from the same replay)."""
    tr = trace.parse(open(os.path.join(FIXTURES, name)).read())
    g = np.load(os.path.join(HERE, "golden", "golden_fixture_traces.npz"))
    sim = oracle.RefSimulator(tr.num_qubits, 16, 1)
    states = []
    trace.replay(sim, tr, verify=lambda s: states.append(s.amplitudes()) or 0.0,
                 insert_gate=ref_insert)
    sim.close()
    want = g[name.replace(".trace", "")]
    assert len(states) == len(want)
    for a, b in zip(states, want):
        assert np.abs(a - b).max() == 0.0


QFT_QASM = None


def qft_qasm(n):
    """A decomposed QFT as QASM text (H, CP via RZ/CX, final swaps)."""
    out = ["OPENQASM 2.0;", f"qreg q[{n}];"]
    for j in range(n - 1, -1, -1):
        out.append(f"h q[{j}];")
        for k in range(j - 1, -1, -1):
            lam = math.pi / 2 ** (j - k)
            out += [f"rz({lam / 2!r}) q[{k}];", f"cx q[{k}],q[{j}];", f"rz({-lam / 2!r}) q[{j}];",
                    f"cx q[{k}],q[{j}];", f"rz({lam / 2!r}) q[{j}];"]
    for i in range(n // 2):
        out.append(f"swap q[{i}],q[{n - 1 - i}];")
    return "\n".join(out) + "\n"


def present_gates(plan, present_levels):
    rows = []
    for lv in sorted(present_levels):
        for st in plan[lv]:
            g = K(st.gate)
            if g == K.Cnot:
                rows.append(gate(g, st.qubits[1], st.qubits[0]))
            elif g == K.Swap:
                rows.append(gate(g, st.qubits[0], st.qubits[1]))
            else:
                rows.append(gate(g, st.qubits[0], -1, st.theta))
    return gate_array(rows)


@needs_ref
@pytest.mark.parametrize("mode", ["insert-sweep", "remove-sweep", "mix"])
def test_harness_modes_on_reference_engine(mode):
    n = 6
    plan = trace.level_plan(qasm.parse(qft_qasm(n)))
    final = {}

    def finish(sim):
        final["amps"] = sim.amplitudes()
        return sim

    rows, _ = trace.run_iterations(lambda q: oracle.RefSimulator(q, 16, 1), n, plan, mode,
                                   seed=3, per_iter=3, iters=6, insert_gate=ref_insert,
                                   finish=finish)
    assert rows and all(r["wall_time_ms"] >= 0 for r in rows)
    assert "iteration,wall_time_ms" in trace.rows_csv(rows)
    if mode == "insert-sweep":  # everything inserted: the full QFT
        want = oracle.simulate(n, present_gates(plan, range(len(plan))))
        assert np.abs(final["amps"] - want).max() < 1e-12
    if mode == "remove-sweep":  # everything removed: |0...0>
        assert abs(final["amps"][0] - 1) < 1e-15


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_random_traces_match_reference_engine(gpu, seed):
    from paper_2210_01076_b200 import Config, Simulator
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(2, 9))
    tr = trace.parse(random_trace(rng, n, 80))
    ours, ref = [], []
    sim = Simulator(n, Config())
    trace.replay(sim, tr, verify=lambda s: ours.append(s.amplitudes(0, (1 << n) - 1)) or 0.0)
    sim.close()
    rs = oracle.RefSimulator(n, 16, 1)
    trace.replay(rs, tr, verify=lambda s: ref.append(s.amplitudes()) or 0.0, insert_gate=ref_insert)
    rs.close()
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        assert np.abs(a - b).max() < 1e-10


@pytest.mark.gpu
def test_fixture_goldens_on_b200(gpu):
    """The reference fixture traces (stored as parsed statements + the
    reference engine's amplitudes per update) replayed on the B200 engine."""
    from paper_2210_01076_b200 import Config, Simulator
    g = np.load(os.path.join(HERE, "golden", "golden_fixture_traces.npz"))
    for name in ("entangle5", "mixed8"):
        tr = trace_from_arrays(g[name + "_stmts"], g[name + "_ids"], int(g[name + "_n"]))
        got = []
        sim = Simulator(tr.num_qubits, Config())
        trace.replay(sim, tr, verify=lambda s: got.append(s.amplitudes(0, (1 << tr.num_qubits) - 1))
                     or 0.0)
        sim.close()
        want = g[name]
        assert len(got) == len(want)
        for a, b in zip(got, want):
            assert np.abs(a - b).max() < 1e-10


_KIND_CODE = {"net": 0, "gate": 1, "remove_gate": 2, "remove_net": 3, "update": 4}


def trace_to_arrays(tr):
    """Parsed statements as numbers: [kind, front, gate, has_theta, theta,
    target, control] + string ids [id, anchor, net] (dump lines dropped)."""
    rows, ids = [], []
    for s in tr.stmts:
        if s.kind not in _KIND_CODE:
            continue
        rows.append([_KIND_CODE[s.kind], int(s.front), int(s.gate), int(s.has_theta), s.theta,
                     s.target, s.control])
        ids.append([s.id, s.anchor, s.net])
    return np.array(rows, dtype=np.float64), np.array(ids, dtype="U32")


def trace_from_arrays(rows, ids, n):
    inv = {v: k for k, v in _KIND_CODE.items()}
    tr = trace.Trace(num_qubits=n)
    for r, (i, a, net) in zip(rows, ids):
        tr.stmts.append(trace.TraceStmt(kind=inv[int(r[0])], id=str(i), anchor=str(a),
                                        front=bool(r[1]), gate=K(int(r[2])),
                                        has_theta=bool(r[3]), theta=float(r[4]),
                                        net=str(net), target=int(r[5]), control=int(r[6])))
    return tr
