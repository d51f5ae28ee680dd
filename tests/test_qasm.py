"""OpenQASM 2.0 front end: the reference's qtask::qasm
(qasm.hpp:11-66, qasm.cpp:34-426) -- parser, ASAP levelling, build_circuit.

CPU: known-answer cases restated from the reference's test strategy
(test_qasm.cpp) and a differential fuzz against the reference parser itself
(oracle/_ref, compiled from its sources): identical statements, levels and
error class / line / column on valid and corrupted programs.
GPU: build_circuit + update_state against the reference engine's amplitudes.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import qasm
from paper_2210_01076_b200.gates import GateKind as K

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")

HDR = "OPENQASM 2.0;\n"


def test_two_qubit_program():
    p = qasm.parse(HDR + "qreg r[3];\nh r[2];\ncx r[2],r[0];\n")
    assert p.num_qubits == 3 and p.qreg_name == "r"
    assert [s.gate for s in p.statements] == [K.H, K.Cnot]
    assert p.statements[1].qubits == [2, 0]  # control first


def test_tolerated_lines():
    p = qasm.parse("// a comment line\n" + HDR + 'include "qelib1.inc";\n'
                   "qreg q[4];\ncreg m[4];\n\ny q[3];   // comment after a statement\n")
    assert p.num_qubits == 4 and len(p.statements) == 1 and p.statements[0].gate == K.Y


@pytest.mark.parametrize("expr,val", [("pi", math.pi), ("-pi/4", -math.pi / 4),
                                      ("3*pi/2", 3 * math.pi / 2), ("0.125", 0.125),
                                      ("-2.5e-1", -0.25), ("pi*pi", math.pi * math.pi)])
def test_angle_expressions(expr, val):
    p = qasm.parse(HDR + f"qreg q[1];\nrz({expr}) q[0];\n")
    assert p.statements[0].has_theta and p.statements[0].theta == pytest.approx(val, abs=0)


@pytest.mark.parametrize("body", ["creg c[1];\nmeasure q[0] -> c[0];\n", "ccx q[0],q[1],q[2];\n",
                                  "u1(0.5) q[0];\n", "id q[1];\n", "cz q[0],q[1];\n",
                                  "reset q[0];\n"])
def test_unsupported_statements(body):
    with pytest.raises(qasm.UnsupportedGateError):
        qasm.parse(HDR + "qreg q[3];\n" + body)


@pytest.mark.parametrize("src,line", [
    (HDR + "qreg q[2];\nx q[2];\n", 3),                 # index out of range
    (HDR + "qreg q[2];\nx q;\n", 3),                    # whole register
    ("OPENQASM 3.0;\nqreg q[2];\n", 1),                 # version
    (HDR + "qreg q[2];\nqreg p[2];\n", 3),              # second qreg
    (HDR + "qreg q[2];\nswap q[1],q[1];\n", 3),         # repeated operand
    (HDR + "qreg q[2];\nh q[0]\nh q[1];\n", 4),         # missing ';'
    (HDR + "qreg q[2];\nrx q[0];\n", 3),                # missing angle
    (HDR + "qreg q[2];\nh(0.1) q[0];\n", 3),            # parameter on a fixed gate
    (HDR + "qreg q[2];\ncx q[0];\n", 3),                # operand count
    (HDR + "h q[0];\n", 2),                             # gate before qreg
])
def test_parse_errors_locate_the_token(src, line):
    with pytest.raises(qasm.ParseError) as e:
        qasm.parse(src)
    assert e.value.line == line


def test_asap_levels_and_barriers():
    p = qasm.parse(HDR + "qreg q[4];\nh q[0]; h q[1]; h q[2]; h q[3];\n"
                   "cx q[0],q[1];\ncx q[2],q[3];\ncx q[1],q[2];\n")
    assert [len(lv) for lv in qasm.levelize(p)] == [4, 2, 1]
    p = qasm.parse(HDR + "qreg q[3];\nx q[0];\nbarrier q;\nx q[1];\nbarrier q[0],q[2];\nx q[2];\n")
    assert qasm.levelize(p) == [[0], [2], [4]]


def test_round_trip():
    src = (HDR + "qreg q[3];\nh q[0];\ncx q[0],q[1];\nry(0.3) q[2];\nbarrier q;\n"
           "swap q[0],q[2];\nrz(-pi/3) q[1];\n")
    a = qasm.parse(src)
    b = qasm.parse(qasm.to_qasm(a))
    assert [(s.kind, s.gate, s.qubits, s.theta) for s in a.statements] == \
           [(s.kind, s.gate, s.qubits, s.theta) for s in b.statements]


# ---- differential fuzz against the reference parser --------------------------

_GATES1 = ["h", "x", "y", "z", "s", "sdg", "t", "tdg"]
_ROT = ["rx", "ry", "rz"]
_ANGLES = ["pi", "-pi/2", "0.25", "1e-3", "2*pi/3", "-3.5e+2", ".5", "pi*2/4", "7", "-0",
           "1.5E2", "pi/8*3"]
_JUNK = list(";[](),qx1 \n/-*.e\"") + ["measure", "ccx", "pi", "//", "qreg", "barrier"]


def random_program(rng):
    """A VALID program (errors only come from `corrupt`)."""
    n = int(rng.integers(1, 9))
    one_line = rng.random() < 0.2  # then no // comments (they would end the program)
    out = []
    if rng.random() < 0.3 and not one_line:
        out.append("// generated")
    out.append("OPENQASM 2.0;")
    if rng.random() < 0.5:
        out.append('include "qelib1.inc";')
    out.append(f"qreg q[{n}];")
    if rng.random() < 0.3:
        out.append(f"creg c[{n}];")
    for _ in range(int(rng.integers(0, 25))):
        r = rng.random()
        if r < 0.08:
            out.append("barrier q;" if rng.random() < 0.5 else f"barrier q[{int(rng.integers(n))}];")
        elif r < 0.35 and n >= 2:
            a, b = rng.choice(n, 2, replace=False)
            out.append(f"{'cx' if rng.random() < 0.7 else 'swap'} q[{a}],q[{b}];")
        elif r < 0.6:
            out.append(f"{_ROT[int(rng.integers(3))]}({_ANGLES[int(rng.integers(len(_ANGLES)))]}) "
                       f"q[{int(rng.integers(n))}];")
        else:
            out.append(f"{_GATES1[int(rng.integers(len(_GATES1)))]} q[{int(rng.integers(n))}];")
        if rng.random() < 0.1 and not one_line:
            out[-1] += "  // note"
    return (" " if one_line else "\n").join(out) + "\n"


def corrupt(rng, text):
    for _ in range(int(rng.integers(1, 3))):
        i = int(rng.integers(0, len(text) + 1))
        op = rng.random()
        if op < 0.4 and text:
            text = text[:i] + text[i + 1:]
        elif op < 0.8:
            text = text[:i] + _JUNK[int(rng.integers(len(_JUNK)))] + text[i:]
        else:
            text = text.replace("q[", "q[1", 1) if rng.random() < 0.5 else text.replace("h ", "u1 ", 1)
    return text


def ours(text):
    try:
        p = qasm.parse(text)
    except qasm.ParseError as e:
        return ("parse", e.line, e.column)
    except qasm.UnsupportedGateError as e:
        return ("unsupported", e.line, e.column)
    return ("ok", p)


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_parser_matches_reference(seed):
    rng = np.random.default_rng(1000 + seed)
    checked = {"ok": 0, "parse": 0, "unsupported": 0}
    for trial in range(300):
        text = random_program(rng)
        if trial % 2:
            text = corrupt(rng, text)
        want = oracle.ref_qasm_parse(text)
        got = ours(text)
        assert got[0] == want[0], (text, got, want)
        checked[want[0]] += 1
        if want[0] != "ok":
            assert got[1:] == want[1:], (text, got, want)
            continue
        p = got[1]
        _, nq, rows, levels = want
        assert p.num_qubits == nq and len(p.statements) == len(rows)
        for st, r in zip(p.statements, rows):
            assert st.kind == int(r[0])
            if st.kind == qasm.GATE:
                assert int(st.gate) == int(r[1]) and st.has_theta == bool(r[3])
                assert st.theta == r[2]  # same strtod, same operation order: exact
                assert st.qubits == [int(x) for x in r[4:6] if x >= 0]
            assert (st.line, st.column) == (int(r[6]), int(r[7]))
        lv = np.full(len(p.statements), -1)
        for k, idx in enumerate(qasm.levelize(p)):
            lv[idx] = k
        assert (lv == levels).all()
    assert min(checked.values()) > 0, checked


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_build_circuit_matches_reference_engine(gpu, seed):
    """Same QASM text -> reference parse + build_circuit + update_state
    (engine.cpp) vs ours (both the Python build_circuit and the library's
    qt_qasm_build): amplitudes within 1e-10, nets one per ASAP level."""
    from paper_2210_01076_b200 import Config, Simulator
    rng = np.random.default_rng(2000 + seed)
    for _ in range(5):
        text = random_program(rng)
        p = qasm.parse(text)
        ref = oracle.RefSimulator(p.num_qubits, 16, 1)
        ref.qasm_build(text)
        ref.update_state()
        want = ref.amplitudes()
        ref.close()
        for use_lib in (False, True):
            sim = Simulator(p.num_qubits, Config())
            if use_lib:
                qasm.build_text(sim, text)
            else:
                qasm.build_circuit(sim, p)
            assert len(sim.circuit().net_order()) == len(qasm.levelize(p))
            sim.update_state()
            got = sim.amplitudes(0, (1 << p.num_qubits) - 1)
            sim.close()
            assert np.abs(got - want).max() < 1e-10
