"""OpenQASM 2.0 front end -- the reference's ``qtask::qasm`` (qasm.hpp:11-66,
qasm.cpp:34-426) for Python callers.

Parsing runs in the library (``qt_qasm_parse``, implemented by the C++
drop-in header ``include/qtask/qasm.hpp``), so Python and C++ callers share
one parser; ``levelize`` / ``to_qasm`` / ``build_circuit`` are restated here
over the parsed statements (the reference's test suite builds programs by
hand and levelizes them, so they must work on any ``QasmProgram``).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import _ffi
from .errors import Error
from .gates import GateKind as K


class ParseError(Error):
    """qtask::qasm::ParseError: malformed input at (line, column)."""

    def __init__(self, message: str, line: int, column: int):
        super().__init__(message)
        self.line = line
        self.column = column


class UnsupportedGateError(Error):
    """qtask::qasm::UnsupportedGateError: a statement outside the subset."""

    def __init__(self, message: str, line: int, column: int):
        super().__init__(message)
        self.line = line
        self.column = column


GATE = 0
BARRIER = 1
_ROTATIONS = (K.Rx, K.Ry, K.Rz)
_WORDS = {K.Cnot: "cx", K.X: "x", K.Y: "y", K.Z: "z", K.H: "h", K.S: "s", K.Sdg: "sdg",
          K.T: "t", K.Tdg: "tdg", K.Rx: "rx", K.Ry: "ry", K.Rz: "rz", K.Swap: "swap"}


@dataclass
class Statement:
    kind: int = GATE
    gate: K = K.X
    theta: float = 0.0
    has_theta: bool = False
    qubits: list = field(default_factory=list)  # cx: control, target; swap: target, control
    line: int = 0
    column: int = 0


@dataclass
class QasmProgram:
    num_qubits: int = 0
    qreg_name: str = "q"
    statements: list = field(default_factory=list)


class _Stmt(ctypes.Structure):  # qt_qasm_stmt (include/qtask_c.h)
    _fields_ = [("kind", ctypes.c_int32), ("gate", ctypes.c_int32), ("theta", ctypes.c_double),
                ("has_theta", ctypes.c_int32), ("nqubits", ctypes.c_int32),
                ("qubits", ctypes.c_int32 * 2), ("line", ctypes.c_int32),
                ("column", ctypes.c_int32), ("level", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


def _raise(rc: int, line: ctypes.c_int, col: ctypes.c_int):
    msg = _ffi.lib().qt_last_error().decode("utf-8", "replace")
    if rc == -10:
        raise ParseError(msg, line.value, col.value)
    if rc == -11:
        raise UnsupportedGateError(msg, line.value, col.value)
    _ffi.check(rc)


def parse(text: str) -> QasmProgram:
    """Parses OpenQASM 2.0 text (the reference's subset)."""
    data = text.encode("utf-8")
    n = ctypes.c_size_t(0)
    nq = ctypes.c_uint32(0)
    line, col = ctypes.c_int(0), ctypes.c_int(0)
    L = _ffi.lib()
    rc = L.qt_qasm_parse(data, len(data), None, 0, ctypes.byref(n), ctypes.byref(nq),
                         ctypes.byref(line), ctypes.byref(col))
    if rc < 0:
        _raise(rc, line, col)
    buf = (_Stmt * max(1, n.value))()
    rc = L.qt_qasm_parse(data, len(data), buf, n.value, ctypes.byref(n), ctypes.byref(nq),
                         ctypes.byref(line), ctypes.byref(col))
    if rc < 0:
        _raise(rc, line, col)
    prog = QasmProgram(num_qubits=nq.value, qreg_name=_qreg_name(text))
    for r in buf[:n.value]:
        prog.statements.append(Statement(
            kind=r.kind, gate=K(r.gate), theta=r.theta, has_theta=bool(r.has_theta),
            qubits=[r.qubits[i] for i in range(r.nqubits)], line=r.line, column=r.column))
    return prog


def _qreg_name(text: str) -> str:
    import re
    m = re.search(r"\bqreg\s+([A-Za-z_][A-Za-z0-9_]*)\s*\[", text)
    return m.group(1) if m else "q"


def to_qasm(prog: QasmProgram) -> str:
    """Regenerates QASM text, statement order preserved (17 significant digits)."""
    out = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg {prog.qreg_name}[{prog.num_qubits}];"]
    for st in prog.statements:
        if st.kind == BARRIER:
            out.append(f"barrier {prog.qreg_name};")
            continue
        par = f"({st.theta:.17g})" if st.has_theta else ""
        ops = ",".join(f"{prog.qreg_name}[{q}]" for q in st.qubits)
        out.append(f"{_WORDS[K(st.gate)]}{par} {ops};")
    return "\n".join(out) + "\n"


def levelize(prog: QasmProgram):
    """ASAP levels (qasm.cpp:376-405): one past the deepest earlier gate on any
    of the statement's qubits; a barrier moves later gates past every level."""
    depth = [-1] * prog.num_qubits
    levels, floor_level, deepest = [], 0, -1
    for i, st in enumerate(prog.statements):
        if st.kind == BARRIER:
            floor_level = deepest + 1
            continue
        lv = max([floor_level] + [depth[q] + 1 for q in st.qubits])
        for q in st.qubits:
            depth[q] = lv
        deepest = max(deepest, lv)
        while len(levels) <= lv:
            levels.append([])
        levels[lv].append(i)
    return levels


def build_circuit(sim, prog: QasmProgram) -> None:
    """One net per level appended to ``sim`` (qasm.cpp:407-426)."""
    for level in levelize(prog):
        net = sim.insert_net_back()
        for i in level:
            st = prog.statements[i]
            g = K(st.gate)
            if g == K.Cnot:
                sim.insert_gate(K.Cnot, net, st.qubits[1], st.qubits[0])
            elif g == K.Swap:
                sim.insert_gate(K.Swap, net, st.qubits[0], st.qubits[1])
            elif st.has_theta:
                sim.insert_gate(g, st.theta, net, st.qubits[0])
            else:
                sim.insert_gate(g, net, st.qubits[0])


def build_text(sim, text: str) -> None:
    """parse + build_circuit in the library (``qt_qasm_build``) on a Simulator."""
    data = text.encode("utf-8")
    line, col = ctypes.c_int(0), ctypes.c_int(0)
    rc = _ffi.lib().qt_qasm_build(sim._h, data, len(data), ctypes.byref(line), ctypes.byref(col))
    if rc < 0:
        _raise(rc, line, col)
