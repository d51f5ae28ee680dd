"""Gate kinds (reference GateKind order, gate.hpp:13-27) + additive U3 / CZ,
and helpers to build qt_gate arrays."""
from __future__ import annotations

import enum

import numpy as np

from ._ffi import GATE_DTYPE


class GateKind(enum.IntEnum):
    Cnot = 0
    X = 1
    Y = 2
    Z = 3
    H = 4
    S = 5
    Sdg = 6
    T = 7
    Tdg = 8
    Rx = 9
    Ry = 10
    Rz = 11
    Swap = 12
    U3 = 13  # additive: RZ(phi) RY(theta) RZ(lambda)
    Cz = 14  # additive: H CX H


TWO_QUBIT = {GateKind.Cnot, GateKind.Swap, GateKind.Cz}
ROTATION = {GateKind.Rx, GateKind.Ry, GateKind.Rz, GateKind.U3}


def is_two_qubit(kind) -> bool:
    return GateKind(kind) in TWO_QUBIT


def is_rotation(kind) -> bool:
    return GateKind(kind) in ROTATION


def gate(kind, target, control=-1, theta=0.0, phi=0.0, lam=0.0):
    return (int(kind), int(target), int(control), 0, float(theta), float(phi), float(lam))


def gate_array(rows) -> np.ndarray:
    """rows: iterable of gate(...) tuples -> qt_gate structured array."""
    rows = list(rows)
    arr = np.zeros(len(rows), dtype=GATE_DTYPE)
    for i, r in enumerate(rows):
        arr[i] = r
    return arr


def lower_to_reference(gates: np.ndarray) -> np.ndarray:
    """Rewrites additive kinds into reference gates in time order
    (SURVEY.md 8(d)): U3 -> RZ(lam), RY(theta), RZ(phi); CZ -> H, CX, H."""
    out = []
    for g in gates:
        k = int(g["kind"])
        t, c = int(g["target"]), int(g["control"])
        if k == GateKind.U3:
            out.append(gate(GateKind.Rz, t, theta=g["lam"]))
            out.append(gate(GateKind.Ry, t, theta=g["theta"]))
            out.append(gate(GateKind.Rz, t, theta=g["phi"]))
        elif k == GateKind.Cz:
            out.append(gate(GateKind.H, t))
            out.append(gate(GateKind.Cnot, t, c))
            out.append(gate(GateKind.H, t))
        else:
            out.append(tuple(g.tolist()))
    return gate_array(out)
