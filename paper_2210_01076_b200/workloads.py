"""Seeded synthetic workloads of BASELINE.json's five configs.

The reference measures on QASMBench circuits, which are not
in this environment; these generators stand in with the shapes BASELINE.json
names. Each gate list is generated ONCE and fed identically
to the GPU engine, the dense oracle and the reference (numpy PCG64, seed =
config index). Additive kinds (U3, CZ) are lowered to reference gates with
``gates.lower_to_reference`` for the reference / oracle side.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .gates import GateKind as K
from .gates import gate, gate_array

TWO_PI = 2.0 * math.pi
C1_KINDS = [K.H, K.X, K.Y, K.Z, K.S, K.T, K.Rx, K.Ry, K.Rz, K.Cnot, K.Cz]
C4_KINDS = [K.H, K.Rx, K.Ry, K.Rz, K.Cnot, K.Cz]
C5_KINDS = [K.H, K.X, K.T, K.Rz, K.Ry, K.Cnot, K.Cz]


def random_gate(rng: np.random.Generator, n: int, kinds, global_qubits=None,
                p_global: float = 0.0):
    """One gate: kind uniform; target uniform; control (2-qubit kinds) uniform
    and distinct; angle uniform in [0, 2pi). With global_qubits, a gate acts
    on one of them with probability p_global (target in the set, control over
    the other qubits), otherwise all operands avoid them (config 4)."""
    kind = kinds[int(rng.integers(len(kinds)))]
    two = kind in (K.Cnot, K.Cz, K.Swap)
    if global_qubits:
        if rng.random() < p_global:
            target = int(global_qubits[int(rng.integers(len(global_qubits)))])
            pool = [q for q in range(n) if q != target]
        else:
            pool = [q for q in range(n) if q not in global_qubits]
            target = int(pool[int(rng.integers(len(pool)))])
            pool = [q for q in pool if q != target]
        control = int(pool[int(rng.integers(len(pool)))]) if two else -1
    else:
        target = int(rng.integers(n))
        control = -1
        if two:
            control = target
            while control == target:
                control = int(rng.integers(n))
    theta = float(rng.uniform(0.0, TWO_PI)) if kind in (K.Rx, K.Ry, K.Rz) else 0.0
    return gate(kind, target, control, theta)


@dataclass
class Workload:
    name: str
    n: int
    gates: np.ndarray                  # logical gate list (may hold U3 / CZ)
    metric_gates: int                  # G of the metric (logical gates)
    modifiers: list = field(default_factory=list)  # [("insert", pos, gate) | ("remove", pos)]
    basis: int = 0
    note: str = ""


def _modifiers(rng, n, kinds, base_len, count, tail_split=False):
    """count modifiers over a circuit of base_len gates. Config 1: insert or
    remove 50/50, position uniform over [0, len]. Config 5 (tail_split):
    modifier m inserts if m even, removes if odd; the position is uniform over
    the whole circuit if floor(m/2) is even, else over the last ceil(10%)."""
    mods = []
    length = base_len
    for m in range(count):
        if tail_split:
            insert = m % 2 == 0
            tail = (m // 2) % 2 == 1
        else:
            insert = bool(rng.integers(2) == 0) or length == 0
            tail = False
        hi = length + 1 if insert else length
        if tail:
            span = max(1, math.ceil(0.1 * length))
            lo = max(0, hi - span)
        else:
            lo = 0
        pos = int(rng.integers(lo, hi))
        if insert:
            mods.append(("insert", pos, random_gate(rng, n, kinds)))
            length += 1
        else:
            mods.append(("remove", pos))
            length -= 1
    return mods


def config1(seed: int = 1, n: int = 16, ngates: int = 400, nmods: int = 20) -> Workload:
    rng = np.random.default_rng(seed)
    gates = gate_array(random_gate(rng, n, C1_KINDS) for _ in range(ngates))
    mods = _modifiers(rng, n, C1_KINDS, ngates, nmods)
    return Workload("c1_random16", n, gates, ngates, mods,
                    note="16q random {H,X,Y,Z,S,T,RX,RY,RZ,CX,CZ}, 400 gates + 20 modifiers")


def qft_gates(n: int, basis: int):
    """X on the set bits of `basis`, then the QFT: for j = n-1..0: H(j), then
    CP(pi/2^(j-k)) (control k, target j) for k = j-1..0, each CP lowered to
    RZ_c(l/2), CX(c->t), RZ_t(-l/2), CX(c->t), RZ_t(l/2) (= e^{-il/4} CP);
    then SWAP(i, n-1-i) for i < n/2 as three CX."""
    rows = [gate(K.X, q) for q in range(n) if (basis >> q) & 1]
    for j in range(n - 1, -1, -1):
        rows.append(gate(K.H, j))
        for k in range(j - 1, -1, -1):
            lam = math.pi / (2 ** (j - k))
            rows.append(gate(K.Rz, k, theta=lam / 2))
            rows.append(gate(K.Cnot, j, k))
            rows.append(gate(K.Rz, j, theta=-lam / 2))
            rows.append(gate(K.Cnot, j, k))
            rows.append(gate(K.Rz, j, theta=lam / 2))
    for i in range(n // 2):
        a, b = i, n - 1 - i
        rows.append(gate(K.Cnot, b, a))
        rows.append(gate(K.Cnot, a, b))
        rows.append(gate(K.Cnot, b, a))
    return gate_array(rows)


def qft_closed_form(n: int, basis: int) -> np.ndarray:
    """Exact output of qft_gates(n, basis) on |0>: a_k = 2^(-n/2) *
    exp(i (2 pi ((b k) mod 2^n) / 2^n - Phi)), Phi = sum over CPs of l/4 =
    (pi/4)(n - 2 + 2^-(n-1))."""
    dim = 1 << n
    k = np.arange(dim, dtype=np.uint64)
    phase_idx = (np.uint64(basis) * k) & np.uint64(dim - 1)
    phi = (math.pi / 4.0) * (n - 2 + 2.0 ** (-(n - 1)))
    ang = 2.0 * math.pi * phase_idx.astype(np.float64) / dim - phi
    return (2.0 ** (-n / 2.0)) * np.exp(1j * ang)


def config2(seed: int = 2, n: int = 24) -> Workload:
    rng = np.random.default_rng(seed)
    basis = int(rng.integers(1 << n))
    gates = qft_gates(n, basis)
    return Workload("c2_qft24", n, gates, len(gates), basis=basis,
                    note="24q QFT of a seeded basis state, CP as RZ+CX, swaps as 3 CX")


def config3(seed: int = 3, n: int = 30, layers: int = 20) -> Workload:
    rng = np.random.default_rng(seed)
    rows = []
    for layer in range(layers):
        for q in range(n):
            th, ph, la = rng.uniform(0.0, TWO_PI, 3)
            rows.append(gate(K.U3, q, theta=th, phi=ph, lam=la))
        start = 0 if layer % 2 == 0 else 1
        for a in range(start, n - 1, 2):
            rows.append(gate(K.Cz, a + 1, a))
    g = gate_array(rows)
    return Workload("c3_layered30", n, g, len(g),
                    note=f"{n}q, {layers} layers of U3 on every qubit + CZ brick-wall")


def config4(seed: int = 4, n: int = 33, ngates: int = 1500, nglobal: int = 3) -> Workload:
    rng = np.random.default_rng(seed)
    glob = list(range(n - nglobal, n))
    g = gate_array(random_gate(rng, n, C4_KINDS, glob, 0.3) for _ in range(ngates))
    return Workload("c4_random33", n, g, ngates,
                    note=f"{n}q random {{H,RX,RY,RZ,CX,CZ}}, 30% on the top {nglobal} qubits")


def config5(seed: int = 5, n: int = 28, ngates: int = 5000, nmods: int = 1000) -> Workload:
    rng = np.random.default_rng(seed)
    g = gate_array(random_gate(rng, n, C5_KINDS) for _ in range(ngates))
    mods = _modifiers(rng, n, C5_KINDS, ngates, nmods, tail_split=True)
    return Workload("c5_incremental28", n, g, ngates, mods,
                    note=f"{n}q, {ngates} random {{H,X,T,RZ,RY,CX,CZ}} + {nmods} modifiers")


def apply_modifier(gates: np.ndarray, mod) -> np.ndarray:
    """The logical gate list after one modifier."""
    if mod[0] == "insert":
        row = gate_array([mod[2]])
        return np.concatenate([gates[:mod[1]], row, gates[mod[1]:]])
    return np.concatenate([gates[:mod[1]], gates[mod[1] + 1:]])


class NetDriver:
    """Replays a logical gate list + modifiers through a Simulator-like object
    (the GPU drop-in or the reference), one net per gate.
    With ``reference_gates`` every additive gate takes 3 nets (CZ -> H,CX,H;
    U3 -> RZ,RY,RZ), as the reference has no U3/CZ."""

    def __init__(self, sim, reference_gates: bool = False):
        self.sim = sim
        self.ref = reference_gates
        self.nets = []  # per logical gate: list of net ids

    def _expand(self, row):
        kind, t, c, _, th, ph, la = row
        kind = K(int(kind))
        if self.ref and kind == K.Cz:
            return [(K.H, t, -1, 0.0), (K.Cnot, t, c, 0.0), (K.H, t, -1, 0.0)]
        if self.ref and kind == K.U3:
            return [(K.Rz, t, -1, la), (K.Ry, t, -1, th), (K.Rz, t, -1, ph)]
        return [(kind, t, c, (th, ph, la) if kind == K.U3 else th)]

    def _insert_gate_nets(self, anchor, row):
        ids = []
        for (kind, t, c, th) in self._expand(row):
            net = self.sim.insert_net_front() if anchor is None else self.sim.insert_net_after(anchor)
            if kind in (K.Cnot, K.Cz, K.Swap):
                if self.ref:
                    self.sim.insert_gate(int(kind), net, int(t), int(c))
                else:
                    self.sim.insert_gate(kind, net, int(t), int(c))
            else:
                if self.ref:
                    self.sim.insert_gate(int(kind), net, int(t), -1, float(th))
                else:
                    self.sim.insert_gate(kind, th, net, int(t))
            ids.append(net)
            anchor = net
        return ids

    def build(self, gates: np.ndarray):
        anchor = None
        for row in gates.tolist():
            ids = self._insert_gate_nets(anchor, row)
            self.nets.append(ids)
            anchor = ids[-1]

    def modify(self, mod):
        if mod[0] == "insert":
            pos = mod[1]
            anchor = self.nets[pos - 1][-1] if pos > 0 else None
            ids = self._insert_gate_nets(anchor, mod[2])
            self.nets.insert(pos, ids)
        else:
            for net in self.nets.pop(mod[1]):
                self.sim.remove_net(net)
