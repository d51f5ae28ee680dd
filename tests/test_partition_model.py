"""The drop-in's host partition model (csrc/qt_partition.hpp: the
reference's partition DAG restated for reference-unit UpdateStats and the
introspection members) against the reference engine itself, compiled from
its sources (oracle/_ref): after every modifier the DOT dumps (node names,
read ranges, every edge -- graph.cpp:302-327) must be identical, and after
every update_state the accounting (executed partitions, materialised
blocks, rewritten blocks and amplitudes -- engine.cpp:392-504). CPU only.
Plus the reference acceptance suite's structural goldens (acceptance.cpp:
180-395, criteria 3, 4, 5, 8) on the model."""
import math

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.partition import PartitionModel

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")

KINDS = [K.Cnot, K.X, K.Y, K.Z, K.H, K.S, K.Sdg, K.T, K.Tdg, K.Rx, K.Ry, K.Rz, K.Swap]


def random_gate(rng, n):
    """test_support.hpp:137-167's distribution: all 13 kinds, rotations at
    pi, pi/2, 0 or uniform in (-2pi, 2pi)."""
    kind = KINDS[int(rng.integers(0, 13 if n >= 2 else 12))]
    if n < 2 and kind in (K.Cnot, K.Swap):
        kind = K.H
    t = int(rng.integers(0, n))
    c = -1
    if kind in (K.Cnot, K.Swap):
        c = t
        while c == t:
            c = int(rng.integers(0, n))
    theta = 0.0
    if kind in (K.Rx, K.Ry, K.Rz):
        theta = [math.pi, math.pi / 2, 0.0, float(rng.uniform(-2 * math.pi, 2 * math.pi))][int(rng.integers(0, 4))]
    return int(kind), t, c, theta


class Pair:
    """The reference engine and the model, driven with the same modifiers."""

    def __init__(self, n, block):
        self.ref = oracle.RefSimulator(n, block, 1)
        self.pm = PartitionModel(n, block)
        self.members = {}  # net -> its live gates

    def check_graph(self):
        assert self.pm.dump_graph() == self.ref.dump_graph()

    def net(self, where, after=0):
        code = {"front": 0, "back": 1, "after": 2}[where]
        nid = self.ref.lib.ref_sim_insert_net(self.ref.h, code, after)
        assert nid > 0
        self.pm.insert_net(nid, where, after)
        return nid

    def gate(self, kind, net, t, c=-1, theta=0.0):
        gid = self.ref.lib.ref_sim_insert_gate(self.ref.h, kind, theta, net, t, c)
        if gid < 0:
            return None  # rejected by the reference (net conflict ...)
        self.pm.insert_gate(gid, kind, net, t, c, theta)
        self.members.setdefault(net, []).append(gid)
        return gid

    def remove_gate(self, g):
        self.ref.remove_gate(g)
        self.pm.remove_gate(g)
        for gs in self.members.values():
            if g in gs:
                gs.remove(g)

    def remove_net(self, n):
        self.ref.remove_net(n)
        self.pm.remove_net(n)
        return self.members.pop(n, [])

    def update(self):
        self.ref.update_state()
        self.pm.update()
        want = self.ref.stats()
        got = self.pm.account()
        assert got == want
        return got


@pytest.mark.parametrize("seed", range(80))
def test_random_modifier_sequences_match_the_reference(seed):
    rng = np.random.default_rng(31000 + seed)
    n = int(rng.integers(1, 10))
    block = 1 << int(rng.integers(1, 8))
    p = Pair(n, block)
    nets, gates = [], []
    for _ in range(int(rng.integers(10, 120))):
        roll = int(rng.integers(0, 12))
        if roll < 3 or not nets:
            if not nets or rng.integers(0, 2) == 0:
                nets.append(p.net("back" if rng.integers(0, 4) else "front"))
            else:
                nets.append(p.net("after", nets[int(rng.integers(0, len(nets)))]))
        elif roll < 9:
            kind, t, c, theta = random_gate(rng, n)
            g = p.gate(kind, nets[int(rng.integers(0, len(nets)))], t, c, theta)
            if g is not None:
                gates.append(g)
        elif roll < 10 and gates:
            g = gates.pop(int(rng.integers(0, len(gates))))
            p.remove_gate(g)
        elif roll < 11 and len(nets) > 1:
            at = int(rng.integers(0, len(nets)))
            net = nets.pop(at)
            mine = set(p.remove_net(net))
            gates = [g for g in gates if g not in mine]
        else:
            p.update()
        p.check_graph()
    p.update()
    p.check_graph()


def entangle5(block):
    """acceptance.cpp:43-63: H on all 5 qubits, then CNOTs G6..G9."""
    p = Pair(5, block)
    n1, n2, n3, n4, n5 = (p.net("back") for _ in range(5))
    for q in range(4, -1, -1):
        p.gate(int(K.H), n1, q)
    g6 = p.gate(int(K.Cnot), n2, 3, 4)
    g7 = p.gate(int(K.Cnot), n3, 1, 4)
    g8 = p.gate(int(K.Cnot), n4, 2, 3)
    g9 = p.gate(int(K.Cnot), n5, 0, 2)
    return p, (n1, n2, n3, n4, n5), (g6, g7, g8, g9)


def test_golden_impact_criterion_4():
    """After the G8 -> G10 edit: 4 partitions, 24 amplitudes, blocks
    1,2,3,5,6,7 rewritten (acceptance.cpp:231-261)."""
    p, nets, (g6, g7, g8, g9) = entangle5(4)
    p.update()
    p.remove_gate(g8)
    g10 = p.gate(int(K.Cnot), nets[3], 1, 2)
    assert g10 is not None
    acc = p.update()
    assert acc["executed_partitions"] == 4 and acc["rewritten_amplitudes"] == 24
    assert acc["rewritten_blocks"] == [1, 2, 3, 5, 6, 7]


def test_golden_connectivity_criterion_5():
    """G10 gains 5 predecessors + 2 successors and 5 transitive edges drop
    (acceptance.cpp:267-319): the model's edge set equals the reference's,
    named, before and after the insertion."""
    p, nets, (g6, g7, g8, g9) = entangle5(4)
    p.remove_gate(g8)
    p.check_graph()
    p.gate(int(K.Cnot), nets[3], 1, 2)
    p.check_graph()
    dot = p.pm.dump_graph()
    for e in ["MxV1_1 -> g10_p0", "g7_p0 -> g10_p1", "g10_p0 -> g9_p0", "g10_p1 -> g9_p1"]:
        assert e in dot
    assert "MxV1_1 -> g9_p0" not in dot


def test_locality_criterion_8():
    """A last-net edit executes <= 10% of the partitions of a first-net edit
    (acceptance.cpp:362-395): 100 CNOTs on a 15-qubit chain."""
    n = 15
    p = Pair(n, 256)
    nets, gates, qs = [], [], []
    for i in range(100):
        c = i % (n - 1)
        t = c + 1
        net = p.net("back")
        nets.append(net)
        gates.append(p.gate(int(K.Cnot), net, t, c))
        qs.append((c, t))
    p.update()

    def touch(at):
        p.remove_gate(gates[at])
        gates[at] = p.gate(int(K.Cnot), nets[at], qs[at][1], qs[at][0])
        return p.update()["executed_partitions"]

    last = touch(99)
    first = touch(0)
    assert first > 0 and last * 10 <= first
