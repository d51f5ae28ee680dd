"""Does dirty-block tracking pay on the GPU engine? (VERDICT r1 item 8,
SURVEY 7.3 caveat.) Replays workloads through the host partition model
(csrc/qt_partition.hpp, pinned to the reference engine by
tests/test_partition_model.py) and reports, per update, the share of the
state the REFERENCE's partition DAG rewrites (its block-level locality)
next to the share the GPU engine re-streams (every re-simulated segment
rewrites the whole state). CPU only.

  python tools/locality_study.py > profiles/r02_locality.json
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_01076_b200 import workloads as W  # noqa: E402
from paper_2210_01076_b200.gates import GateKind as K  # noqa: E402
from paper_2210_01076_b200.partition import PartitionModel  # noqa: E402


class ModelSim:
    """Simulator-like adapter: assigns net / gate ids like the engine (1, 2,
    ...) and forwards every modifier to the partition model."""

    def __init__(self, n, block=256):
        self.pm = PartitionModel(n, block)
        self.next_net = 1
        self.next_gate = 1
        self.net_gates = {}
        self.n = n

    def _net(self, where, after=0):
        nid = self.next_net
        self.next_net += 1
        self.pm.insert_net(nid, where, after)
        self.net_gates[nid] = []
        return nid

    def insert_net_front(self):
        return self._net("front")

    def insert_net_after(self, a):
        return self._net("after", a)

    def insert_gate(self, kind, *args):
        gid = self.next_gate
        self.next_gate += 1
        ph = la = 0.0
        if len(args) == 3 and isinstance(args[0], (float, tuple)):   # (theta, net, target)
            theta, net, t = args
            c = -1
            if isinstance(theta, tuple):
                theta, ph, la = theta
        else:                                               # (net, target, control)
            net, t, c = args
            theta = 0.0
        self.pm.insert_gate(gid, int(kind), net, int(t), int(c), float(theta), ph, la)
        self.net_gates[net].append(gid)
        return gid

    def remove_net(self, net):
        self.pm.remove_net(net)
        self.net_gates.pop(net, None)

    def update_state(self):
        self.pm.update()
        return self.pm.account()


def study(name, n, gates, mods, block=256):
    sim = ModelSim(n, block)
    drv = W.NetDriver(sim)
    drv.build(gates)
    sim.update_state()
    shares = {"uniform": [], "tail": []}
    for m, mod in enumerate(mods):
        cls = "tail" if (m // 2) % 2 == 1 else "uniform"
        drv.modify(mod)
        acc = sim.update_state()
        shares[cls].append(acc["rewritten_amplitudes"] / float(1 << n))
    out = {"workload": name, "qubits": n, "block_size": block}
    for cls, xs in shares.items():
        if xs:
            out[cls] = {"updates": len(xs), "mean_share_rewritten": statistics.mean(xs),
                        "min_share": min(xs), "max_share": max(xs)}
    return out


def cnot_chain(n=15, count=100):
    """acceptance.cpp:362-395's locality workload: a CNOT chain; edits touch
    the first / last net."""
    from paper_2210_01076_b200.gates import gate, gate_array
    g = gate_array([gate(K.Cnot, (i % (n - 1)) + 1, i % (n - 1)) for i in range(count)])
    mods = []
    for at in (count - 1, 0, count // 2, count - 2):
        row = tuple(g[at].tolist())
        mods += [("remove", at), ("insert", at, row)]
    return g, mods


rows = []
w1 = W.config1()
rows.append(study("c1_random16", w1.n, w1.gates, w1.modifiers))
w5 = W.config5(n=16, nmods=40)
rows.append(study("c5_incremental@n=16", 16, w5.gates, w5.modifiers))
g, mods = cnot_chain()
rows.append(study("cnot_chain15 (acceptance criterion 8)", 15, g, mods))
w3 = W.config3(n=16, layers=20)
rows.append(study("c3_layered@n=16 (no modifiers: full only)", 16, w3.gates, []))
print(json.dumps({"tool": "tools/locality_study.py", "rows": rows,
                  "gpu_engine": "re-simulates whole-state segments: share rewritten = 1.0 per "
                                "re-simulated segment"}, indent=1))
