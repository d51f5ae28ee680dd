"""Loads the golden fixtures and replays modifier logs on any engine with the
Simulator API (the GPU drop-in or the reference handle)."""
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def load_random():
    d = np.load(os.path.join(HERE, "golden_random.npz"))
    go, so = d["gate_offsets"], d["state_offsets"]
    for i, n in enumerate(d["n"]):
        yield int(n), d["gates"][go[i]:go[i + 1]], d["states"][so[i]:so[i + 1]]


def load_logs(name):
    d = np.load(os.path.join(HERE, name))
    meta = json.loads(str(d["meta"]))
    so = d["state_offsets"]
    states = [d["states"][so[i]:so[i + 1]] for i in range(len(so) - 1)]
    k = 0
    for entry in meta:
        nupd = sum(1 for op in entry["ops"] if op[0] == "update")
        yield entry["n"], entry["ops"], states[k:k + nupd]
        k += nupd


def replay(sim, ops, on_update, reference_kinds=True):
    """Replays a log on `sim` (GPU Simulator API); calls on_update(i) after
    each update_state with the index of the golden state."""
    from paper_2210_01076_b200.gates import GateKind
    nets, gates = [], []
    for op in ops:
        if op[0] == "net_back":
            nets.append(sim.insert_net_back())
        elif op[0] == "net_after":
            nets.append(sim.insert_net_after(nets[op[1]]))
        elif op[0] == "gate":
            _, i, k, t, c, th = op
            kind = GateKind(k)
            if k in (0, 12):
                gates.append(sim.insert_gate(kind, nets[i], t, c))
            else:
                gates.append(sim.insert_gate(kind, th, nets[i], t))
        elif op[0] == "remove_gate":
            sim.remove_gate(gates.pop(op[1]))
        elif op[0] == "remove_net":
            sim.remove_net(nets.pop(op[1]))
        elif op[0] == "update":
            sim.update_state()
            on_update(op[1])
        else:
            raise ValueError(op)
