"""Modifier traces and the incremental-iteration harness.

* The reference's trace wire format (tools/qtask_cli.cpp:118-359): one
  statement per line --
      qubits <n>
      net <id> [front | after <net-id>]
      gate <id> <KIND>[(<angle>)] <net-id> <target> [<control>]
      remove_gate <id> | remove_net <id> | update | dump <path>
  '#' lines and blank lines are skipped; KIND is CNOT X Y Z H S SDG T TDG RX
  RY RZ SWAP; an angle is [-](pi | pi/<d> | <number>). `parse` / `replay`
  restate it for any Simulator-like object (this package's Simulator, or the
  reference engine in the tests); `dump` writes the circuit (net order and
  gates: the partition-DAG DOT of the reference is out of scope).
* The paper's incremental iterations (qtask_cli.cpp:365-502, PAPER.md
  "Performance of Incremental Simulation"): a QASM program's ASAP levels are
  inserted / removed a few levels at a time, one update_state per iteration
  -- modes insert-sweep, remove-sweep, mix. `run_iterations` returns one row
  (iteration, wall ms, executed partitions) per update.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import qasm as _qasm
from .errors import Error
from .gates import GateKind as K

_KINDS = {"CNOT": K.Cnot, "X": K.X, "Y": K.Y, "Z": K.Z, "H": K.H, "S": K.S, "SDG": K.Sdg,
          "T": K.T, "TDG": K.Tdg, "RX": K.Rx, "RY": K.Ry, "RZ": K.Rz, "SWAP": K.Swap}
_NAMES = {v: k for k, v in _KINDS.items()}


@dataclass
class TraceStmt:
    kind: str                      # net | gate | remove_gate | remove_net | update | dump
    id: str = ""
    anchor: str = ""               # net: `after` anchor
    front: bool = False
    gate: K = K.X
    theta: float = 0.0
    has_theta: bool = False
    net: str = ""
    target: int = 0
    control: int = -1
    path: str = ""
    line: int = 0


@dataclass
class Trace:
    num_qubits: int = 0
    stmts: list = field(default_factory=list)


def _angle(text: str, line: int) -> float:
    sign = 1.0
    if text.startswith("-"):
        sign, text = -1.0, text[1:]
    if text == "pi":
        return sign * math.pi
    if text.startswith("pi/"):
        try:
            d = float(text[3:])
        except ValueError:
            d = 0.0
        if d == 0.0:
            raise Error(f"bad angle at trace line {line}")
        return sign * math.pi / d
    try:
        return sign * float(text)
    except ValueError:
        raise Error(f"bad angle at trace line {line}") from None


def parse(text: str) -> Trace:
    tr = Trace()
    seen_qubits = False
    for no, raw in enumerate(text.splitlines(), start=1):
        words = raw.split()
        if not words or words[0].startswith("#"):
            continue
        head, rest = words[0], words[1:]
        if head == "qubits":
            try:
                tr.num_qubits = int(rest[0])
            except (IndexError, ValueError):
                tr.num_qubits = 0
            if tr.num_qubits < 1:
                raise Error(f"bad qubits line {no}")
            seen_qubits = True
            continue
        if not seen_qubits:
            raise Error("trace must start with 'qubits <n>'")
        st = TraceStmt(kind=head, line=no)
        if head == "net":
            if not rest:
                raise Error(f"net needs an id, line {no}")
            st.id = rest[0]
            if len(rest) > 1:
                if rest[1] == "front":
                    st.front = True
                elif rest[1] == "after":
                    if len(rest) < 3:
                        raise Error(f"'after' needs a net id, line {no}")
                    st.anchor = rest[2]
                else:
                    raise Error(f"unexpected '{rest[1]}', line {no}")
        elif head == "gate":
            if len(rest) < 4:
                raise Error(f"malformed gate line {no}")
            st.id, token, st.net = rest[0], rest[1], rest[2]
            try:
                st.target = int(rest[3])
            except ValueError:
                raise Error(f"malformed gate line {no}") from None
            if "(" in token:
                if not token.endswith(")"):
                    raise Error(f"malformed angle, line {no}")
                p = token.index("(")
                st.theta = _angle(token[p + 1:-1], no)
                st.has_theta = True
                token = token[:p]
            if token not in _KINDS:
                raise Error(f"unknown gate kind '{token}' at trace line {no}")
            st.gate = _KINDS[token]
            st.control = int(rest[4]) if len(rest) > 4 and _is_int(rest[4]) else -1
        elif head in ("remove_gate", "remove_net"):
            st.id = rest[0] if rest else ""
        elif head == "update":
            pass
        elif head == "dump":
            if not rest:
                raise Error(f"dump needs a path, line {no}")
            st.path = rest[0]
        else:
            raise Error(f"unknown trace statement '{head}', line {no}")
        tr.stmts.append(st)
    if not seen_qubits:
        raise Error("trace must start with 'qubits <n>'")
    return tr


def _is_int(s: str) -> bool:
    try:
        int(s)
        return True
    except ValueError:
        return False


def dump_circuit(sim, path: str) -> None:
    """Net order and gates of ``sim`` (this package's Simulator) as text."""
    view = sim.circuit()
    with open(path, "w") as f:
        for net in view.net_order():
            f.write(f"net {net}:")
            for g in view.net(net):
                rec = view.gate(g)
                f.write(f" {_NAMES.get(K(rec.kind), rec.kind)}[{rec.target},{rec.control}]")
            f.write("\n")


def replay(sim, trace: Trace, verify=None, insert_gate=None):
    """Replays ``trace`` on ``sim``; returns one dict per `update`
    (time_ms, partitions, amplitudes rewritten; maxdev if ``verify(sim)`` is
    given). ``insert_gate(sim, kind, theta_or_None, net, target, control)``
    adapts other Simulator-like APIs (default: this package's)."""
    if insert_gate is None:
        def insert_gate(s, kind, theta, net, target, control):
            if control >= 0:
                return s.insert_gate(kind, net, target, control)
            if theta is not None:
                return s.insert_gate(kind, theta, net, target)
            return s.insert_gate(kind, net, target)
    nets, gates, rows = {}, {}, []

    def net_of(i):
        if i not in nets:
            raise Error(f"unknown net id '{i}'")
        return nets[i]

    for st in trace.stmts:
        if st.kind == "net":
            if st.id in nets:
                raise Error(f"duplicate net id '{st.id}'")
            if st.front:
                nets[st.id] = sim.insert_net_front()
            elif st.anchor:
                nets[st.id] = sim.insert_net_after(net_of(st.anchor))
            else:
                nets[st.id] = sim.insert_net_back()
        elif st.kind == "gate":
            if st.id in gates:
                raise Error(f"duplicate gate id '{st.id}'")
            gates[st.id] = insert_gate(sim, st.gate, st.theta if st.has_theta else None,
                                       net_of(st.net), st.target, st.control)
        elif st.kind == "remove_gate":
            if st.id not in gates:
                raise Error(f"unknown gate id '{st.id}'")
            sim.remove_gate(gates.pop(st.id))
        elif st.kind == "remove_net":
            sim.remove_net(net_of(st.id))
            del nets[st.id]
        elif st.kind == "update":
            t0 = time.perf_counter()
            sim.update_state()
            row = {"update": len(rows) + 1, "time_ms": (time.perf_counter() - t0) * 1e3}
            stats = getattr(sim, "last_update", None)
            if callable(stats):
                s = stats()
                row.update(partitions=s.executed_partitions,
                           amplitudes=s.rewritten_amplitudes)
            if verify is not None:
                row["maxdev"] = verify(sim)
            rows.append(row)
        elif st.kind == "dump":
            dump_circuit(sim, st.path)
    return rows


# ---- incremental iterations over QASM levels (the paper's benchmark) -------


def level_plan(program: _qasm.QasmProgram):
    """[[Statement, ...] per ASAP level] of a parsed QASM program."""
    return [[program.statements[i] for i in lv] for lv in _qasm.levelize(program)]


def _insert_level(sim, present, plan, level, insert_gate):
    below = [l for l in present if l < level]
    net = sim.insert_net_after(present[max(below)]) if below else sim.insert_net_front()
    present[level] = net
    for st in plan[level]:
        g = K(st.gate)
        if g == K.Cnot:
            insert_gate(sim, g, None, net, st.qubits[1], st.qubits[0])
        elif g == K.Swap:
            insert_gate(sim, g, None, net, st.qubits[0], st.qubits[1])
        else:
            insert_gate(sim, g, st.theta if st.has_theta else None, net, st.qubits[0], -1)


def run_iterations(make_sim, num_qubits, plan, mode, seed=0, per_iter=1, iters=10,
                   insert_gate=None, finish=None):
    """insert-sweep: levels inserted in a shuffled order, `per_iter` per
    iteration; remove-sweep: full circuit, then random levels removed;
    mix: full circuit, then `iters` iterations of random removes / re-inserts.
    One update_state per iteration. Returns (rows, sim-result of `finish`)."""
    if insert_gate is None:
        def insert_gate(s, kind, theta, net, target, control):
            if control >= 0:
                return s.insert_gate(kind, net, target, control)
            if theta is not None:
                return s.insert_gate(kind, theta, net, target)
            return s.insert_gate(kind, net, target)
    rng = np.random.default_rng(seed)
    sim = make_sim(num_qubits)
    present, rows = {}, []

    def update():
        t0 = time.perf_counter()
        sim.update_state()
        ms = (time.perf_counter() - t0) * 1e3
        stats = getattr(sim, "last_update", None)
        part = stats().executed_partitions if callable(stats) else None
        rows.append({"iteration": len(rows), "wall_time_ms": ms, "executed_partitions": part})

    def full():
        for lv in range(len(plan)):
            _insert_level(sim, present, plan, lv, insert_gate)
        update()

    if mode == "insert-sweep":
        order = rng.permutation(len(plan))
        for i in range(0, len(order), per_iter):
            for lv in order[i:i + per_iter]:
                _insert_level(sim, present, plan, int(lv), insert_gate)
            update()
    elif mode == "remove-sweep":
        full()
        while present:
            for _ in range(per_iter):
                if not present:
                    break
                lv = sorted(present)[int(rng.integers(len(present)))]
                sim.remove_net(present.pop(lv))
            update()
    elif mode == "mix":
        full()
        absent = []
        for _ in range(iters):
            for _ in range(per_iter):
                remove = bool(present) and (not absent or rng.integers(2) == 0)
                if remove:
                    lv = sorted(present)[int(rng.integers(len(present)))]
                    sim.remove_net(present.pop(lv))
                    absent.append(lv)
                elif absent:
                    lv = absent.pop(int(rng.integers(len(absent))))
                    _insert_level(sim, present, plan, lv, insert_gate)
            update()
    else:
        raise Error(f"unknown bench mode '{mode}'")
    out = finish(sim) if finish else None
    close = getattr(sim, "close", None)
    if close:
        close()
    return rows, out


def rows_csv(rows) -> str:
    """The reference harness's CSV (iteration,wall_time_ms,executed_partitions)."""
    lines = ["iteration,wall_time_ms,executed_partitions"]
    lines += [f"{r['iteration']},{r['wall_time_ms']:.3f},{r['executed_partitions']}" for r in rows]
    return "\n".join(lines) + "\n"
