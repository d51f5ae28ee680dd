"""Python mirror of ``qtask::Simulator`` (reference engine.hpp:46-151).

Same member names, argument meaning and exceptions as the reference C++ API,
over the qt_sim_* C ABI (incremental engine on the GPU):

    sim = Simulator(5, Config(block_size=4, threads=1))
    n1 = sim.insert_net_back()
    g = sim.insert_gate(GateKind.H, n1, 0)                 # insert_gate(kind, net, t)
    sim.insert_gate(GateKind.Rx, 0.5, n2, 1)               # (kind, theta, net, t)
    sim.insert_gate(GateKind.Cnot, n3, 1, 0)               # (kind, net, t, control)
    sim.update_state()
    sim.amplitude(3); sim.amplitudes(0, 31); sim.norm_squared()
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _ffi
from ._ffi import GATE_DTYPE, check, lib
from .errors import Error
from .gates import GateKind, is_two_qubit


@dataclass
class Config:
    """Reference Config (plan.hpp:17-20) + GPU knobs (0 = auto)."""
    block_size: int = 256
    threads: int = 0
    device: int = -1
    tile_qubits: int = 0
    max_checkpoints: int = 0
    checkpoint_fraction: float = 0.0
    segment_gates: int = 0
    compiled: int = 0          # 0: hybrid compiled passes (default), -1: interpreter only


@dataclass
class UpdateStats:
    """Reference UpdateStats (engine.hpp:32-39) in GPU terms."""
    full: bool
    executed_partitions: int
    rewritten_amplitudes: int
    passes: int
    segments: int
    restart_gate: int
    gates: int
    hbm_bytes: int
    wall_ms: float


@dataclass
class GateRecord:
    """Reference Gate (circuit.hpp:14-21)."""
    id: int
    kind: GateKind
    theta: float
    net: int
    target: int
    control: int
    phi: float = 0.0
    lam: float = 0.0


class CircuitView:
    """Read-only view of the simulator's circuit (Circuit, circuit.hpp:32-66)."""

    def __init__(self, sim: "Simulator"):
        self._sim = sim

    def num_qubits(self) -> int:
        return self._sim.num_qubits()

    def net_order(self):
        n = lib().qt_sim_num_nets(self._sim._h)
        out = np.zeros(n, dtype=np.uint32)
        check(lib().qt_sim_net_order(self._sim._h, out.ctypes.data, n))
        return out.tolist()

    def net(self, net_id: int):
        cnt = ctypes.c_size_t(0)
        check(lib().qt_sim_net_gates(self._sim._h, net_id, None, 0, ctypes.byref(cnt)))
        out = np.zeros(cnt.value, dtype=np.uint32)
        check(lib().qt_sim_net_gates(self._sim._h, net_id, out.ctypes.data, cnt.value,
                                     ctypes.byref(cnt)))
        return out.tolist()

    def gate(self, gate_id: int) -> GateRecord:
        g = np.zeros(1, dtype=GATE_DTYPE)
        net = ctypes.c_uint32(0)
        check(lib().qt_sim_gate_info(self._sim._h, gate_id, g.ctypes.data, ctypes.byref(net)))
        r = g[0]
        return GateRecord(gate_id, GateKind(int(r["kind"])), float(r["theta"]), net.value,
                          int(r["target"]), int(r["control"]), float(r["phi"]), float(r["lam"]))

    def num_gates(self) -> int:
        return lib().qt_sim_num_gates(self._sim._h)

    def gates(self) -> np.ndarray:
        """Flattened qt_gate array in simulation order (nets in order, gates in
        insertion order) -- what the dense oracle consumes."""
        cnt = ctypes.c_size_t(0)
        check(lib().qt_sim_export_gates(self._sim._h, None, 0, ctypes.byref(cnt)))
        out = np.zeros(cnt.value, dtype=GATE_DTYPE)
        check(lib().qt_sim_export_gates(self._sim._h, out.ctypes.data, cnt.value,
                                        ctypes.byref(cnt)))
        return out


class Simulator:
    """Incremental state-vector simulator; see module docstring."""

    def __init__(self, num_qubits: int, cfg: Config | None = None):
        cfg = cfg or Config()
        bs = cfg.block_size
        if bs < 2 or bs & (bs - 1):  # validate_config (plan.cpp:7-13); the C ABI reads 0 as default
            raise Error("block size must be a power of two >= 2")
        self._cfg = cfg
        c = _ffi.make_config(cfg.block_size, cfg.threads, cfg.device, cfg.tile_qubits,
                             cfg.max_checkpoints, cfg.checkpoint_fraction, cfg.segment_gates,
                             cfg.compiled)
        self._h = ctypes.c_void_p()
        check(lib().qt_sim_create(num_qubits, ctypes.byref(c), ctypes.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().qt_sim_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- properties (engine.hpp:50-55)
    def num_qubits(self) -> int:
        return lib().qt_sim_num_qubits(self._h)

    def config(self) -> Config:
        return self._cfg

    def block_size(self) -> int:
        return lib().qt_sim_block_size(self._h)

    def total_blocks(self) -> int:
        return lib().qt_sim_total_blocks(self._h)

    def circuit(self) -> CircuitView:
        return CircuitView(self)

    # -- modifiers (engine.hpp:57-64)
    def _net(self, fn, *args) -> int:
        out = ctypes.c_uint32(0)
        check(fn(self._h, *args, ctypes.byref(out)))
        return out.value

    def insert_net_front(self) -> int:
        return self._net(lib().qt_sim_insert_net_front)

    def insert_net_back(self) -> int:
        return self._net(lib().qt_sim_insert_net_back)

    def insert_net_after(self, after: int) -> int:
        return self._net(lib().qt_sim_insert_net_after, after)

    def remove_net(self, net: int) -> None:
        check(lib().qt_sim_remove_net(self._h, net))

    def insert_gate(self, kind, *args) -> int:
        """insert_gate(kind, net, target) | insert_gate(kind, theta, net, target) |
        insert_gate(kind, net, target, control) | insert_gate(U3, (t, p, l), net, target)."""
        kind = GateKind(kind)
        params = (ctypes.c_double * 3)(0.0, 0.0, 0.0)
        if is_two_qubit(kind):
            net, target, control = args
        elif len(args) == 3:
            theta, net, target = args
            if isinstance(theta, (tuple, list)):
                params[0], params[1], params[2] = theta
            else:
                params[0] = theta
            control = -1
        else:
            net, target = args
            control = -1
        out = ctypes.c_uint32(0)
        check(lib().qt_sim_insert_gate(self._h, int(kind), params, net, target, control,
                                       ctypes.byref(out)))
        return out.value

    def remove_gate(self, gate: int) -> None:
        check(lib().qt_sim_remove_gate(self._h, gate))

    # -- state update (engine.hpp:71)
    def update_state(self) -> None:
        check(lib().qt_sim_update_state(self._h))

    def pending_modifiers(self) -> bool:
        return bool(lib().qt_sim_pending(self._h))

    # -- queries (engine.hpp:77-83)
    def amplitude(self, index: int) -> complex:
        out = np.zeros(1, dtype=np.complex128)
        check(lib().qt_sim_amplitude(self._h, index, out.ctypes.data))
        return complex(out[0])

    def amplitudes(self, first: int, last: int) -> np.ndarray:
        out = np.empty(max(0, last - first + 1), dtype=np.complex128)
        check(lib().qt_sim_amplitudes(self._h, first, last, out.ctypes.data))
        return out

    def top_k(self, k: int):
        """The reference's amplitude report (qtask_cli.cpp:53-86): indices and
        amplitudes of the k largest |a|^2 (ties: smaller index first),
        selected on the device. StaleStateError while modifiers pend."""
        k = min(int(k), 1 << self.num_qubits())
        idx = np.empty(max(1, k), dtype=np.uint64)
        amps = np.empty(max(1, k), dtype=np.complex128)
        cnt = ctypes.c_uint64(0)
        check(lib().qt_sim_top_k(self._h, k, idx.ctypes.data, amps.ctypes.data,
                                 ctypes.byref(cnt)))
        return idx[:cnt.value], amps[:cnt.value]

    def norm_squared(self) -> float:
        v = ctypes.c_double(0.0)
        check(lib().qt_sim_norm_squared(self._h, ctypes.byref(v)))
        return v.value

    def last_update(self) -> UpdateStats:
        s = _ffi.QtRunStats()
        check(lib().qt_sim_last_update(self._h, ctypes.byref(s)))
        return UpdateStats(bool(s.full), s.executed_partitions, s.rewritten_amplitudes,
                           s.passes, s.segments, s.restart_gate, s.gates, s.hbm_bytes,
                           s.device_ms)
