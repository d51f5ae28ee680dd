"""Host-only handle on the reference-unit partition model (qt_pm_*,
csrc/qt_partition.hpp): the restatement of the reference's partition DAG
that the incremental engine runs for UpdateStats and introspection, driven
directly by modifier events (no device). For differential tests against the
reference engine and for locality studies."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _ffi
from ._ffi import check, lib


class PartitionModel:
    def __init__(self, num_qubits: int, block_size: int = 256):
        self._h = ctypes.c_void_p()
        check(lib().qt_pm_create(num_qubits, block_size, ctypes.byref(self._h)))
        self.n = num_qubits

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().qt_pm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def insert_net(self, net: int, where: str = "back", after: int = 0):
        code = {"front": 0, "back": 1, "after": 2}[where]
        check(lib().qt_pm_insert_net(self._h, net, code, after))

    def remove_net(self, net: int):
        check(lib().qt_pm_remove_net(self._h, net))

    def insert_gate(self, gate: int, kind: int, net: int, target: int, control: int = -1,
                    theta: float = 0.0, phi: float = 0.0, lam: float = 0.0):
        from .gates import gate as row, gate_array
        g = gate_array([row(kind, target, control, theta, phi, lam)])
        check(lib().qt_pm_insert_gate(self._h, gate, g.ctypes.data, net))

    def remove_gate(self, gate: int):
        check(lib().qt_pm_remove_gate(self._h, gate))

    def update(self):
        check(lib().qt_pm_update(self._h))

    def account(self) -> dict:
        a = _ffi.QtUpdateAccount()
        check(lib().qt_pm_account(self._h, ctypes.byref(a), None, 0))
        blocks = np.zeros(max(1, a.rewritten_block_count), dtype=np.uint64)
        check(lib().qt_pm_account(self._h, ctypes.byref(a), blocks.ctypes.data, len(blocks)))
        return dict(full=bool(a.full), executed_partitions=int(a.executed_partitions),
                    materialized_blocks=int(a.materialized_blocks),
                    rewritten_amplitudes=int(a.rewritten_amplitudes),
                    rewritten_blocks=[int(b) for b in blocks[:a.rewritten_block_count]])

    def dump_graph(self) -> str:
        need = ctypes.c_size_t(0)
        check(lib().qt_pm_dump_graph(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        check(lib().qt_pm_dump_graph(self._h, buf, need.value, ctypes.byref(need)))
        return buf.value.decode()
