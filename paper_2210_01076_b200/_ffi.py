"""ctypes binding of libqtask_b200.so (include/qtask_c.h).

The product path: every call goes through the in-tree CUDA library. There
is no CPU fallback -- if the library is missing the import fails loudly, and
calls that need a GPU return QT_ERR_NO_DEVICE (raised as NoDeviceError).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqtask_b200.so")
if os.environ.get("QTB_LIB"):  # tuning builds only (tools/); product = in-tree .so
    LIB_PATH = os.path.join(HERE, os.environ["QTB_LIB"])

# qt_gate (40 bytes): int32 kind, target, control, reserved; f64 theta, phi, lambda
GATE_DTYPE = np.dtype(
    [("kind", "<i4"), ("target", "<i4"), ("control", "<i4"), ("reserved", "<i4"),
     ("theta", "<f8"), ("phi", "<f8"), ("lam", "<f8")], align=False)
assert GATE_DTYPE.itemsize == 40


class QtUpdateAccount(ctypes.Structure):
    """qt_update_account: UpdateStats in the reference's units (partition
    model, csrc/qt_partition.hpp)."""
    _fields_ = [("valid", ctypes.c_int32), ("full", ctypes.c_int32),
                ("executed_partitions", ctypes.c_uint64), ("materialized_blocks", ctypes.c_uint64),
                ("rewritten_amplitudes", ctypes.c_uint64), ("rewritten_block_count", ctypes.c_uint64)]


class QtConfig(ctypes.Structure):
    _fields_ = [("block_size", ctypes.c_uint64), ("threads", ctypes.c_uint32),
                ("device", ctypes.c_int32), ("tile_qubits", ctypes.c_int32),
                ("max_checkpoints", ctypes.c_int32),
                ("checkpoint_fraction", ctypes.c_double),
                ("segment_gates", ctypes.c_int32), ("compiled", ctypes.c_int32),
                ("partition_model", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class QtRunStats(ctypes.Structure):
    _fields_ = [("full", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("executed_partitions", ctypes.c_uint64),
                ("rewritten_amplitudes", ctypes.c_uint64), ("gates", ctypes.c_uint64),
                ("passes", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("hbm_bytes", ctypes.c_uint64), ("exchanged_bytes", ctypes.c_uint64),
                ("swaps", ctypes.c_uint64), ("restart_gate", ctypes.c_uint64),
                ("segments", ctypes.c_uint64), ("device_ms", ctypes.c_double),
                ("plan_ms", ctypes.c_double), ("exchange_local_bytes", ctypes.c_uint64),
                ("fused_exchanges", ctypes.c_uint64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_
                if not name.startswith("reserved")}


# Every symbol include/qtask_c.h declares (checked by tests/test_abi.py).
HEADER_SYMBOLS = [
    "qt_last_error", "qt_device_count", "qt_version",
    "qt_state_create", "qt_state_create_sharded", "qt_state_create_loopback",
    "qt_group_create", "qt_group_destroy", "qt_state_create_group",
    "qt_nccl_unique_id", "qt_state_destroy", "qt_state_num_qubits", "qt_set_basis",
    "qt_write", "qt_read", "qt_apply", "qt_norm_squared", "qt_sync", "qt_last_stats",
    "qt_checkpoint_save", "qt_checkpoint_restore", "qt_plan_json", "qt_plan_probe", "qt_jit_probe", "qt_jit_stats", "qt_jit_disk_stats", "qt_jit_pending",
    "qt_sim_create", "qt_sim_destroy", "qt_sim_num_qubits", "qt_sim_block_size",
    "qt_sim_total_blocks", "qt_sim_insert_net_front", "qt_sim_insert_net_back",
    "qt_sim_insert_net_after", "qt_sim_remove_net", "qt_sim_insert_gate",
    "qt_sim_remove_gate", "qt_sim_update_state", "qt_sim_pending", "qt_sim_amplitude",
    "qt_sim_amplitudes", "qt_sim_norm_squared", "qt_sim_last_update",
    "qt_sim_num_gates", "qt_sim_num_nets", "qt_sim_net_order", "qt_sim_net_gates",
    "qt_sim_gate_info", "qt_sim_export_gates", "qt_qasm_parse", "qt_qasm_build",
    "qt_exchange_schedule", "qt_top_k", "qt_sim_top_k", "qt_netindex_audit", "qt_fused_exchange_map",
    "qt_sim_update_account", "qt_sim_model_snapshot", "qt_sim_node_name", "qt_sim_dump_graph",
    "qt_gate_matrix", "qt_classify_gate",
    "qt_pm_create", "qt_pm_destroy", "qt_pm_insert_net", "qt_pm_remove_net", "qt_pm_insert_gate",
    "qt_pm_remove_gate", "qt_pm_update", "qt_pm_account", "qt_pm_dump_graph",
]

_lib = None

_c = ctypes
_vp = _c.c_void_p
_SIGS = {
    "qt_last_error": ([], _c.c_char_p),
    "qt_version": ([], _c.c_char_p),
    "qt_device_count": ([_c.POINTER(_c.c_int)], _c.c_int),
    "qt_state_create": ([_c.c_int, _vp, _c.POINTER(_vp)], _c.c_int),
    "qt_state_create_sharded": ([_c.c_int, _c.c_int, _c.c_int, _vp, _vp,
                                 _c.POINTER(_vp)], _c.c_int),
    "qt_state_create_loopback": ([_c.c_int, _c.c_int, _vp, _c.POINTER(_vp)], _c.c_int),
    "qt_group_create": ([_c.c_int, _c.POINTER(_vp)], _c.c_int),
    "qt_group_destroy": ([_vp], _c.c_int),
    "qt_state_create_group": ([_c.c_int, _vp, _c.c_int, _vp, _c.POINTER(_vp)], _c.c_int),
    "qt_nccl_unique_id": ([_vp], _c.c_int),
    "qt_pm_create": ([_c.c_int, _c.c_uint64, _c.POINTER(_vp)], _c.c_int),
    "qt_pm_destroy": ([_vp], _c.c_int),
    "qt_pm_insert_net": ([_vp, _c.c_uint32, _c.c_int, _c.c_uint32], _c.c_int),
    "qt_pm_remove_net": ([_vp, _c.c_uint32], _c.c_int),
    "qt_pm_insert_gate": ([_vp, _c.c_uint32, _vp, _c.c_uint32], _c.c_int),
    "qt_pm_remove_gate": ([_vp, _c.c_uint32], _c.c_int),
    "qt_pm_update": ([_vp], _c.c_int),
    "qt_pm_account": ([_vp, _vp, _vp, _c.c_size_t], _c.c_int),
    "qt_pm_dump_graph": ([_vp, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_sim_update_account": ([_vp, _vp, _vp, _c.c_size_t], _c.c_int),
    "qt_sim_dump_graph": ([_vp, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_sim_node_name": ([_vp, _c.c_uint64, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_gate_matrix": ([_c.c_int, _c.c_double, _c.c_double, _c.c_double, _vp, _c.POINTER(_c.c_int)], _c.c_int),
    "qt_classify_gate": ([_c.c_int, _c.c_double, _c.c_double, _c.c_double], _c.c_int),
    "qt_state_destroy": ([_vp], _c.c_int),
    "qt_state_num_qubits": ([_vp], _c.c_int),
    "qt_set_basis": ([_vp, _c.c_uint64], _c.c_int),
    "qt_write": ([_vp, _c.c_uint64, _c.c_uint64, _vp], _c.c_int),
    "qt_read": ([_vp, _c.c_uint64, _c.c_uint64, _vp], _c.c_int),
    "qt_apply": ([_vp, _vp, _c.c_size_t], _c.c_int),
    "qt_norm_squared": ([_vp, _c.POINTER(_c.c_double)], _c.c_int),
    "qt_sync": ([_vp], _c.c_int),
    "qt_last_stats": ([_vp, _c.POINTER(QtRunStats)], _c.c_int),
    "qt_checkpoint_save": ([_vp, _c.c_int], _c.c_int),
    "qt_checkpoint_restore": ([_vp, _c.c_int], _c.c_int),
    "qt_plan_json": ([_vp, _vp, _c.c_size_t, _c.c_char_p, _c.c_size_t,
                      _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_plan_probe": ([_c.c_int, _c.c_int, _c.c_int, _vp, _c.c_size_t, _c.c_char_p,
                       _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_plan_probe_ex": ([_c.c_int, _c.c_int, _c.c_int, _c.c_int, _vp, _c.c_size_t,
                          _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_jit_probe": ([_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _vp,
                      _c.c_size_t, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_jit_stats": ([_c.POINTER(_c.c_uint64), _c.POINTER(_c.c_uint64), _c.POINTER(_c.c_double)],
                     _c.c_int),
    "qt_jit_pending": ([_c.POINTER(_c.c_uint64)], _c.c_int),
    "qt_jit_disk_stats": ([_c.POINTER(_c.c_uint64), _c.POINTER(_c.c_uint64)], _c.c_int),
    "qt_state_stream": ([_vp], _vp),
    "qt_set_timing": ([_vp, _c.c_int], _c.c_int),
    "qt_last_timings": ([_vp, _vp, _vp, _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_probe_fp64": ([_c.c_int, _c.POINTER(_c.c_double)], _c.c_int),
    "qt_sim_create": ([_c.c_int, _vp, _c.POINTER(_vp)], _c.c_int),
    "qt_sim_destroy": ([_vp], _c.c_int),
    "qt_sim_num_qubits": ([_vp], _c.c_int),
    "qt_sim_block_size": ([_vp], _c.c_uint64),
    "qt_sim_total_blocks": ([_vp], _c.c_uint64),
    "qt_sim_insert_net_front": ([_vp, _c.POINTER(_c.c_uint32)], _c.c_int),
    "qt_sim_insert_net_back": ([_vp, _c.POINTER(_c.c_uint32)], _c.c_int),
    "qt_sim_insert_net_after": ([_vp, _c.c_uint32, _c.POINTER(_c.c_uint32)], _c.c_int),
    "qt_sim_remove_net": ([_vp, _c.c_uint32], _c.c_int),
    "qt_sim_insert_gate": ([_vp, _c.c_int, _vp, _c.c_uint32, _c.c_int, _c.c_int,
                            _c.POINTER(_c.c_uint32)], _c.c_int),
    "qt_sim_remove_gate": ([_vp, _c.c_uint32], _c.c_int),
    "qt_sim_update_state": ([_vp], _c.c_int),
    "qt_sim_pending": ([_vp], _c.c_int),
    "qt_sim_amplitude": ([_vp, _c.c_uint64, _vp], _c.c_int),
    "qt_sim_amplitudes": ([_vp, _c.c_uint64, _c.c_uint64, _vp], _c.c_int),
    "qt_sim_norm_squared": ([_vp, _c.POINTER(_c.c_double)], _c.c_int),
    "qt_sim_last_update": ([_vp, _c.POINTER(QtRunStats)], _c.c_int),
    "qt_sim_num_gates": ([_vp], _c.c_size_t),
    "qt_sim_num_nets": ([_vp], _c.c_size_t),
    "qt_sim_net_order": ([_vp, _vp, _c.c_size_t], _c.c_int),
    "qt_sim_net_gates": ([_vp, _c.c_uint32, _vp, _c.c_size_t, _c.POINTER(_c.c_size_t)],
                         _c.c_int),
    "qt_sim_gate_info": ([_vp, _c.c_uint32, _vp, _c.POINTER(_c.c_uint32)], _c.c_int),
    "qt_sim_export_gates": ([_vp, _vp, _c.c_size_t, _c.POINTER(_c.c_size_t)], _c.c_int),
    "qt_qasm_parse": ([_c.c_char_p, _c.c_size_t, _vp, _c.c_size_t, _c.POINTER(_c.c_size_t),
                       _c.POINTER(_c.c_uint32), _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)],
                      _c.c_int),
    "qt_qasm_build": ([_vp, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_int),
                       _c.POINTER(_c.c_int)], _c.c_int),
    "qt_top_k": ([_vp, _c.c_uint64, _vp, _vp, _c.POINTER(_c.c_uint64)], _c.c_int),
    "qt_sim_top_k": ([_vp, _c.c_uint64, _vp, _vp, _c.POINTER(_c.c_uint64)], _c.c_int),
    "qt_fused_exchange_map": ([_c.c_int, _c.c_int, _c.c_int, _vp, _vp, _vp, _c.POINTER(_c.c_uint64)], _c.c_int),
    "qt_netindex_audit": ([_c.c_uint64, _c.c_uint32, _c.POINTER(_c.c_uint64)], _c.c_int),
    "qt_exchange_schedule": ([_c.c_int, _c.c_int, _c.c_int, _vp, _vp, _c.c_uint64, _vp,
                              _c.c_size_t, _c.POINTER(_c.c_size_t),
                              _c.POINTER(_c.c_uint64)], _c.c_int),
}


def lib():
    """Loads libqtask_b200.so. Raises ImportError if it is not built --
    there is deliberately no fallback implementation."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2210_01076_b200/csrc)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int) -> int:
    if rc < 0:
        msg = lib().qt_last_error().decode("utf-8", "replace")
        raise errors.from_code(rc, msg)
    return rc


def make_config(block_size=256, threads=0, device=-1, tile_qubits=0, max_checkpoints=0,
                checkpoint_fraction=0.0, segment_gates=0, compiled=False,
                partition_model=0) -> QtConfig:
    cfg = QtConfig()
    cfg.block_size = block_size
    cfg.threads = threads
    cfg.device = device
    cfg.tile_qubits = tile_qubits
    cfg.max_checkpoints = max_checkpoints
    cfg.checkpoint_fraction = checkpoint_fraction
    cfg.segment_gates = segment_gates
    cfg.compiled = int(compiled) if not isinstance(compiled, bool) else (1 if compiled else 0)
    cfg.partition_model = partition_model
    return cfg


def device_count() -> int:
    n = ctypes.c_int(0)
    check(lib().qt_device_count(ctypes.byref(n)))
    return n.value


def gates_array(gates) -> np.ndarray:
    return np.ascontiguousarray(gates, dtype=GATE_DTYPE)


def plan_probe(n: int, gates, global_qubits: int = 0, tile_qubits: int = 0,
               detail: bool = False) -> str:
    """Host-only pass plan (JSON) -- no GPU needed."""
    g = gates_array(gates)
    need = ctypes.c_size_t(0)
    d = 1 if detail else 0
    check(lib().qt_plan_probe_ex(n, global_qubits, tile_qubits, d, g.ctypes.data, len(g),
                                 None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    check(lib().qt_plan_probe_ex(n, global_qubits, tile_qubits, d, g.ctypes.data, len(g),
                                 buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def jit_probe(n: int, gates, tile_qubits: int = 0, reg_bits: int = 0, low_bits: int = 0,
              compile: bool = False, source_pass: int = -1) -> str:
    """Host-only compiled-pass probe (JSON stats, or one pass's CUDA source)
    -- no GPU needed; compile=True runs NVRTC on every pass."""
    g = gates_array(gates)
    need = ctypes.c_size_t(0)
    args = (n, tile_qubits, reg_bits, low_bits, 1 if compile else 0, source_pass, g.ctypes.data, len(g))
    check(lib().qt_jit_probe(*args, None, 0, ctypes.byref(need)))
    while True:
        # the text carries timings (compile_ms): its length can differ by a few
        # bytes between the sizing call and the filling one
        cap = need.value + 64
        buf = ctypes.create_string_buffer(cap)
        check(lib().qt_jit_probe(*args, buf, cap, ctypes.byref(need)))
        if need.value <= cap:
            return buf.value.decode()


def jit_stats() -> dict:
    """Process-wide compiled-pass statistics: passes compiled, cache hits and
    total NVRTC + load time."""
    c, h, ms = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_double(0.0)
    check(lib().qt_jit_stats(ctypes.byref(c), ctypes.byref(h), ctypes.byref(ms)))
    dh, dw = ctypes.c_uint64(0), ctypes.c_uint64(0)
    check(lib().qt_jit_disk_stats(ctypes.byref(dh), ctypes.byref(dw)))
    return {"compiled": c.value, "cache_hits": h.value, "compile_ms": ms.value,
            "disk_hits": dh.value, "disk_writes": dw.value}


def jit_wait(timeout_s: float = 120.0) -> bool:
    """Waits until no pass is queued or compiling in the background (hybrid
    mode); False on timeout."""
    import time
    n = ctypes.c_uint64(0)
    t_end = time.time() + timeout_s
    while True:
        check(lib().qt_jit_pending(ctypes.byref(n)))
        if n.value == 0:
            return True
        if time.time() > t_end:
            return False
        time.sleep(0.05)


def fused_exchange_map(rank: int, nlocal: int, pairs):
    """(peer ranks by victim-bit pattern, rfix) of a fused exchange on `rank`
    (qt_fused_exchange_map); pairs: (global bit above the local bits, victim bit)."""
    k = len(pairs)
    g = np.array([p[0] for p in pairs], dtype=np.int32)
    v = np.array([p[1] for p in pairs], dtype=np.int32)
    peers = np.zeros(1 << k, dtype=np.int32)
    rfix = ctypes.c_uint64(0)
    check(lib().qt_fused_exchange_map(rank, nlocal, k, g.ctypes.data, v.ctypes.data, peers.ctypes.data,
                                      ctypes.byref(rfix)))
    return peers, rfix.value


def netindex_audit(seed: int, ops: int) -> int:
    """Failed comparisons of the net order index against a plain array over
    `ops` seeded random operations (qt_netindex_audit; host only)."""
    bad = ctypes.c_uint64(0)
    check(lib().qt_netindex_audit(seed, ops, ctypes.byref(bad)))
    return bad.value


def exchange_schedule(rank: int, nlocal: int, pairs, tmp_amps: int):
    """The grouped send/recv steps of a sharded exchange on `rank`
    (qt_exchange_schedule): (rows [step, peer, send_off, recv_off], piece).
    pairs: (global bit index above the local bits, local victim bit)."""
    k = len(pairs)
    g = np.array([p[0] for p in pairs], dtype=np.int32)
    v = np.array([p[1] for p in pairs], dtype=np.int32)
    n = ctypes.c_size_t(0)
    piece = ctypes.c_uint64(0)
    check(lib().qt_exchange_schedule(rank, nlocal, k, g.ctypes.data, v.ctypes.data, tmp_amps,
                                     None, 0, ctypes.byref(n), ctypes.byref(piece)))
    rows = np.zeros((max(1, n.value), 4), dtype=np.uint64)
    check(lib().qt_exchange_schedule(rank, nlocal, k, g.ctypes.data, v.ctypes.data, tmp_amps,
                                     rows.ctypes.data, n.value, ctypes.byref(n),
                                     ctypes.byref(piece)))
    return rows[:n.value], piece.value
