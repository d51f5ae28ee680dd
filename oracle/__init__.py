"""TEST INFRASTRUCTURE ONLY -- the parity checkers for the B200 engine.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package. The product path
(``paper_2210_01076_b200``) never imports it and has no CPU fallback.

* :func:`oracle_lib` -- ``oracle/liboracle.so``: C restatement of the
  reference dense oracle (``/root/reference/proj/src/oracle.cpp:15-50``) and
  gate matrices (``gate.cpp:42-90``), bit-identical, multithreaded.
* :func:`ref_lib` -- ``oracle/_ref/libqtask_ref.so``: the unmodified
  reference library compiled from its own sources plus ``ref_shim.cpp``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqtask_ref.so")

# qt_gate layout (include/qtask_c.h): int32 kind, target, control, reserved;
# double theta, phi, lambda  -> 40 bytes.
GATE_DTYPE = np.dtype(
    [("kind", "<i4"), ("target", "<i4"), ("control", "<i4"), ("reserved", "<i4"),
     ("theta", "<f8"), ("phi", "<f8"), ("lam", "<f8")], align=False)
assert GATE_DTYPE.itemsize == 40

_oracle = None
_ref = None


def build(force: bool = False) -> None:
    """Compile the checkers (make -C oracle). The reference part is only
    compiled where /root/reference exists."""
    if force or not os.path.exists(ORACLE_SO) or (
            os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)


def oracle_lib():
    global _oracle
    if _oracle is None:
        build()
        lib = ctypes.CDLL(ORACLE_SO)
        lib.qo_apply.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_size_t, ctypes.c_int]
        lib.qo_apply.restype = ctypes.c_int
        lib.qo_init_basis.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64]
        lib.qo_norm_squared.argtypes = [ctypes.c_int, ctypes.c_void_p]
        lib.qo_norm_squared.restype = ctypes.c_double
        lib.qo_max_abs_diff.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        lib.qo_max_abs_diff.restype = ctypes.c_double
        lib.qo_gate_matrix.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
        lib.qo_gate_matrix.restype = ctypes.c_int
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (no /root/reference?)")
        lib = ctypes.CDLL(REF_SO)
        lib.ref_oracle_run.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
                                       ctypes.c_size_t, ctypes.c_void_p,
                                       ctypes.POINTER(ctypes.c_double)]
        lib.ref_oracle_run.restype = ctypes.c_int
        lib.ref_gate_matrix.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
        lib.ref_gate_matrix.restype = ctypes.c_int
        lib.ref_classify.argtypes = [ctypes.c_int, ctypes.c_double]
        lib.ref_classify.restype = ctypes.c_int
        lib.ref_sim_create.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint]
        lib.ref_sim_create.restype = ctypes.c_void_p
        lib.ref_sim_destroy.argtypes = [ctypes.c_void_p]
        lib.ref_sim_insert_net.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32]
        lib.ref_sim_insert_net.restype = ctypes.c_int64
        lib.ref_sim_remove_net.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
        lib.ref_sim_remove_net.restype = ctypes.c_int
        lib.ref_sim_insert_gate.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_uint32, ctypes.c_int, ctypes.c_int]
        lib.ref_sim_insert_gate.restype = ctypes.c_int64
        lib.ref_sim_remove_gate.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
        lib.ref_sim_remove_gate.restype = ctypes.c_int
        lib.ref_sim_update.argtypes = [ctypes.c_void_p]
        lib.ref_sim_update.restype = ctypes.c_int
        lib.ref_sim_amplitudes.argtypes = [ctypes.c_void_p, ctypes.c_uint64,
                                           ctypes.c_uint64, ctypes.c_void_p]
        lib.ref_sim_amplitudes.restype = ctypes.c_int
        lib.ref_sim_norm.argtypes = [ctypes.c_void_p]
        lib.ref_sim_norm.restype = ctypes.c_double
        lib.ref_sim_stats.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.ref_sim_dump.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]
        lib.ref_sim_dump.restype = ctypes.c_size_t
        lib.ref_sim_rewritten_blocks.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
        lib.ref_sim_rewritten_blocks.restype = ctypes.c_size_t
        lib.ref_qasm_parse.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.POINTER(ctypes.c_uint32),
                                       ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_int)]
        lib.ref_qasm_parse.restype = ctypes.c_int64
        lib.ref_qasm_build.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]
        lib.ref_qasm_build.restype = ctypes.c_int
        _ref = lib
    return _ref


def ref_qasm_parse(text: str):
    """The reference parser (qasm.cpp:34-405) on ``text``: ("ok", num_qubits,
    rows, levels) with rows = [kind, gate, theta, has_theta, q0, q1, line,
    column] per statement, or ("parse" | "unsupported", line, column)."""
    lib = ref_lib()
    data = text.encode("utf-8")
    cap = max(1, data.count(b";") + 1)
    rows = np.zeros((cap, 8), dtype=np.float64)
    levels = np.zeros(cap, dtype=np.int32)
    nq = ctypes.c_uint32(0)
    line, col = ctypes.c_int(0), ctypes.c_int(0)
    n = lib.ref_qasm_parse(data, len(data), rows.ctypes.data, levels.ctypes.data, cap,
                           ctypes.byref(nq), ctypes.byref(line), ctypes.byref(col))
    if n == -1:
        return ("parse", line.value, col.value)
    if n == -2:
        return ("unsupported", line.value, col.value)
    if n < 0:
        raise ValueError("reference qasm parser failed")
    return ("ok", nq.value, rows[:n], levels[:n])


def _gates_arg(gates: np.ndarray):
    gates = np.ascontiguousarray(gates, dtype=GATE_DTYPE)
    return gates, gates.ctypes.data


def simulate(n: int, gates: np.ndarray, basis: int = 0, threads: int | None = None,
             state: np.ndarray | None = None) -> np.ndarray:
    """Dense oracle (C restatement): returns the complex128 state after
    applying ``gates`` to |basis> (or in place to ``state``)."""
    lib = oracle_lib()
    if state is None:
        state = np.zeros(1 << n, dtype=np.complex128)
        state[basis] = 1.0
    if threads is None:
        threads = min(os.cpu_count() or 1, 64)
    g, p = _gates_arg(gates)
    rc = lib.qo_apply(n, state.ctypes.data, p, len(g), int(threads))
    if rc != 0:
        raise ValueError("oracle rejected the gate list")
    return state


def norm_squared(state: np.ndarray) -> float:
    n = int(len(state)).bit_length() - 1
    return oracle_lib().qo_norm_squared(n, np.ascontiguousarray(state).ctypes.data)


def gate_matrix(kind: int, theta: float = 0.0) -> np.ndarray:
    m = np.zeros(4, dtype=np.complex128)
    if oracle_lib().qo_gate_matrix(kind, float(theta), m.ctypes.data) != 0:
        raise ValueError("no 2x2 matrix for kind %d" % kind)
    return m.reshape(2, 2)


def ref_simulate(n: int, gates: np.ndarray, basis: int = 0):
    """The reference's own oracle::apply_gate_dense over the gate list.
    Returns (state, seconds of the gate loop)."""
    lib = ref_lib()
    out = np.empty(1 << n, dtype=np.complex128)
    secs = ctypes.c_double(0.0)
    g, p = _gates_arg(gates)
    rc = lib.ref_oracle_run(n, basis, p, len(g), out.ctypes.data, ctypes.byref(secs))
    if rc != 0:
        raise ValueError(f"reference oracle failed: {rc}")
    return out, secs.value


def ref_time_gates(n: int, gates: np.ndarray, basis: int = 0) -> float:
    """Seconds the reference oracle spends in its gate loop (no readout)."""
    lib = ref_lib()
    secs = ctypes.c_double(0.0)
    g, p = _gates_arg(gates)
    rc = lib.ref_oracle_run(n, basis, p, len(g), None, ctypes.byref(secs))
    if rc != 0:
        raise ValueError(f"reference oracle failed: {rc}")
    return secs.value


class RefSimulator:
    """Thin handle over the reference ``qtask::Simulator`` (engine.hpp:46-100)."""

    def __init__(self, n: int, block_size: int = 256, threads: int = 0):
        self.lib = ref_lib()
        self.h = self.lib.ref_sim_create(n, block_size, threads)
        if not self.h:
            raise ValueError("reference Simulator construction failed")
        self.n = n

    def close(self):
        if self.h:
            self.lib.ref_sim_destroy(self.h)
            self.h = None

    __del__ = close

    def _chk(self, rc):
        if rc < 0:
            raise RuntimeError(f"reference error {rc}")
        return rc

    def insert_net_front(self):
        return self._chk(self.lib.ref_sim_insert_net(self.h, 0, 0))

    def insert_net_back(self):
        return self._chk(self.lib.ref_sim_insert_net(self.h, 1, 0))

    def insert_net_after(self, after):
        return self._chk(self.lib.ref_sim_insert_net(self.h, 2, after))

    def remove_net(self, net):
        self._chk(self.lib.ref_sim_remove_net(self.h, net))

    def insert_gate(self, kind, net, target, control=-1, theta=0.0):
        return self._chk(self.lib.ref_sim_insert_gate(self.h, kind, theta, net, target,
                                                      control))

    def remove_gate(self, gate):
        self._chk(self.lib.ref_sim_remove_gate(self.h, gate))

    def update_state(self):
        self._chk(self.lib.ref_sim_update(self.h))

    def amplitudes(self, first=0, last=None):
        if last is None:
            last = (1 << self.n) - 1
        out = np.empty(last - first + 1, dtype=np.complex128)
        self._chk(self.lib.ref_sim_amplitudes(self.h, first, last, out.ctypes.data))
        return out

    def norm_squared(self):
        return self.lib.ref_sim_norm(self.h)

    def qasm_build(self, text: str):
        """qtask::qasm::build_circuit(parse(text)) on this handle."""
        data = text.encode("utf-8")
        self._chk(self.lib.ref_qasm_build(self.h, data, len(data)))

    def stats(self):
        out = np.zeros(4, dtype=np.uint64)
        self.lib.ref_sim_stats(self.h, out.ctypes.data)
        n = self.lib.ref_sim_rewritten_blocks(self.h, None, 0)
        blocks = np.zeros(max(1, n), dtype=np.uint64)
        self.lib.ref_sim_rewritten_blocks(self.h, blocks.ctypes.data, n)
        return dict(full=bool(out[0]), executed_partitions=int(out[1]),
                    materialized_blocks=int(out[2]), rewritten_amplitudes=int(out[3]),
                    rewritten_blocks=[int(b) for b in blocks[:n]])

    def dump_graph(self) -> str:
        need = self.lib.ref_sim_dump(self.h, None, 0)
        buf = ctypes.create_string_buffer(need)
        self.lib.ref_sim_dump(self.h, buf, need)
        return buf.value.decode()
