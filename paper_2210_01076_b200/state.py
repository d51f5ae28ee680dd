"""Device-resident state vector (qt_state_* of include/qtask_c.h)."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _ffi
from ._ffi import check, lib


class StateVector:
    """2^n complex128 amplitudes in HBM, gates applied by fused sm_100a tile
    passes.

    mode: "single" (one GPU), "loopback" (``shards`` emulated ranks on one
    GPU, exchanges by device copies) or "sharded" (one rank of a
    ``world``-GPU state, NCCL exchanges; pass ``rank``, ``world``, ``nccl_id``)
    or "group" (rank ``rank`` of an in-process RankGroup: the sharded kernels and
    exchange schedule with an in-process transport; see RankGroup).
    compiled=True runs every tile pass as its own NVRTC-compiled straight-line
    kernel (cached process-wide by the pass's content: for circuits applied more
    than once); compiled=2: hybrid (cached passes compiled, the others on the
    interpreter while they compile in the background).
    """

    def __init__(self, num_qubits: int, mode: str = "single", shards: int = 1,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 device: int = -1, tile_qubits: int = 0, compiled: bool = False,
                 group: "RankGroup | None" = None):
        self._h = ctypes.c_void_p()
        cfg = _ffi.make_config(device=device, tile_qubits=tile_qubits, compiled=compiled)
        if mode == "single":
            check(lib().qt_state_create(num_qubits, ctypes.byref(cfg), ctypes.byref(self._h)))
        elif mode == "loopback":
            check(lib().qt_state_create_loopback(num_qubits, shards, ctypes.byref(cfg),
                                                 ctypes.byref(self._h)))
        elif mode == "group":
            if group is None:
                raise ValueError("group mode needs a RankGroup")
            self._group = group  # keeps the group alive
            check(lib().qt_state_create_group(num_qubits, group.handle, rank, ctypes.byref(cfg),
                                              ctypes.byref(self._h)))
        elif mode == "sharded":
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("sharded mode needs the 128-byte NCCL unique id")
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            check(lib().qt_state_create_sharded(num_qubits, rank, world, idbuf,
                                                ctypes.byref(cfg), ctypes.byref(self._h)))
        else:
            raise ValueError(mode)
        self.n = num_qubits
        self.mode = mode

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().qt_state_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def stream_ptr(self) -> int:
        return lib().qt_state_stream(self._h) or 0

    def set_basis(self, index: int = 0):
        check(lib().qt_set_basis(self._h, index))

    def apply(self, gates: np.ndarray):
        g = _ffi.gates_array(gates)
        check(lib().qt_apply(self._h, g.ctypes.data, len(g)))

    def write(self, amps: np.ndarray, first: int = 0):
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        check(lib().qt_write(self._h, first, len(a), a.ctypes.data))

    def read(self, first: int = 0, count: int | None = None, out: np.ndarray | None = None):
        if count is None:
            count = (1 << self.n) - first
        if out is None:
            out = np.empty(count, dtype=np.complex128)
        check(lib().qt_read(self._h, first, count, out.ctypes.data))
        return out

    def top_k(self, k: int):
        """(indices, amplitudes) of the k largest |a|^2, largest first, ties by
        smaller index -- selected on the device (qt_top_k)."""
        k = min(int(k), 1 << self.n)
        idx = np.empty(max(1, k), dtype=np.uint64)
        amps = np.empty(max(1, k), dtype=np.complex128)
        cnt = ctypes.c_uint64(0)
        check(lib().qt_top_k(self._h, k, idx.ctypes.data, amps.ctypes.data, ctypes.byref(cnt)))
        return idx[:cnt.value], amps[:cnt.value]

    def norm_squared(self) -> float:
        v = ctypes.c_double(0.0)
        check(lib().qt_norm_squared(self._h, ctypes.byref(v)))
        return v.value

    def sync(self):
        check(lib().qt_sync(self._h))

    def stats(self) -> dict:
        s = _ffi.QtRunStats()
        check(lib().qt_last_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def set_timing(self, on: bool = True):
        check(lib().qt_set_timing(self._h, 1 if on else 0))

    def last_timings(self):
        """[(kind, ms)] per launch of the last apply (0 = tile pass,
        1 = exchange); needs set_timing(True) before the apply."""
        cnt = ctypes.c_size_t(0)
        check(lib().qt_last_timings(self._h, None, None, 0, ctypes.byref(cnt)))
        kinds = np.zeros(cnt.value, dtype=np.int32)
        ms = np.zeros(cnt.value, dtype=np.float32)
        check(lib().qt_last_timings(self._h, kinds.ctypes.data, ms.ctypes.data, cnt.value,
                                    ctypes.byref(cnt)))
        return list(zip(kinds.tolist(), ms.tolist()))

    def checkpoint_save(self, slot: int):
        check(lib().qt_checkpoint_save(self._h, slot))

    def checkpoint_restore(self, slot: int):
        check(lib().qt_checkpoint_restore(self._h, slot))

    def plan_json(self, gates: np.ndarray) -> str:
        g = _ffi.gates_array(gates)
        need = ctypes.c_size_t(0)
        check(lib().qt_plan_json(self._h, g.ctypes.data, len(g), None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        check(lib().qt_plan_json(self._h, g.ctypes.data, len(g), buf, need.value,
                                 ctypes.byref(need)))
        return buf.value.decode()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().qt_nccl_unique_id(buf))
    return buf.raw


def probe_fp64(device: int = 0) -> float:
    """Measured FP64 FMA instructions per second of the device."""
    v = ctypes.c_double(0.0)
    check(lib().qt_probe_fp64(device, ctypes.byref(v)))
    return v.value


class RankGroup:
    """An in-process group of ``world`` emulated ranks of one sharded state
    (qt_group_create / qt_state_create_group): the same kernels, rank offsets,
    exchange schedule and norm combine as one-process-per-GPU NCCL sharding,
    with the exchanges as device-to-device copies between the ranks' buffers
    (csrc/qt_comm.hpp LocalComm). Every collective call (apply with exchanges,
    norm_squared) must be made by all ranks concurrently: ``run`` calls a
    function on every rank, each on its own host thread (ctypes releases the
    GIL during the native calls)."""

    def __init__(self, num_qubits: int, world: int, device: int = -1, tile_qubits: int = 0,
                 compiled: bool = False):
        self._g = ctypes.c_void_p()
        check(lib().qt_group_create(world, ctypes.byref(self._g)))
        self.n = num_qubits
        self.world = world
        self.ranks = [StateVector(num_qubits, mode="group", rank=r, device=device,
                                  tile_qubits=tile_qubits, compiled=compiled, group=self)
                      for r in range(world)]

    @property
    def handle(self):
        return self._g

    def run(self, fn):
        """[fn(rank_state) for every rank], concurrently; re-raises the first error."""
        import threading
        out = [None] * self.world
        errs = [None] * self.world

        def go(r):
            try:
                out[r] = fn(self.ranks[r])
            except BaseException as e:  # reported to the caller
                errs[r] = e

        th = [threading.Thread(target=go, args=(r,)) for r in range(self.world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        # the root cause first: a rank whose peers failed reports "a peer
        # rank failed: ..." (in-process transport), so prefer another error
        first = [e for e in errs if e is not None]
        root = [e for e in first if "peer rank failed" not in str(e)]
        if first:
            raise (root or first)[0]
        return out

    def set_basis(self, index: int = 0):
        self.run(lambda st: st.set_basis(index))

    def apply(self, gates: np.ndarray):
        self.run(lambda st: st.apply(gates))

    def top_k(self, k: int):
        """The k largest-|amplitude|^2 basis states of the sharded state
        (collective: every rank selects in its shard, the ranks all-gather
        and merge); every rank returns the same list."""
        vals = self.run(lambda st: st.top_k(k))
        for v in vals[1:]:
            assert np.array_equal(v[0], vals[0][0]) and np.array_equal(v[1], vals[0][1]), \
                "ranks disagree on the top-k list"
        return vals[0]

    def norm_squared(self) -> float:
        vals = self.run(lambda st: st.norm_squared())
        assert all(v == vals[0] for v in vals), "ranks disagree on the norm"
        return vals[0]

    def read(self, first: int = 0, count: int | None = None) -> np.ndarray:
        """Logical amplitudes [first, first+count): each rank fills the ones it
        holds (zeros elsewhere), summed here."""
        if count is None:
            count = (1 << self.n) - first
        acc = np.zeros(count, dtype=np.complex128)
        buf = np.empty(count, dtype=np.complex128)
        for st in self.ranks:
            st.read(first, count, buf)
            acc += buf
        return acc

    def stats(self):
        return [st.stats() for st in self.ranks]

    def close(self):
        for st in getattr(self, "ranks", []):
            st.close()
        self.ranks = []
        if getattr(self, "_g", None) and self._g.value:
            lib().qt_group_destroy(self._g)
            self._g = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
