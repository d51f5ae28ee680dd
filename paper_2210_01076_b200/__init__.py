"""B200-native qTask hot path (arXiv 2210.01076): fused sm_100a gate
application on a device-resident complex128 state vector plus the
incremental re-simulation engine, behind the reference's Simulator API.

The compute lives in ``libqtask_b200.so`` (CUDA, built in-tree by
``csrc/Makefile``); this package is the host mirror of the reference's
interface over its C ABI (``include/qtask_c.h``).
"""
from ._ffi import GATE_DTYPE, device_count, jit_probe, jit_stats, jit_wait, lib, plan_probe  # noqa: F401
from .errors import (BadQubitError, Error, InvalidPositionError,  # noqa: F401
                     NetConflictError, NumericError, StaleStateError,
                     SuperpositionGateError, UnknownGateError, UnknownNetError)
from .gates import GateKind, gate, gate_array, lower_to_reference  # noqa: F401
from .simulator import Config, Simulator, UpdateStats  # noqa: F401
from .state import RankGroup, StateVector, nccl_unique_id, probe_fp64  # noqa: F401

__all__ = ["GateKind", "Simulator", "Config", "StateVector", "gate", "gate_array"]
