"""CPU tests of the drop-in boundary: libqtask_b200.so loads, exports every
symbol include/qtask_c.h declares (and nothing else), and fails loudly --
never silently on a CPU path -- when no GPU is present."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2210_01076_b200 as qb
from paper_2210_01076_b200 import _ffi
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qtask_c.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qt_[a-z0-9_]+)\s*\(", txt)))


def exported_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", _ffi.LIB_PATH], check=True,
                         capture_output=True, text=True).stdout
    return sorted({line.split()[-1] for line in out.splitlines() if " T " in line})


def test_library_loads():
    assert qb.lib() is not None
    assert b"sm_100a" in qb.lib().qt_version()


def test_every_header_function_is_exported():
    hdr = header_functions()
    exp = set(exported_symbols())
    missing = [f for f in hdr if f not in exp]
    assert not missing, missing
    assert sorted(_ffi.HEADER_SYMBOLS) == hdr


def test_only_c_abi_is_exported():
    for sym in exported_symbols():
        assert sym.startswith("qt_"), sym


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _ffi.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly():
    if qb.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(qb.errors.NoDeviceError):
        qb.StateVector(4)
    with pytest.raises(qb.errors.NoDeviceError):
        qb.Simulator(3)


def test_host_only_planner_works_without_gpu():
    js = qb.plan_probe(6, gate_array([gate(K.H, q) for q in range(6)]))
    assert '"kind":"tile"' in js


def test_status_codes_map_to_reference_exceptions():
    from paper_2210_01076_b200 import errors
    assert errors.from_code(-2, "x").__class__ is errors.NetConflictError
    assert errors.from_code(-7, "x").__class__ is errors.StaleStateError
    assert errors.from_code(-8, "x").__class__ is errors.NumericError
    assert issubclass(errors.NoDeviceError, errors.Error)


def test_bad_gate_rejected_by_planner():
    with pytest.raises(qb.errors.BadQubitError):
        qb.plan_probe(3, gate_array([gate(K.H, 5)]))
    with pytest.raises(qb.errors.BadQubitError):
        qb.plan_probe(3, gate_array([gate(K.Cnot, 1, 1)]))
    bad = gate_array([gate(K.Rx, 0, theta=float("nan"))])
    with pytest.raises(qb.errors.Error):
        qb.plan_probe(3, bad)


def test_gate_struct_layout():
    assert _ffi.GATE_DTYPE.itemsize == 40
    assert ctypes.sizeof(_ffi.QtConfig) == 48


def test_config_block_size_validated_like_the_reference():
    """validate_config (plan.cpp:7-13): non power of two (incl. 0) -> Error,
    before any device work."""
    from paper_2210_01076_b200 import Config, Error, Simulator
    for bs in (0, 1, 3, 384):
        with pytest.raises(Error):
            Simulator(4, Config(block_size=bs))


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_net_order_index_matches_a_plain_array(seed):
    """csrc/qt_netindex.hpp (O(log nets) positions) against an array walk."""
    assert _ffi.netindex_audit(seed, 3000) == 0
