"""Compiled tile passes (csrc/qt_jit.cpp): every lowered pass becomes one
straight-line NVRTC kernel.

CPU part (no device): the generated source of every pass of every config
family compiles for sm_100a, generation is deterministic, and the FP64
accounting of the lowering matches the layer content.
GPU part: compiled-mode states against the dense oracle / closed forms at
the same bar as the interpreter kernel (max |diff| <= 1e-10, norm 1e-12),
including sharded (loopback) plans with exchanges, and compiled vs
interpreted agreement plus the compile cache."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import StateVector, jit_probe, jit_stats, workloads as W
from paper_2210_01076_b200.gates import GateKind as K
from paper_2210_01076_b200.gates import gate, gate_array, lower_to_reference
from tests.test_planner import random_circuit, random_state

TOL = 1e-10
NORM_TOL = 1e-12


# ---------------------------------------------------------------- CPU ------

@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "random"])
def test_generated_passes_compile(name):
    w = {"c1": lambda: W.config1(),
         "c2": lambda: W.config2(n=12),
         "c3": lambda: W.config3(n=14, layers=4),
         "c4": lambda: W.config4(n=14, ngates=60),
         "c5": lambda: W.config5(n=14, ngates=80, nmods=0),
         "random": lambda: None}[name]()
    if w is None:
        rng = np.random.default_rng(3)
        n, gates = 10, random_circuit(rng, 10, 60)
    else:
        n, gates = w.n, w.gates
    js = json.loads(jit_probe(n, gates, compile=True))
    assert js["passes"] >= 1
    # every lowered pass compiles; the config families lower completely
    # (random circuits with SWAP / off-register diagonals keep generic passes)
    assert js["compiled"] == js["lowered"]
    if name != "random":
        assert js["lowered"] >= 1 and js["cubin_bytes"] > 0


_VARIANT_SCRIPT = """
import json, sys
sys.path.insert(0, %r)
from paper_2210_01076_b200 import workloads as W
from paper_2210_01076_b200._ffi import jit_probe
out = []
for w in (W.config3(n=16, layers=3), W.config5(n=16, ngates=120, nmods=0)):
    js = json.loads(jit_probe(w.n, w.gates, tile_qubits=12, reg_bits=4, compile=True))
    src = jit_probe(w.n, w.gates, tile_qubits=12, reg_bits=4, source_pass=0)
    out.append({"lowered": js["lowered"], "compiled": js["compiled"], "fuse": "fx.peer[" in src and "fx.rfix" in src,
                "bulk": "cp.async.bulk.global.shared::cta" in src})
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{"QTB_PROBE_FUSE": "13,12"}, {"QTB_PROBE_FUSE": "13,12,5"},
                                 {"QTB_JIT_TMA": "1"}, {"QTB_JIT_TMA": "2"}, {"QTB_JIT_EARLY": "0"},
                                 {"QTB_SHRINK_MIN": "10"}])
def test_ring_kernel_variants_compile(env):
    """The ring kernel's variants keep compiling for sm_100a (each in its own
    process: the switches are read once): the fused-exchange stores (victim
    bits on outer, thread and register positions), the two TMA-store
    experiments, the late refill and the shrunk tiles."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    run = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT % root], capture_output=True, text=True,
                         env=dict(os.environ, QTB_JIT_CACHE_DIR="off", **env), timeout=600)
    assert run.returncode == 0, run.stderr[-2000:]
    for rec in json.loads(run.stdout.strip().splitlines()[-1]):
        assert rec["lowered"] >= 1 and rec["compiled"] == rec["lowered"]
        if "QTB_PROBE_FUSE" in env:
            assert rec["fuse"]
        if env.get("QTB_JIT_TMA"):
            assert rec["bulk"]


_DISK_SCRIPT = """
import json, sys
sys.path.insert(0, %r)
from paper_2210_01076_b200 import workloads as W
from paper_2210_01076_b200._ffi import jit_probe, jit_stats
w = W.config3(n=14, layers=4)
js = json.loads(jit_probe(w.n, w.gates, compile=True))
print(json.dumps({"probe": js, "stats": jit_stats()}))
"""


def test_persistent_cubin_cache(tmp_path):
    """A second process finds every compiled pass on disk (no NVRTC run), an
    entry whose stored source differs is ignored, and "off" disables it."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(cache_dir):
        env = dict(os.environ, QTB_JIT_CACHE_DIR=cache_dir)
        out = subprocess.run([sys.executable, "-c", _DISK_SCRIPT % root], env=env, check=True,
                             capture_output=True, text=True).stdout
        return json.loads(out.strip().splitlines()[-1])

    d = str(tmp_path / "cubins")
    a = run(d)
    n = a["probe"]["compiled"]
    # (jit_probe runs twice per call: size query, then fill -- the second
    # run of the first process already finds its own entries)
    assert n >= 1 and a["stats"]["disk_hits"] == n and a["stats"]["disk_writes"] == n
    files = sorted(os.listdir(d))
    assert len(files) == n and all(f.endswith(".qtc") for f in files)
    b = run(d)
    assert b["stats"]["disk_hits"] == 2 * n and b["stats"]["disk_writes"] == 0
    assert b["probe"]["cubin_bytes"] == a["probe"]["cubin_bytes"]
    # corrupt one entry's stored source: it must be recompiled, not trusted
    path = os.path.join(d, files[0])
    blob = bytearray(open(path, "rb").read())
    blob[200] ^= 0x20
    open(path, "wb").write(bytes(blob))
    c = run(d)
    assert c["stats"]["disk_hits"] == 2 * n - 1 and c["stats"]["disk_writes"] == 1
    off = run("off")
    assert off["stats"]["disk_hits"] == 0 and off["stats"]["disk_writes"] == 0


def test_source_is_deterministic_and_literal():
    w = W.config3(n=14, layers=3)
    a = jit_probe(w.n, w.gates, source_pass=0)
    b = jit_probe(w.n, w.gates, source_pass=0)
    assert a == b
    assert 'extern "C" __global__' in a and "qtjit" in a
    # constants are hex-float literals, no pool reads
    assert "pool" not in a and "0x1." in a


def test_fp64_accounting_layered():
    """A layer of RY rotations on every qubit of a 12-qubit state: one scaled
    rotation (2 FP64 / amplitude) per qubit, no tables; the product of the
    rotations' scales is folded into one complex table at the end (4)."""
    n = 12
    g = gate_array([gate(K.Ry, q, -1, 0.1 + q) for q in range(n)])
    js = json.loads(jit_probe(n, g, tile_qubits=12, reg_bits=3, low_bits=3))
    assert js["fp64_per_amp"] == pytest.approx(2.0 * n + 4.0)


# ---------------------------------------------------------------- GPU ------

def run(n, gates, psi0=None, **kw):
    st = StateVector(n, compiled=True, **kw)
    if psi0 is not None:
        st.write(psi0)
    st.apply(gates)
    out = st.read()
    nrm = st.norm_squared()
    st.close()
    return out, nrm


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_compiled_random_vs_oracle(gpu, seed):
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.integers(4, 17))
    g = random_circuit(rng, n, int(rng.integers(20, 250)))
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, g, state=psi0.copy())
    for tile in (0, 6):
        got, nrm = run(n, g, psi0, tile_qubits=tile)
        assert np.abs(got - want).max() <= TOL
        assert abs(nrm - 1) <= NORM_TOL


@pytest.mark.gpu
def test_compiled_config_families(gpu):
    w = W.config1()
    got, nrm = run(w.n, w.gates)
    assert np.abs(got - oracle.simulate(w.n, lower_to_reference(w.gates))).max() <= TOL
    w = W.config2(n=20)
    got, nrm = run(20, w.gates)
    assert np.abs(got - W.qft_closed_form(20, w.basis)).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL
    w = W.config3(n=20, layers=20)
    got, nrm = run(20, w.gates)
    assert np.abs(got - oracle.simulate(20, w.gates)).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL
    w = W.config5(n=18, ngates=600, nmods=0)
    got, _ = run(18, w.gates)
    assert np.abs(got - oracle.simulate(18, w.gates)).max() <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("shards", [2, 8])
def test_compiled_sharded_loopback(gpu, shards):
    w = W.config4(n=18, ngates=300)
    want = oracle.simulate(18, w.gates)
    got, nrm = run(18, w.gates, mode="loopback", shards=shards)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL


@pytest.mark.gpu
def test_compiled_matches_interpreted_and_caches(gpu):
    w = W.config3(n=22, layers=8)
    st = StateVector(22)
    st.apply(w.gates)
    ref = st.read()
    st.close()
    got, _ = run(22, w.gates)
    assert np.abs(got - ref).max() <= 1e-12
    before = jit_stats()
    got2, _ = run(22, w.gates)           # same circuit: every pass from the cache
    after = jit_stats()
    assert after["compiled"] == before["compiled"]
    assert after["cache_hits"] > before["cache_hits"]
    assert got2.tobytes() == got.tobytes()


@pytest.mark.gpu
def test_plan_search_window_plan_vs_oracle(gpu):
    """From 24 local qubits the compiled mode searches plans (FP64 caps x
    {first-need greedy, window search}, then the beam over the window choices):
    on the layered config the window plan wins and needs fewer passes than the
    greedy one; its state must match the oracle (C3 family at 24 q, ~10 s of
    multithreaded oracle)."""
    w = W.config3(n=24, layers=20)
    st = StateVector(24, compiled=True)
    st.apply(w.gates)
    searched = st.stats()["passes"]
    got = st.read()
    nrm = st.norm_squared()
    st.close()
    want = oracle.simulate(24, lower_to_reference(w.gates), threads=os.cpu_count() or 1)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1) <= NORM_TOL
    os.environ["QTB_PLAN_SEARCH"] = "0"
    try:
        st = StateVector(24, compiled=True)
        st.apply(w.gates)
        greedy = st.stats()["passes"]
        got2 = st.read()
        st.close()
    finally:
        del os.environ["QTB_PLAN_SEARCH"]
    assert np.abs(got2 - want).max() <= TOL
    assert searched < greedy, (searched, greedy)


@pytest.mark.gpu
def test_config3_full_size_two_independent_paths(gpu, monkeypatch):
    """The headline config at its full 30 qubits through two device paths that
    share no plan, tile geometry or kernel: the compiled ring passes of the
    searched plan (R = 4, 2^12 tiles, window + beam) and the layer-word
    interpreter on the first-need greedy plan (R = 3, 2^10 tiles,
    QTB_PLAN_SEARCH=0). 2^18 amplitudes sampled in 64 runs across the state
    and the norms must agree to 1e-12 (each path matches the oracle at 24
    qubits in test_plan_search_window_plan_vs_oracle / test_gpu_state)."""
    w = W.config3()
    rng = np.random.default_rng(30)
    starts = np.sort(rng.integers(0, (1 << 30) - (1 << 12), size=64))

    def sample(st):
        return np.concatenate([st.read(int(a), 1 << 12) for a in starts])

    st = StateVector(30, compiled=True)
    st.apply(w.gates)
    a, na, pa = sample(st), st.norm_squared(), st.stats()["passes"]
    st.close()
    monkeypatch.setenv("QTB_PLAN_SEARCH", "0")
    st = StateVector(30, compiled=False)
    st.apply(w.gates)
    b, nb, pb = sample(st), st.norm_squared(), st.stats()["passes"]
    st.close()
    assert pa < pb
    assert np.abs(a - b).max() <= 1e-12
    assert abs(na - 1) <= NORM_TOL and abs(nb - 1) <= NORM_TOL
    assert np.abs(a).max() > 0


@pytest.mark.gpu
def test_compiled_config3_full_size_mirror(gpu):
    """The headline config at its full size (30 q, 16 GiB) in compiled mode:
    C then C^dagger returns |0...0> (no CPU state needed), norm after C."""
    from tests.test_gpu_state import inverse
    w = W.config3()
    st = StateVector(30, compiled=True)
    st.apply(w.gates)
    nrm = st.norm_squared()
    st.apply(inverse(w.gates))
    head = st.read(0, 1 << 12)
    nrm2 = st.norm_squared()
    st.close()
    assert abs(nrm - 1) <= NORM_TOL and abs(nrm2 - 1) <= NORM_TOL
    assert abs(head[0] - 1) <= TOL and np.abs(head[1:]).max() <= TOL


@pytest.mark.gpu
def test_hybrid_compiled_bitwise_equals_interpreter(gpu):
    """Hybrid mode: the first apply runs every pass on the interpreter kernel
    while the passes compile in the background; once they are cached the
    same apply runs compiled. Both paths do the same FP64 operations in the
    same order, so the states are bit-identical (the incremental engine's
    results do not depend on the cache state)."""
    from paper_2210_01076_b200 import jit_wait
    w = W.config3(n=20, layers=12)
    st = StateVector(20, compiled=2)
    st.apply(w.gates)
    first = st.read()
    assert jit_wait(300)
    before = jit_stats()
    st.set_basis(0)
    st.apply(w.gates)
    second = st.read()
    after = jit_stats()
    st.close()
    assert after["cache_hits"] > before["cache_hits"]
    assert first.tobytes() == second.tobytes()
    assert np.abs(first - oracle.simulate(20, w.gates)).max() <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("compiled", [0, 1])
def test_repeated_apply_reuses_plan(gpu, compiled):
    """apply() of the previous gate list reuses its plan (and compiled passes);
    a different list, or a changed state, is planned afresh -- results stay
    those of the oracle either way."""
    rng = np.random.default_rng(77)
    n = 14
    a = random_circuit(rng, n, 120, kinds=[K.H, K.Rx, K.Ry, K.Rz, K.Cnot, K.Cz, K.T])
    b = random_circuit(rng, n, 90, kinds=[K.H, K.Ry, K.Cnot, K.S])
    st = StateVector(n, compiled=compiled)
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1
    for g in (a, a, b, a, b, b):
        st.apply(g)
        psi = oracle.simulate(n, g, state=psi)
        assert np.abs(st.read() - psi).max() <= TOL
    st.close()
