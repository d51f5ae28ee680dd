"""The sharded (one-rank-per-GPU) path on one GPU: an in-process group of
emulated ranks (RankGroup, csrc/qt_comm.hpp LocalComm) runs every rank's real
State::exchange step loop, the kernels with their rank offsets
(gbase_hi = rank << nlocal) and the fixed-order norm combine -- the code NCCL
mode runs, with device copies instead of NCCL send/recv. Checked against the
oracle (oracle/, pinned to the reference oracle.cpp:15-50) and bit-for-bit
against the loopback shards (same plan, bit-swap exchanges)."""
import numpy as np
import pytest

import oracle
from paper_2210_01076_b200 import RankGroup, StateVector, workloads as W
from paper_2210_01076_b200.gates import lower_to_reference
from tests.test_planner import random_circuit

pytestmark = pytest.mark.gpu

TOL = 1e-10
NORM_TOL = 1e-12


def run_group(n, gates, world, compiled=False, basis=0):
    g = RankGroup(n, world, compiled=compiled)
    try:
        g.set_basis(basis)
        g.apply(gates)
        nrm = g.norm_squared()
        psi = g.read()
        stats = g.stats()
    finally:
        g.close()
    return psi, nrm, stats


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_family_n26_vs_oracle(gpu, world):
    """BASELINE config 4's circuit family (1500 gates, 30% on the top 3
    qubits) at 26 qubits on 2 / 4 / 8 ranks."""
    w = W.config4(n=26)
    want = oracle.simulate(w.n, lower_to_reference(w.gates))
    got, nrm, stats = run_group(w.n, w.gates, world)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1.0) <= NORM_TOL
    # the plan exchanged qubits, and every rank moved the same bytes
    assert stats[0]["swaps"] > 0 and stats[0]["exchanged_bytes"] > 0
    assert len({s["exchanged_bytes"] for s in stats}) == 1


@pytest.mark.parametrize("world,scheme", [(2, "two"), (8, "two"), (4, "tmp"), (8, "tmp")])
def test_group_bitwise_equals_loopback(gpu, world, scheme, monkeypatch):
    """Same plan, same per-amplitude operations: the group's rank-offset
    kernels + transport must give exactly the loopback shards' state, with
    either exchange scheme (two-buffer, or receive buffer + copy back:
    QTB_EXCHANGE_TMP=1)."""
    if scheme == "tmp":
        monkeypatch.setenv("QTB_EXCHANGE_TMP", "1")
    w = W.config4(n=22, ngates=600)
    got, nrm, stats = run_group(w.n, w.gates, world)
    # local HBM copy traffic of the exchanges: the own region only (two) or
    # every received region copied back (tmp)
    k_sent = stats[0]["exchanged_bytes"]
    if scheme == "two":
        # 2 x own region per exchange: a 1/(2^k - 1) share of what was sent
        if world == 2:
            assert stats[0]["exchange_local_bytes"] == 2 * k_sent
        else:
            assert stats[0]["exchange_local_bytes"] < 2 * k_sent
    else:
        assert stats[0]["exchange_local_bytes"] == 2 * k_sent
    lb = StateVector(w.n, mode="loopback", shards=world)
    lb.apply(w.gates)
    want = lb.read()
    lb.close()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("world", [2, 4])
def test_group_compiled_passes(gpu, world):
    w = W.config4(n=24, ngates=800)
    want = oracle.simulate(w.n, lower_to_reference(w.gates))
    got, nrm, _ = run_group(w.n, w.gates, world, compiled=True)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1.0) <= NORM_TOL


@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_exchange_equals_send_recv(gpu, world, monkeypatch):
    """Compiled mode on a transport with peer memory fuses every exchange into
    the pass before it (the pass stores each amplitude straight to the rank
    and index it has after the exchange): no exchange step, no local copy
    traffic, and bit for bit the state of the send/recv path
    (QTB_FUSE_EXCHANGE=0) -- both against the oracle."""
    w = W.config4(n=22, ngates=600)
    want = oracle.simulate(w.n, lower_to_reference(w.gates))
    fused, nrm, stats = run_group(w.n, w.gates, world, compiled=True)
    assert np.abs(fused - want).max() <= TOL
    assert abs(nrm - 1.0) <= NORM_TOL
    assert stats[0]["swaps"] > 0
    # exchanges whose preceding pass is a compiled tile pass are fused
    assert stats[0]["fused_exchanges"] > 0
    assert len({s["fused_exchanges"] for s in stats}) == 1
    monkeypatch.setenv("QTB_FUSE_EXCHANGE", "0")
    plain, nrm2, stats2 = run_group(w.n, w.gates, world, compiled=True)
    assert stats2[0]["fused_exchanges"] == 0
    assert stats2[0]["swaps"] == stats[0]["swaps"]
    assert stats2[0]["exchanged_bytes"] == stats[0]["exchanged_bytes"]
    assert stats[0]["exchange_local_bytes"] < stats2[0]["exchange_local_bytes"]
    assert np.array_equal(fused, plain)
    assert nrm == nrm2


@pytest.mark.parametrize("seed", range(6))
def test_group_random_circuits(gpu, seed):
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(8, 15))
    world = [2, 4, 8][seed % 3]
    g = random_circuit(rng, n, int(rng.integers(40, 300)))
    basis = int(rng.integers(0, 1 << n))
    want = oracle.simulate(n, g, basis=basis)
    got, nrm, _ = run_group(n, g, world, basis=basis)
    assert np.abs(got - want).max() <= TOL
    assert abs(nrm - 1.0) <= NORM_TOL


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_top_k_matches_one_gpu(gpu, world):
    """top_k on a sharded state: every rank selects in its shard (in logical
    index order), the ranks all-gather and merge; same list (indices and the
    stored amplitudes) as selecting from the gathered state, on every rank --
    after a circuit with exchanges, so the qubit map is not the identity."""
    from tests.test_gpu_topk import expected
    w = W.config4(n=20, ngates=400)
    g = RankGroup(w.n, world)
    try:
        g.apply(w.gates)
        psi = g.read()
        for k in (1, 50, 3000):
            idx, amps = g.top_k(k)
            want_i, want_a = expected(psi, k)
            assert (idx == want_i).all()
            assert (amps == want_a).all()
    finally:
        g.close()


def test_sharded_top_k_ties(gpu):
    """Every |a|^2 equal (H on every qubit, then exchanges through a CX ladder
    on the top qubits): the ties break by logical index across shards."""
    from paper_2210_01076_b200.gates import GateKind as K, gate, gate_array
    from tests.test_gpu_topk import expected
    n = 16
    rows = [gate(K.H, q) for q in range(n)] + [gate(K.Rx, n - 1, -1, 0.0), gate(K.H, n - 1), gate(K.H, n - 1)]
    g = RankGroup(n, 4)
    try:
        g.apply(gate_array(rows))
        psi = g.read()
        for k in (1, 100, 5000):
            idx, amps = g.top_k(k)
            want_i, _ = expected(psi, k)
            assert (idx == want_i).all()
    finally:
        g.close()
