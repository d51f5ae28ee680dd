"""Multi-process (world_size 2 and 4, gloo, CPU) test of the sharded path's
host logic: the planner's exchange insertion for global (sharded) qubits and
the exchange semantics of State::exchange (qt_state.cpp) -- each rank sends
the region of its shard whose victim local bits equal the partner's global
bits and receives the partner's matching region in place. Tile passes are
replayed per shard by tests/emulator.py with global-index predicates
(controls / diagonals on global qubits act without communication). The
gathered, un-permuted state must equal the dense oracle."""
import json
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2210_01076_b200 import plan_probe, workloads as W
from tests.emulator import _bit, apply_plan, logical_view
from tests.test_planner import random_circuit, random_state


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def exchange_gloo(psi, pairs, rank, nlocal):
    """Restates the NCCL exchange of qt_state.cpp (State::exchange)."""
    k = len(pairs)
    gbit = [g - nlocal for g, _ in pairs]
    vbit = [v for _, v in pairs]
    rho = sum(((rank >> gbit[j]) & 1) << j for j in range(k))
    loc = np.arange(len(psi), dtype=np.uint64)
    reqs, bufs = [], []
    for c in range(1 << k):
        if c == rho:
            continue
        partner = rank
        for j in range(k):
            partner = (partner & ~(1 << gbit[j])) | (((c >> j) & 1) << gbit[j])
        sel = np.ones(len(psi), dtype=bool)
        for j in range(k):
            sel &= _bit(loc, vbit[j]) == ((c >> j) & 1)
        region = np.nonzero(sel)[0]
        send = torch.from_numpy(np.ascontiguousarray(psi[region]).view(np.float64))
        recv = torch.empty_like(send)
        reqs.append(dist.isend(send, partner))
        reqs.append(dist.irecv(recv, partner))
        bufs.append((region, send, recv))
    for r in reqs:
        r.wait()
    out = psi.copy()
    for region, _, recv in bufs:
        out[region] = recv.numpy().view(np.complex128)
    return out


def _worker(rank, world, port, n, gates, psi0, want, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        g = int(math.log2(world))
        nlocal = n - g
        plan = json.loads(plan_probe(n, gates, global_qubits=g, tile_qubits=5, detail=True))
        assert any(p["kind"] == "exchange" for p in plan["passes"])
        shard = psi0[rank << nlocal:(rank + 1) << nlocal]
        out = apply_plan(shard, plan, base=rank << nlocal,
                         exchange=lambda s, pairs: exchange_gloo(s, pairs, rank, nlocal))
        t = torch.from_numpy(out.view(np.float64).copy())
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        if rank == 0:
            full = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            got = logical_view(full, plan["perm_after"])
            q.put(float(np.abs(got - want).max()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 0), (2, 1), (4, 2), (4, 3)])
def test_sharded_plan_over_gloo(world, seed):
    rng = np.random.default_rng(900 + seed)
    n = 10
    gates = random_circuit(rng, n, 120)
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, gates, state=psi0.copy(), threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, gates, psi0, want, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=5) <= 1e-12


def test_config4_shape_plan_exchanges():
    """C4 (30% of gates on the 3 global qubits): exchanges only bring global
    qubits local for non-diagonal targets; diagonal gates and controls on
    global qubits never trigger one."""
    w = W.config4(n=16, ngates=400)
    plan = json.loads(plan_probe(16, w.gates, global_qubits=3))
    ex = [p for p in plan["passes"] if p["kind"] == "exchange"]
    assert 0 < len(ex) < 150
    for p in ex:
        for g, v in p["swap"]:
            assert g >= 13 and v < 13
