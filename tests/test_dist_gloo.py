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


def exchange_gloo_lib(psi, pairs, rank, nlocal, tmp_amps):
    """Runs the library's own exchange schedule (qt_exchange_schedule, the
    steps State::exchange issues to NCCL) with gloo send/recv: every step
    sends each peer's piece, receives into a buffer of tmp_amps amplitudes,
    then copies the received pieces over the sent ones."""
    from paper_2210_01076_b200._ffi import exchange_schedule
    rows, piece = exchange_schedule(rank, nlocal, [(g - nlocal, v) for g, v in pairs], tmp_amps)
    out = psi.copy()
    tmp = np.zeros(tmp_amps, dtype=np.complex128)
    for step in np.unique(rows[:, 0]):
        sel = rows[rows[:, 0] == step]
        reqs, bufs = [], []
        for _, peer, soff, roff in sel.tolist():
            send = torch.from_numpy(out[soff:soff + piece].view(np.float64).copy())
            recv = torch.empty_like(send)
            reqs += [dist.isend(send, int(peer)), dist.irecv(recv, int(peer))]
            bufs.append((soff, roff, recv))
        for r in reqs:
            r.wait()
        for soff, roff, recv in bufs:
            tmp[roff:roff + piece] = recv.numpy().view(np.complex128)
            out[soff:soff + piece] = tmp[roff:roff + piece]
    return out


def _worker(rank, world, port, n, gates, psi0, want, q, use_lib=False):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        g = int(math.log2(world))
        nlocal = n - g
        plan = json.loads(plan_probe(n, gates, global_qubits=g, tile_qubits=5, detail=True))
        assert any(p["kind"] == "exchange" for p in plan["passes"])
        shard = psi0[rank << nlocal:(rank + 1) << nlocal]
        if use_lib:  # small buffer: several pieces per run
            ex = lambda s, pairs: exchange_gloo_lib(s, pairs, rank, nlocal, 1 << (nlocal - 4))
        else:
            ex = lambda s, pairs: exchange_gloo(s, pairs, rank, nlocal)
        out = apply_plan(shard, plan, base=rank << nlocal, exchange=ex)
        t = torch.from_numpy(out.view(np.float64).copy())
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        if rank == 0:
            full = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            got = logical_view(full, plan["perm_after"])
            q.put(float(np.abs(got - want).max()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed,use_lib", [(2, 0, False), (2, 1, False), (4, 2, False),
                                                (4, 3, False), (2, 4, True), (4, 5, True)])
def test_sharded_plan_over_gloo(world, seed, use_lib):
    """use_lib: the exchanges run the library's NCCL step schedule
    (qt_exchange_schedule) instead of the restated region semantics."""
    rng = np.random.default_rng(900 + seed)
    n = 10
    gates = random_circuit(rng, n, 120)
    psi0 = random_state(rng, n)
    want = oracle.simulate(n, gates, state=psi0.copy(), threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, gates, psi0, want, q, use_lib))
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


@pytest.mark.parametrize("g,k,tmp_div", [(1, 1, 1), (2, 1, 8), (2, 2, 4), (3, 3, 16), (3, 2, 64)])
def test_exchange_schedule_all_ranks(g, k, tmp_div):
    """All ranks' schedules (qt_exchange_schedule) executed together in numpy
    swap the k chosen global bits with the k victim local bits of the whole
    vector -- the sharded exchange's index math, for any buffer size."""
    from paper_2210_01076_b200._ffi import exchange_schedule
    rng = np.random.default_rng(17 * g + k)
    nlocal = 9
    world = 1 << g
    gsel = sorted(rng.choice(g, k, replace=False).tolist())
    vsel = sorted(rng.choice(nlocal, k, replace=False).tolist())
    full = rng.normal(size=world << nlocal) + 1j * rng.normal(size=world << nlocal)
    shards = [full[r << nlocal:(r + 1) << nlocal].copy() for r in range(world)]
    tmp = max(1, (1 << nlocal) // tmp_div)
    scheds = [exchange_schedule(r, nlocal, list(zip(gsel, vsel)), tmp) for r in range(world)]
    new = [s.copy() for s in shards]
    for r, (rows, piece) in enumerate(scheds):
        for _, peer, soff, roff in rows.tolist():
            # what `peer` sends to r in the matching step: its row addressed to r
            prow = scheds[peer][0]
            mine = [x for x in prow.tolist() if x[1] == r]
            # pieces are matched by order: the i-th piece r sends to peer pairs
            # with the i-th piece peer sends to r
            idx = [x for x in rows.tolist() if x[1] == peer].index([_, peer, soff, roff])
            src = mine[idx][2]
            new[r][soff:soff + piece] = shards[peer][src:src + piece]
    got = np.concatenate(new)
    idx = np.arange(world << nlocal)
    perm = idx.copy()
    for gb, vb in zip(gsel, vsel):
        G = nlocal + gb
        bg, bv = (perm >> G) & 1, (perm >> vb) & 1
        perm = perm & ~((1 << G) | (1 << vb)) | (bg << vb) | (bv << G)
    want = full[perm]
    assert np.abs(got - want).max() == 0.0


def _fused_worker(rank, world, port, nlocal, pairs, seed, q):
    """Every rank scatters its shard as the fused pass would (amplitude x goes
    to rank peer[v(x)], index (x & ~V) | rfix, from the library's own map) and
    compares what it receives with the send/recv exchange of the same shards."""
    from paper_2210_01076_b200._ffi import fused_exchange_map
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        rng = np.random.default_rng(seed + rank)
        shard = rng.normal(size=1 << nlocal) + 1j * rng.normal(size=1 << nlocal)
        want = exchange_gloo(shard, pairs, rank, nlocal)
        peers, rfix = fused_exchange_map(rank, nlocal, [(g - nlocal, v) for g, v in pairs])
        x = np.arange(1 << nlocal, dtype=np.uint64)
        vmask = 0
        vpat = np.zeros(1 << nlocal, dtype=np.int64)
        for i, (_, vb) in enumerate(pairs):
            vmask |= 1 << vb
            vpat |= (((x >> np.uint64(vb)) & np.uint64(1)).astype(np.int64) << i)
        dest_rank = peers[vpat]
        dest_idx = (x & np.uint64(~vmask & ((1 << nlocal) - 1))) | np.uint64(rfix)
        # the "peer stores": one (indices, values) message per destination rank
        send = []
        for r in range(world):
            sel = dest_rank == r
            idx = dest_idx[sel].astype(np.int64)
            val = shard[sel]
            send.append(torch.from_numpy(np.concatenate([idx.astype(np.float64), val.view(np.float64)])))
        # ragged messages: exchanged pairwise (sizes first)
        got = np.zeros(1 << nlocal, dtype=np.complex128)
        filled = np.zeros(1 << nlocal, dtype=bool)
        for r in range(world):
            if r == rank:
                msg = send[r]
            else:
                n_out = torch.tensor([len(send[r])], dtype=torch.int64)
                n_in = torch.zeros(1, dtype=torch.int64)
                reqs = [dist.isend(n_out, r), dist.irecv(n_in, r)]
                for rq in reqs:
                    rq.wait()
                msg = torch.empty(int(n_in.item()), dtype=torch.float64)
                reqs = []
                if len(send[r]):
                    reqs.append(dist.isend(send[r], r))
                if len(msg):
                    reqs.append(dist.irecv(msg, r))
                for rq in reqs:
                    rq.wait()
            m = msg.numpy()
            cnt = len(m) // 3
            idx = m[:cnt].astype(np.int64)
            got[idx] = m[cnt:].view(np.complex128)
            assert not filled[idx].any()
            filled[idx] = True
        assert filled.all()
        q.put((rank, bool(np.array_equal(got, want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,pairs", [(2, [(8, 7)]), (2, [(8, 2)]), (4, [(9, 7), (8, 3)]), (4, [(9, 0)]),
                                         (8, [(10, 7), (9, 6), (8, 1)])])
def test_fused_exchange_map_equals_send_recv(world, pairs):
    """The destination map of the fused exchange (qt_fused_exchange_map: what
    the compiled pass's stores follow) moves every amplitude exactly where the
    send/recv exchange does, on every rank of a gloo world."""
    nlocal = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, nlocal, pairs, 77, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(res[r] for r in range(world)), res
