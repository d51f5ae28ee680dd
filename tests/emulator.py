"""Test-only numpy replay of a detailed pass plan (qt_plan_probe_ex JSON).

Independent of the CUDA kernels: it re-derives each encoded device op's
physical action from the tile / register-slot encoding and applies it to a
full state vector, so planner legality (hoisting, rounds) and op encoding
are checked against the dense oracle on the CPU. Exchanges are bit swaps.
"""
from __future__ import annotations

import json

import numpy as np

(D_DENSE, D_REAL, D_DIAG, D_SIGN, D_XPERM, D_ANTI, D_SWAP2, D_PHASE1) = range(8)
D_LAYER = 9


def _bit(idx, pos):
    return (idx >> np.uint64(pos)) & np.uint64(1)


def _signs(psi, terms, slot, idx, tile):
    """Sign terms [slots, lcond, gcond]: negate where the slot is in `slots`
    and the tile bits `lcond` / global bits `gcond` are all 1."""
    neg = np.zeros(len(psi), dtype=bool)
    for slots, lcond, gcond in terms:
        on = np.ones(len(psi), dtype=bool)
        for tb in range(len(tile)):
            if (lcond >> tb) & 1:
                on &= _bit(idx, tile[tb]) == 1
        for pb in range(64):
            if (gcond >> pb) & 1:
                on &= _bit(idx, pb) == 1
        neg ^= on & (((slots >> slot) & 1) == 1)
    return np.where(neg, -psi, psi)


def apply_plan(state: np.ndarray, plan_json: str, base: int = 0, exchange=None) -> np.ndarray:
    """Replays the plan on `state`. For one shard of a sharded state, `base`
    is the shard's global index offset (rank << nlocal: predicates see global
    indices) and `exchange(psi, pairs)` performs the exchange passes."""
    plan = json.loads(plan_json) if isinstance(plan_json, str) else plan_json
    psi = state.copy()
    nl = int(len(psi)).bit_length() - 1
    idx = np.uint64(base) + np.arange(1 << nl, dtype=np.uint64)  # global indices
    for ps in plan["passes"]:
        if ps["kind"] == "exchange" and exchange is not None:
            psi = exchange(psi, ps["swap"])
            continue
        if ps["kind"] == "exchange":
            for g, v in ps["swap"]:
                sel = (_bit(idx, g) == 1) & (_bit(idx, v) == 0)
                a = idx[sel]
                b = a ^ np.uint64((1 << g) | (1 << v))
                psi[a], psi[b] = psi[b].copy(), psi[a].copy()
            continue
        tile = ps["tile"]
        for rd in ps["round_detail"]:
            reg = rd["reg"]
            # slot index of every amplitude in this round
            slot = np.zeros(len(psi), dtype=np.int64)
            for i, tb in enumerate(reg):
                slot |= (_bit(idx, tile[tb]).astype(np.int64) << i)
            for op in rd["ops"]:
                # [type, a, cs, ds, lmask, gmask, dl, dg, [data]]: a = target
                # register slot (MULTI: slot mask), cs / ds = control /
                # diagonal-target slot (-1: not a register bit; SWAP2 keeps
                # its second slot in ds); data = the op's pool slice
                typ, a, cs, ds, lmask, gmask, dl, dg = (int(x) for x in op[:8])
                data = op[8]
                b = ds
                if typ == D_LAYER:
                    # a layer: [table][sign terms] then one 2x2 per slot in a
                    # (op[9] table flag, op[10] table, op[11] sign terms)
                    if int(op[9]):
                        tab = np.array(op[10][0::2]) + 1j * np.array(op[10][1::2])
                        psi = psi * tab[slot]
                    psi = _signs(psi, op[11], slot, idx, tile)
                    # rotations (c, s) on the slots in a, then complex 2x2s
                    # on the slots in lmask (op[4])
                    mats = []
                    k = 0
                    for sl in range(len(reg)):
                        if (a >> sl) & 1:  # rotation [[c, -s], [s, c]]
                            c, sn = data[k], data[k + 1]
                            mats.append((sl, np.array([c, -sn, sn, c], dtype=np.complex128)))
                            k += 2
                    for sl in range(len(reg)):
                        if (lmask >> sl) & 1:
                            mm = np.array(data[k:k + 8])
                            mats.append((sl, mm[0::2] + 1j * mm[1::2]))
                            k += 8
                    for sl, mm in mats:
                        t = tile[reg[sl]]
                        lo = np.nonzero(_bit(idx, t) == 0)[0]
                        hi = lo | (1 << t)
                        x, y = psi[lo].copy(), psi[hi].copy()
                        psi[lo] = mm[0] * x + mm[1] * y
                        psi[hi] = mm[2] * x + mm[3] * y
                    continue
                m = np.array(data[0:8], dtype=np.float64)
                m = m[0::2] + 1j * m[1::2]
                # control predicate over physical bits
                ok = np.ones(len(psi), dtype=bool)
                if cs >= 0:
                    ok &= _bit(idx, tile[reg[cs]]) == 1
                for tb in range(len(tile)):
                    if (lmask >> tb) & 1:
                        ok &= _bit(idx, tile[tb]) == 1
                for pb in range(64):
                    if (gmask >> pb) & 1:
                        ok &= _bit(idx, pb) == 1
                if typ in (D_DENSE, D_REAL, D_XPERM, D_ANTI):
                    t = tile[reg[a]]
                    lo = np.nonzero((_bit(idx, t) == 0) & ok)[0]
                    hi = lo | (1 << t)
                    x, y = psi[lo].copy(), psi[hi].copy()
                    if typ in (D_DENSE, D_REAL):
                        if typ == D_REAL:
                            m = m.real.astype(np.complex128)
                        psi[lo] = m[0] * x + m[1] * y
                        psi[hi] = m[2] * x + m[3] * y
                    elif typ == D_XPERM:
                        psi[lo], psi[hi] = y, x
                    else:
                        psi[lo] = m[1] * y
                        psi[hi] = m[2] * x
                elif typ in (D_DIAG, D_SIGN, D_PHASE1):
                    if ds >= 0:
                        bit = _bit(idx, tile[reg[ds]]) == 1
                    elif dl:
                        tb = int(dl).bit_length() - 1
                        bit = _bit(idx, tile[tb]) == 1
                    else:
                        bit = _bit(idx, int(dg).bit_length() - 1) == 1
                    if typ == D_SIGN:
                        f = np.where(bit, -1.0, 1.0)
                    elif typ == D_PHASE1:
                        f = np.where(bit, m[3], 1.0)
                    else:
                        f = np.where(bit, m[3], m[0])
                    psi = np.where(ok, psi * f, psi)
                elif typ == D_SWAP2:
                    ta, tb2 = tile[reg[a]], tile[reg[b]]
                    sel = (_bit(idx, ta) == 1) & (_bit(idx, tb2) == 0)
                    p0 = np.nonzero(sel)[0]
                    p1 = p0 ^ ((1 << ta) | (1 << tb2))
                    psi[p0], psi[p1] = psi[p1].copy(), psi[p0].copy()
                else:
                    raise ValueError(f"unknown op type {typ}")
    return psi


def logical_view(psi: np.ndarray, perm_after) -> np.ndarray:
    """Maps a physical state (logical qubit q at physical bit perm[q]) back to
    logical index order."""
    n = int(len(psi)).bit_length() - 1
    idx = np.arange(1 << n, dtype=np.uint64)
    phys = np.zeros_like(idx)
    for q in range(n):
        phys |= _bit(idx, q) << np.uint64(perm_after[q])
    return psi[phys]
