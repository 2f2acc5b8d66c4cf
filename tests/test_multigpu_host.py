"""Multi-GPU host logic on the CPU: world sizes 2-4 over gloo.

paper_1406_2628_b200.multigpu runs the joint K-ary split search (one
all_reduce per step), the exchange plan and all_to_all_single exchange
exactly as on the GPU box; only the local merge/sort -- the device kernels,
tested in test_gpu_parity.py -- is replaced by the C restatement here.
Every rank's output slice is checked against the oracle's full merge.
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _np(S, t):
    from oracle.bindings import ELEMENT_DTYPE
    x = t.numpy()
    if S == "el":
        return x.view(ELEMENT_DTYPE)
    if S == "f32":
        return x.view(np.uint32)
    return x


def _t(S, x):
    if S == "el":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy())
    if S == "f32":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.float32).copy())
    return torch.from_numpy(np.ascontiguousarray(x).copy())


def _oracle_merge(S):
    from oracle import bindings as B
    P = B.port()

    def merge(a, b, av, bv, kt):
        out, outv, _, _ = P.merge(S, _np(S, a), _np(S, b),
                                  av=av.numpy() if av is not None else None,
                                  bv=bv.numpy() if bv is not None else None)
        return _t(S, out), (torch.from_numpy(outv) if outv is not None else None)
    return merge


def _oracle_sort(S):
    from oracle import bindings as B
    P = B.port()

    def sort(x, v, kt):
        out, outv, _ = P.merge_sort(S, _np(S, x), vals=v.numpy() if v is not None else None)
        return _t(S, out), (torch.from_numpy(outv) if outv is not None else None)
    return sort


def _keys(S, rng, n, dup):
    from oracle.bindings import ELEMENT_DTYPE
    if S == "el":
        e = np.zeros(n, dtype=ELEMENT_DTYPE)
        e["key"] = rng.integers(-dup, dup, n)
        e["tag"] = np.arange(n, dtype=np.uint32)
        return e
    if S == "f32":
        x = (rng.integers(-dup, dup, n) / 3.0).astype(np.float32)
        x[rng.random(n) < 0.1] = -0.0
        return x.view(np.uint32)
    dt = {"u32": np.uint32, "i32": np.int32, "u64": np.uint64, "i64": np.int64}[S]
    if np.dtype(dt).kind == "u":
        return rng.integers(0, dup, n).astype(dt)
    return rng.integers(-dup, dup, n).astype(dt)


def _sort_keys(S, x):
    from oracle import bindings as B
    out, _, _ = B.port().merge_sort(S, x)
    return out


def _split(n, sizes_seed, world):
    rng = np.random.default_rng(sizes_seed)
    cuts = np.sort(rng.integers(0, n + 1, world - 1))
    return np.concatenate([[0], cuts, [n]]).astype(np.int64)


def _worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1406_2628_b200 import _native as N
        from paper_1406_2628_b200 import multigpu as mg
        S, na, nb, dup, vals, op = case
        kt = {"u32": N.KEY_U32, "i32": N.KEY_I32, "f32": N.KEY_F32, "u64": N.KEY_U64,
              "i64": N.KEY_I64, "el": N.KEY_ELEMENT}[S]
        rng = np.random.default_rng(1234)
        if op == "merge":
            a = _sort_keys(S, _keys(S, rng, na, dup))
            b = _sort_keys(S, _keys(S, rng, nb, dup))
            ca, cb = _split(na, 1, world), _split(nb, 2, world)
            av = np.arange(na, dtype=np.uint32)
            bv = np.arange(nb, dtype=np.uint32) | np.uint32(1 << 31)
            al, bl = a[ca[rank]:ca[rank + 1]], b[cb[rank]:cb[rank + 1]]
            kw = {}
            if vals:
                kw = dict(a_vals=torch.from_numpy(av[ca[rank]:ca[rank + 1]].copy()),
                          b_vals=torch.from_numpy(bv[cb[rank]:cb[rank + 1]].copy()))
            k, v = mg.sharded_merge(_t(S, al), _t(S, bl), key_type=kt,
                                    local_merge=_oracle_merge(S), **kw)
        else:
            x = _keys(S, rng, na, dup)
            cx = _split(na, 3, world)
            xv = np.arange(na, dtype=np.uint32)
            xl = x[cx[rank]:cx[rank + 1]]
            k, v = mg.sharded_sort(_t(S, xl), key_type=kt,
                                   vals=torch.from_numpy(xv[cx[rank]:cx[rank + 1]].copy())
                                   if vals else None,
                                   local_sort=_oracle_sort(S), local_merge=_oracle_merge(S))
        q.put((rank, _np(S, k).tobytes(), v.numpy().tobytes() if v is not None else None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, "ERR", traceback.format_exc() + str(e)))


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, k, v = q.get(timeout=300)
        assert k != "ERR", v
        res[r] = (k, v)
    for p in procs:
        p.join(timeout=60)
    return res


def _expected(case):
    from oracle import bindings as B
    P = B.port()
    S, na, nb, dup, vals, op = case
    rng = np.random.default_rng(1234)
    if op == "merge":
        a = _sort_keys(S, _keys(S, rng, na, dup))
        b = _sort_keys(S, _keys(S, rng, nb, dup))
        av = np.arange(na, dtype=np.uint32)
        bv = np.arange(nb, dtype=np.uint32) | np.uint32(1 << 31)
        out, outv, _, _ = P.merge(S, a, b, av=av if vals else None, bv=bv if vals else None)
        return out, outv
    x = _keys(S, rng, na, dup)
    out, outv, _ = P.merge_sort(S, x, vals=np.arange(na, dtype=np.uint32) if vals else None)
    return out, outv


def _check(world, case):
    from oracle.bindings import DTYPES
    S = case[0]
    res = _run(world, case)
    want_k, want_v = _expected(case)
    got_k = np.frombuffer(b"".join(res[r][0] for r in range(world)), dtype=DTYPES[S])
    if S == "el":
        assert np.array_equal(got_k["key"], want_k["key"])
        assert np.array_equal(got_k["tag"], want_k["tag"])
    else:
        assert got_k.tobytes() == want_k.tobytes()
    if case[4]:
        got_v = np.frombuffer(b"".join(res[r][1] for r in range(world)), dtype=np.uint32)
        assert np.array_equal(got_v, want_v)
    if case[5] == "merge":  # rank r owns exactly S[floor(rN/P), floor((r+1)N/P))
        n = case[1] + case[2]
        for r in range(world):
            assert len(res[r][0]) // DTYPES[S].itemsize == (r + 1) * n // world - r * n // world


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_merge_matches_oracle(world):
    _check(world, ("i32", 5000, 3001, 40, True, "merge"))


@pytest.mark.parametrize("S", ["u32", "f32", "u64", "i64", "el"])
def test_sharded_merge_key_types(S):
    _check(2, (S, 4097, 2999, 1000, S != "el", "merge"))


def test_sharded_merge_one_sided_and_empty():
    _check(3, ("u32", 0, 777, 10, True, "merge"))
    _check(2, ("i64", 1000, 0, 5, False, "merge"))
    _check(4, ("u32", 3, 2, 2, True, "merge"))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_sort_matches_oracle(world):
    _check(world, ("u32", 20000, 0, 1 << 30, False, "sort"))


def test_sharded_sort_is_stable_with_values():
    _check(4, ("i32", 9999, 0, 7, True, "sort"))
    _check(2, ("el", 5000, 0, 30, False, "sort"))


# ---- traffic accounting of the fused multi-GPU sort (bench.py --gpus N) ----
def _a_off(a, b, d):
    """a_off of the stable merge path on diagonal d (ties to A)."""
    lo, hi = max(0, d - len(b)), min(d, len(a))
    while lo < hi:
        mid = (lo + hi) // 2
        if b[d - 1 - mid] < a[mid]:
            hi = mid
        else:
            lo = mid + 1
    return lo


def _traffic_worker(rank, world, port, blocks, q):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1406_2628_b200 import multigpu as mg
        comm = mg._Comm()
        lens = [len(x) for x in blocks]
        rounds, _ = mg.P2PSorter.schedule(lens)
        cur = [np.sort(x) for x in blocks]
        trace = []
        for groups in rounds:
            L, R, gl = next(g for g in groups if rank in g[0] + g[1])
            if not R:
                trace.append(None)
            else:
                owners = L + R
                k = owners.index(rank)
                tot = sum(gl[x] for x in owners)
                o0, o1 = k * tot // len(owners), (k + 1) * tot // len(owners)
                A = np.concatenate([cur[x] for x in L])
                B = np.concatenate([cur[x] for x in R])
                sp = torch.tensor([_a_off(A, B, o0), _a_off(A, B, o1)])
                trace.append((owners, len(L), [gl[x] for x in owners], o0, o1, sp, None))
            # every rank replays the round on the whole data (host stand-in)
            new, nl = list(cur), mg.P2PSorter.schedule(lens)[0]
            for L2, R2, g2 in groups:
                if R2:
                    owners = L2 + R2
                    merged = np.sort(np.concatenate([cur[x] for x in owners]), kind="stable")
                    tot = len(merged)
                    for kk, x in enumerate(owners):
                        new[x] = merged[kk * tot // len(owners):(kk + 1) * tot // len(owners)]
            cur = new
        phases = mg.sort_traffic(comm, trace, lens, run0=4)
        t, tg = mg.roofline_time(phases, 4, 1000.0, 100.0)
        q.put((rank, phases, t, tg))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "ERR", traceback.format_exc(), None))


@pytest.mark.parametrize("world,shape", [(2, "random"), (2, "presorted"), (3, "random"),
                                         (4, "random")])
def test_sort_traffic_accounting(world, shape):
    """sort_traffic over gloo from traced split points: every remote read is
    one rank's NVLink-in and another's NVLink-out; HBM serves every read and
    every write once; a presorted input needs no NVLink at all; the
    roofline is the slowest rank's sum of per-phase maxima."""
    rng = np.random.default_rng(world)
    n = 1000 * world + 7
    x = rng.integers(0, 50, n)
    if shape == "presorted":
        x = np.sort(x)
    cuts = [r * n // world for r in range(world + 1)]
    blocks = [x[cuts[r]:cuts[r + 1]] for r in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_traffic_worker, args=(r, world, port, blocks, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, phases, t, tg = q.get(timeout=300)
        assert phases != "ERR", t
        res[r] = (phases, t, tg)
    for p in procs:
        p.join(timeout=60)
    phases, t, tg = res[0]
    assert all(res[r][0] == phases for r in range(world))  # every rank computes the same
    for ph in phases[1:]:
        assert sum(x["in"] for x in ph) == sum(x["out"] for x in ph)
        reads = sum(x["hbm"] for x in ph)
        assert reads <= 2 * n and reads >= n  # reads + writes of the merged groups
    cross_in = sum(x["in"] for ph in phases[1:] for x in ph)
    if shape == "presorted":
        assert cross_in == 0
    else:
        assert cross_in > 0
    assert t == max(tg) and len(tg) == world
    g = int(np.argmax(tg))
    want = sum(max(ph[g]["hbm"] * 4 / 1e12, ph[g]["in"] * 4 / 1e11, ph[g]["out"] * 4 / 1e11)
               for ph in phases)
    assert abs(want - tg[g]) < 1e-15
