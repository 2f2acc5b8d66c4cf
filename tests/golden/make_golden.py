"""Generate tests/golden/ref_fixtures.npz from the REFERENCE ITSELF.

Runs the unmodified reference library (oracle/_ref/libmergepath_ref.so,
compiled by oracle/Makefile from /root/reference) on seeded inputs for every
key type and records its outputs: partitions (+ comparison counts), merges,
segmented-merge window statistics, plan_segments, both sorts and checksums.
The fixtures pin the C restatement (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_parity.py) to the reference's actual behaviour; they travel
to the GPU box, the reference does not.

    python tests/golden/make_golden.py     # needs /root/reference
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import bindings as B  # noqa: E402

OUT = Path(__file__).resolve().parent / "ref_fixtures.npz"

SIZES = [(0, 0), (0, 5), (5, 0), (1, 1), (7, 3), (40, 40), (100, 37), (300, 211),
         (1000, 999), (4097, 3001)]
PS = (1, 3, 8)
SEG = ((3, 12), (8, 48), (1, 3))
SORT_NS = (0, 1, 2, 31, 33, 257, 4096, 10001)


def f32_order(u):
    u = u.astype(np.uint64)
    return np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000)


def special_floats(rng, n):
    pool = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45,
                     3.4e38, -3.4e38, 0.5, -0.5], dtype=np.float32).view(np.uint32)
    neg_nan = np.array([0xFFC00000, 0x7FC00001], dtype=np.uint32)
    pool = np.concatenate([pool, neg_nan])
    x = rng.integers(0, len(pool) + 8, n)
    vals = rng.standard_normal(n).astype(np.float32).view(np.uint32)
    return np.where(x < len(pool), pool[np.minimum(x, len(pool) - 1)], vals).astype(np.uint32)


def sorted_keys(S, rng, n):
    """Sorted, duplicate-friendly keys (oracles.hpp:114-124 style range n/2)."""
    r = max(4, n // 2)
    if S == "u32":
        k = rng.integers(0, r, n).astype(np.uint32) * np.uint32(97)
    elif S == "i32":
        k = (rng.integers(0, r, n) - r // 2).astype(np.int32)
    elif S == "f32":
        k = special_floats(rng, n)
        return k[np.argsort(f32_order(k), kind="stable")]
    elif S == "u64":
        k = rng.integers(0, r, n).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15 >> 8)
    elif S == "i64":
        k = (rng.integers(0, r, n) - r // 2).astype(np.int64) * np.int64(1 << 33)
    elif S in ("el", "kv"):
        dt = B.DTYPES[S]
        k = np.zeros(n, dtype=dt)
        k["key"] = rng.integers(0, r, n)
        k["tag" if S == "el" else "val"] = np.arange(n, dtype=np.uint32)
        return k[np.argsort(k["key"], kind="stable")]
    return np.sort(k, kind="stable")


def shuffled(S, rng, n):
    r = max(3, n // 3)
    if S in ("el", "kv"):
        dt = B.DTYPES[S]
        k = np.zeros(n, dtype=dt)
        k["key"] = rng.integers(0, r, n)
        k["tag" if S == "el" else "val"] = np.arange(n, dtype=np.uint32)
        return k
    if S == "f32":
        return special_floats(rng, n)
    dt = B.DTYPES[S]
    if dt.kind == "i":
        return (rng.integers(0, r, n) - r // 2).astype(dt)
    return rng.integers(0, r, n).astype(dt)


def same(x, y) -> bool:
    """Bitwise equality; for the reference `element` the 4 padding bytes are
    not part of the value (core.hpp:39-51) so compare key+tag."""
    if x.dtype == B.ELEMENT_DTYPE:
        return (np.array_equal(x["key"], y["key"]) and np.array_equal(x["tag"], y["tag"]))
    return x.tobytes() == y.tobytes()


def clean(x):
    if x.dtype == B.ELEMENT_DTYPE:
        x = x.copy()
        x["pad"] = 0
    return x


def main() -> None:
    R = B.ref()
    rec: dict[str, np.ndarray] = {}
    for si, S in enumerate(("u32", "i32", "f32", "u64", "i64", "el", "kv")):
        rng = np.random.default_rng(1406 + si)
        for ci, (na, nb) in enumerate(SIZES):
            a = sorted_keys(S, rng, na)
            b = sorted_keys(S, rng, nb)
            if S == "el":
                b["tag"] += np.uint32(1 << 20)  # distinguish origins
            if S == "kv":
                b["val"] |= np.uint32(1 << 31)
            key = f"{S}/m{ci}"
            rec[key + "/a"] = a
            rec[key + "/b"] = b
            out, cmp_, steps = R.merge(S, a, b, p=3)
            rec[key + "/merged"] = clean(out)
            for p in PS:
                oa, ob, c = R.partition(S, a, b, p)
                rec[key + f"/part{p}"] = np.stack([oa, ob, np.full_like(oa, c)])
                _, c2, s2 = R.merge(S, a, b, p=p)
                rec[key + f"/mergestats{p}"] = np.array([c2, s2], dtype=np.uint64)
            for p, C in SEG:
                sout, wins, c, s = R.segmented_merge(S, a, b, p, C)
                assert same(sout, out)
                rec[key + f"/seg{p}_{C}"] = np.array(wins, dtype=np.uint64).reshape(-1, 2)
                rec[key + f"/segstats{p}_{C}"] = np.array([c, s], dtype=np.uint64)
                plan = R.plan_segments(S, a, b, p, C)
                rec[key + f"/plan{p}_{C}"] = np.array(
                    [plan["window_len"], plan["p_eff"], plan["iterations"], plan["comparisons"]],
                    dtype=np.uint64)
                rec[key + f"/planstarts{p}_{C}"] = np.array(plan["starts"], dtype=np.uint64).reshape(-1, 2)
        for ni, n in enumerate(SORT_NS):
            d = shuffled(S, rng, n)
            key = f"{S}/s{ni}"
            rec[key + "/in"] = d
            out, rounds = R.merge_sort(S, d, p=3)
            rec[key + "/sorted"] = clean(out)
            rec[key + "/rounds"] = np.array([rounds], dtype=np.uint64)
            ce, levels = R.ce_sort(S, d, p=4, cache=48)
            assert same(ce, out)
            rec[key + "/ce_levels48"] = np.array([levels], dtype=np.uint64)
    # register-sink checksums on the test element (parallel.hpp:181-198)
    rng = np.random.default_rng(67)
    a = sorted_keys("el", rng, 300)
    b = sorted_keys("el", rng, 211)
    rec["checksum/a"], rec["checksum/b"] = a, b
    rec["checksum/sum"] = np.array([R.merge_checksum_el(a, b, 4),
                                    R.segmented_checksum_el(a, b, 4, 48)], dtype=np.uint64)
    np.savez_compressed(OUT, **rec)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(rec)} arrays)")


if __name__ == "__main__":
    main()
