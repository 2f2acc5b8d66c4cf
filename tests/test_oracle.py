"""Pin the C restatement (oracle/mp_oracle.c) before trusting it.

1. Known-answer tests transcribed from the reference's own unit tests
   (tests/golden/kats.json, each case cites its test_*.cpp line).
2. Fixtures recorded from the reference itself (tests/golden/ref_fixtures.npz,
   made by tests/golden/make_golden.py from /root/reference via oracle/_ref):
   merges, partitions with comparison counts, merge statistics, segmented
   window statistics, plan_segments and both sorts, for every key type.
3. When the compiled reference is present (oracle/_ref), a direct
   cross-check at the config-1 shape (u32 2^20 + 2^20, seeds 1/2, p = 8).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import element_array, fixture_cases, same
from oracle import bindings as B

KEYS = ("u32", "i32", "f32", "u64", "i64", "el")


# ---------------------------------------------------------------- KATs
def test_diagonal_search_kats(port, kats):
    for c in kats["diagonal_search"]:
        a, b = element_array(c["a"]), element_array(c["b"])
        got, cmp_ = port.diagonal_search("el", a, b, c["d"])
        assert (got, c["d"] - got) == tuple(c["want"]), c["src"]
        if "comparisons" in c:
            assert cmp_ == c["comparisons"], c["src"]


def test_partition_kats(port, kats):
    for c in kats["partition"]:
        a, b = element_array(c["a"]), element_array(c["b"])
        offs, _ = port.partition("el", a, b, c["p"])
        n = len(a) + len(b)
        got = [[int(o), i * n // c["p"] - int(o)] for i, o in enumerate(offs)]
        assert got == c["want"], c["src"]


def test_stable_merge_kats(port, kats):
    for c in kats["stable_merge"]:
        a = element_array(c["a"], c["a_tag_base"])
        b = element_array(c["b"], c["b_tag_base"])
        lo, hi = c.get("p_range", [1, 1])
        for p in range(lo, hi + 1):
            out, _, _, _ = port.merge("el", a, b, p=p)
            assert out["tag"].tolist() == c["want_tags"], (c["src"], p)


def test_sequential_merge_kats(kats):
    for c in kats["sequential_merge"]:
        a, b = element_array(c["a"]), element_array(c["b"])
        out, end = B.sequential_merge("el", a, b, c["start"], c["length"])
        assert out["key"].tolist() == c["want"], c["src"]
        assert list(end) == c["end"], c["src"]
    for c in kats["sequential_merge_overrun"]:
        a, b = element_array(c["a"]), element_array(c["b"])
        with pytest.raises(ValueError):
            B.sequential_merge("el", a, b, c["start"], c["length"])


def test_plan_segments_kats(port, kats):
    rng = np.random.default_rng(71)
    for c in kats["plan_segments"]:
        na = c.get("a_n", len(c.get("a", [])))
        nb = c.get("b_n", len(c.get("b", [])))
        a = element_array(np.sort(rng.integers(0, 500, na)))
        b = element_array(np.sort(rng.integers(0, 500, nb)))
        plan = port.plan_segments("el", a, b, c["p"], c["C"])
        assert plan["window_len"] == c["window_len"], c["src"]
        assert plan["p_eff"] == c["p_eff"], c["src"]
        assert plan["iterations"] == c["iterations"], c["src"]
        if "starts" in c:
            assert [list(s) for s in plan["starts"]] == c["starts"]
        if "starts_stride" in c:
            sa, sb = c["starts_stride"]
            assert plan["starts"] == [(sa * k, sb * k) for k in range(c["iterations"])]
        if "start_diagonals" in c:
            assert [x + y for x, y in plan["starts"]] == c["start_diagonals"]
        if "comparisons" in c:
            assert plan["comparisons"] == c["comparisons"]


def test_invalid_arguments(port):
    a = element_array([1, 2])
    b = element_array([3])
    with pytest.raises(ValueError):
        port.partition("el", a, b, 0)
    with pytest.raises(ValueError):
        port.merge("el", a, b, p=0)
    with pytest.raises(ValueError):
        port.segmented_merge("el", a, b, 2, 2)
    with pytest.raises(ValueError):
        port.segmented_merge("el", a, b, 0, 48)
    with pytest.raises(ValueError):
        port.plan_segments("el", a, b, 2, 0)
    with pytest.raises(ValueError):
        port.ce_sort("el", a, 2, 2)
    with pytest.raises(ValueError):
        port.merge_sort("el", a, p=0)


def test_mix64_kat(port, kats):
    for c in kats["mix64"]:
        assert port.mix64(c["x"]) == c["want"], c["src"]


def test_f32_total_order(port):
    # -0.0 before +0.0 across A and B; NaNs at the ends; equal +-0 keep A first
    f = lambda *v: np.array(v, dtype=np.float32).view(np.uint32)  # noqa: E731
    a = f(-np.inf, -0.0, 0.0, 1.0)
    b = f(-1.0, -0.0, 0.0, np.inf)
    out, _, _, _ = port.merge("f32", a, b)
    want = f(-np.inf, -1.0, -0.0, -0.0, 0.0, 0.0, 1.0, np.inf)
    assert out.tobytes() == want.tobytes()
    # A's -0.0 comes before B's -0.0 (ties to A): check via values
    av = np.array([0, 1, 2, 3], dtype=np.uint32)
    bv = np.array([10, 11, 12, 13], dtype=np.uint32)
    _, outv, _, _ = port.merge("f32", a, b, av=av, bv=bv)
    assert outv.tolist() == [0, 10, 1, 11, 2, 12, 3, 13]
    neg_nan = np.array([0xFFC00000], dtype=np.uint32)
    pos_nan = np.array([0x7FC00000], dtype=np.uint32)
    out, _, _, _ = port.merge("f32", np.concatenate([neg_nan, f(0.0)]),
                              np.concatenate([f(-np.inf), pos_nan]))
    assert out.tolist() == [0xFFC00000, f(-np.inf)[0], f(0.0)[0], 0x7FC00000]


# ---------------------------------------------------------------- fixtures
def test_fixture_merges_partitions_and_stats(port, fixtures):
    cases = [c for c in fixture_cases(fixtures, "m") if c[0] in KEYS]
    assert len(cases) >= 50
    for S, ci in cases:
        k = f"{S}/{ci}"
        a, b = fixtures[k + "/a"], fixtures[k + "/b"]
        out, _, _, _ = port.merge(S, a, b, p=3)
        assert same(out, fixtures[k + "/merged"]), k
        n = len(a) + len(b)
        for p in (1, 3, 8):
            ref = fixtures[k + f"/part{p}"]
            offs, cmp_ = port.partition(S, a, b, p)
            assert offs.tolist() == ref[0].tolist(), (k, p)
            assert [i * n // p - int(o) for i, o in enumerate(offs)] == ref[1].tolist()
            assert cmp_ == int(ref[2][0]), (k, p)
            _, _, c2, s2 = port.merge(S, a, b, p=p)
            assert [c2, s2] == fixtures[k + f"/mergestats{p}"].tolist(), (k, p)
        for p, C in ((3, 12), (8, 48), (1, 3)):
            sout, _, wins, c, s = port.segmented_merge(S, a, b, p, C)
            assert same(sout, out)
            assert [list(w) for w in wins] == fixtures[k + f"/seg{p}_{C}"].tolist(), (k, p, C)
            assert [c, s] == fixtures[k + f"/segstats{p}_{C}"].tolist(), (k, p, C)
            plan = port.plan_segments(S, a, b, p, C)
            assert [plan["window_len"], plan["p_eff"], plan["iterations"],
                    plan["comparisons"]] == fixtures[k + f"/plan{p}_{C}"].tolist()
            assert [list(x) for x in plan["starts"]] == fixtures[k + f"/planstarts{p}_{C}"].tolist()


def test_fixture_kv_records_match_soa_merge(port, fixtures):
    """Config-3 records: the reference merges {u64 key, u32 val} AoS with a
    key-only comparator; the oracle merges SoA keys + values."""
    for S, ci in fixture_cases(fixtures, "m"):
        if S != "kv":
            continue
        k = f"kv/{ci}"
        a, b, want = fixtures[k + "/a"], fixtures[k + "/b"], fixtures[k + "/merged"]
        out, outv, _, _ = port.merge("u64", a["key"].copy(), b["key"].copy(),
                                     av=a["val"].copy(), bv=b["val"].copy())
        assert out.tolist() == want["key"].tolist(), k
        assert outv.tolist() == want["val"].tolist(), k


def test_fixture_sorts(port, fixtures):
    for S, ci in fixture_cases(fixtures, "s"):
        k = f"{S}/{ci}"
        d = fixtures[k + "/in"]
        if S == "kv":
            out, outv, rounds = port.merge_sort("u64", d["key"].copy(), vals=d["val"].copy())
            want = fixtures[k + "/sorted"]
            assert out.tolist() == want["key"].tolist() and outv.tolist() == want["val"].tolist()
            continue
        out, _, rounds = port.merge_sort(S, d, p=3)
        assert same(out, fixtures[k + "/sorted"]), k
        assert rounds == int(fixtures[k + "/rounds"][0]), k
        ce, _, levels = port.ce_sort(S, d, 4, 48)
        assert same(ce, out), k
        assert levels == int(fixtures[k + "/ce_levels48"][0]), k


def test_fixture_checksum(port, fixtures):
    a, b = fixtures["checksum/a"], fixtures["checksum/b"]
    out, _, _, _ = port.merge("el", a, b)
    want = fixtures["checksum/sum"].tolist()
    assert port.checksum("el", out) == want[0] == want[1]


# ---------------------------------------------------------------- generators
def test_generators_ranges(port):
    x = port.generate(1, 1, 0, 100000)
    assert x.min() >= 0 and x.max() < 1024
    lo = port.generate(3, 2, 0, 10000)
    hi = port.generate(4, 1, 0, 10000)
    assert lo.max() < (1 << 40) <= hi.min()
    # x_i(seed) is the (i+1)-th SplitMix64 output from state `seed`
    first = port.generate(2, 5, 0, 3)
    assert first[0] == port.mix64(5 + 0) and first[2] == port.mix64(5 + 2 * 0x9E3779B97F4A7C15 % (1 << 64))
    # sharded generation equals whole generation
    assert np.array_equal(port.generate(0, 1, 1000, 50), port.generate(0, 1, 0, 1050)[1000:])
    f = port.generate(5, 1, 0, 100000)
    assert abs(float(f.mean())) < 0.02 and abs(float(f.std()) - 1) < 0.02
    e = port.generate(6, 2, 0, 100000)
    assert e.min() >= 0 and abs(float(e.mean()) - 1) < 0.02


def test_radix_sort_helper(port):
    for dt in (np.uint32, np.int32, np.uint64, np.int64):
        rng = np.random.default_rng(5)
        x = rng.integers(-1000 if np.dtype(dt).kind == "i" else 0, 1 << 30, 5000).astype(dt)
        assert np.array_equal(port.radix_sort(x.copy()), np.sort(x))
    f = port.generate(5, 3, 0, 5000)
    s = port.radix_sort(f.copy())
    assert np.all(np.diff(s) >= 0)


# ---------------------------------------------------------------- reference
@pytest.mark.skipif(not B.ref_available(), reason="reference library not built")
def test_port_equals_reference_config1():
    P, R = B.port(), B.ref()
    a = P.radix_sort(P.generate(0, 1, 0, 1 << 20))
    b = P.radix_sort(P.generate(0, 2, 0, 1 << 20))
    out_p, _, cmp_p, _ = P.merge("u32", a, b, p=8)
    out_r, cmp_r, _ = R.merge("u32", a, b, p=8)
    assert out_p.tobytes() == out_r.tobytes()
    assert cmp_p == cmp_r
    offs_p, _ = P.partition("u32", a, b, 8)
    oa, _, _ = R.partition("u32", a, b, 8)
    assert offs_p.tolist() == oa.tolist()
