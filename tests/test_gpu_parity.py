"""Parity of the CUDA path (through the C ABI) with the reference.

Small cases: bit-exact against fixtures recorded from the reference itself
(tests/golden/ref_fixtures.npz) and against the C restatement on the same
seeded inputs.  Full BASELINE.json sizes: size-independent properties
(sortedness, multiset equality, A-before-B on ties, each input appearing in
order in the output) that together pin the unique stable merge.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import element_array, fixture_cases, same

pytestmark = pytest.mark.gpu

KEYS = ("u32", "i32", "f32", "u64", "i64", "el")
TORCH_DT = {}


def _torch():
    import torch
    global TORCH_DT
    TORCH_DT = {"u32": torch.uint32, "i32": torch.int32, "f32": torch.float32,
                "u64": torch.uint64, "i64": torch.int64}
    return torch


def to_dev(x, S, dev):
    torch = _torch()
    if S == "el":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).to(dev)
    if S == "f32":
        x = np.ascontiguousarray(x).view(np.float32)
    return torch.from_numpy(np.ascontiguousarray(x).copy()).to(dev)


def from_dev(t, S):
    from oracle.bindings import ELEMENT_DTYPE
    x = t.cpu().numpy()
    if S == "el":
        return x.view(ELEMENT_DTYPE)
    if S == "f32":
        return x.view(np.uint32)
    return x


def key_type(S):
    from paper_1406_2628_b200 import _native as N
    return {"u32": N.KEY_U32, "i32": N.KEY_I32, "f32": N.KEY_F32, "u64": N.KEY_U64,
            "i64": N.KEY_I64, "el": N.KEY_ELEMENT}[S]


# ------------------------------------------------------------ fixtures
def test_fixture_merges_device(cuda, fixtures):
    from paper_1406_2628_b200 import mergepath as mp
    for S, ci in fixture_cases(fixtures, "m"):
        if S not in KEYS:
            continue
        k = f"{S}/{ci}"
        a, b = fixtures[k + "/a"], fixtures[k + "/b"]
        out = mp.parallel_merge(to_dev(a, S, cuda), to_dev(b, S, cuda), 3, key_type=key_type(S))
        assert same(from_dev(out, S), fixtures[k + "/merged"]), k


def test_fixture_merges_host_entry(cuda, fixtures):
    from paper_1406_2628_b200 import mergepath as mp
    for S, ci in fixture_cases(fixtures, "m"):
        if S not in KEYS:
            continue
        k = f"{S}/{ci}"
        a, b = fixtures[k + "/a"], fixtures[k + "/b"]
        out = mp.parallel_merge(a, b, 8, key_type=key_type(S))
        assert same(out, fixtures[k + "/merged"]), k


def test_fixture_kv_merge_with_values(cuda, fixtures):
    torch = _torch()
    from paper_1406_2628_b200 import mergepath as mp
    for S, ci in fixture_cases(fixtures, "m"):
        if S != "kv":
            continue
        k = f"kv/{ci}"
        a, b, want = fixtures[k + "/a"], fixtures[k + "/b"], fixtures[k + "/merged"]
        ak = torch.from_numpy(a["key"].copy()).to(cuda)
        bk = torch.from_numpy(b["key"].copy()).to(cuda)
        av = torch.from_numpy(a["val"].copy()).to(cuda)
        bv = torch.from_numpy(b["val"].copy()).to(cuda)
        out, outv = mp.parallel_merge(ak, bk, 8, a_vals=av, b_vals=bv)
        assert out.cpu().numpy().tolist() == want["key"].tolist(), k
        assert outv.cpu().numpy().tolist() == want["val"].tolist(), k


def test_fixture_partitions_and_stats(cuda, fixtures):
    from paper_1406_2628_b200 import mergepath as mp
    for S, ci in fixture_cases(fixtures, "m"):
        if S not in KEYS:
            continue
        k = f"{S}/{ci}"
        a, b = to_dev(fixtures[k + "/a"], S, cuda), to_dev(fixtures[k + "/b"], S, cuda)
        kt = key_type(S)
        for p in (1, 3, 8):
            ref = fixtures[k + f"/part{p}"]
            cnt = [0]
            pts = mp.partition(a, b, p, comparisons=cnt, key_type=kt)
            assert [x.a_off for x in pts] == ref[0].tolist(), (k, p)
            assert [x.b_off for x in pts] == ref[1].tolist(), (k, p)
            assert cnt[0] == int(ref[2][0]), (k, p)
            st = mp.MergeStats()
            mp.parallel_merge(a, b, p, stats=st, key_type=kt)
            assert [st.partition_comparisons, st.merge_steps] == \
                fixtures[k + f"/mergestats{p}"].tolist(), (k, p)
        for p, C in ((3, 12), (8, 48), (1, 3)):
            st = mp.MergeStats()
            mp.segmented_parallel_merge(a, b, p, C, stats=st, key_type=kt)
            wins = [[w.a_consumed, w.b_consumed] for w in st.windows]
            assert wins == fixtures[k + f"/seg{p}_{C}"].tolist(), (k, p, C)
            assert [st.partition_comparisons, st.merge_steps] == \
                fixtures[k + f"/segstats{p}_{C}"].tolist(), (k, p, C)
            cnt = [0]
            plan = mp.plan_segments(a, b, p, C, comparisons=cnt, key_type=kt)
            ref = fixtures[k + f"/plan{p}_{C}"].tolist()
            assert [plan.window_len, plan.p_eff, plan.iterations, cnt[0]] == ref, (k, p, C)
            assert [[s.a_off, s.b_off] for s in plan.starting_points] == \
                fixtures[k + f"/planstarts{p}_{C}"].tolist(), (k, p, C)


def test_fixture_sorts(cuda, fixtures):
    from paper_1406_2628_b200 import mergepath as mp
    for S, ci in fixture_cases(fixtures, "s"):
        k = f"{S}/{ci}"
        d = fixtures[k + "/in"]
        want = fixtures[k + "/sorted"]
        if S == "kv":
            torch = _torch()
            keys = torch.from_numpy(d["key"].copy()).to(cuda)
            vals = torch.from_numpy(d["val"].copy()).to(cuda)
            out, outv = mp.parallel_merge_sort(keys, 3, vals=vals)
            assert out.cpu().numpy().tolist() == want["key"].tolist(), k
            assert outv.cpu().numpy().tolist() == want["val"].tolist(), k
            continue
        st = mp.SortStats()
        out = mp.parallel_merge_sort(to_dev(d, S, cuda), 3, stats=st, key_type=key_type(S))
        assert same(from_dev(out, S), want), k
        assert st.merge_rounds == int(fixtures[k + "/rounds"][0])
        out2 = mp.cache_efficient_parallel_sort(d, 4, 48, key_type=key_type(S))
        assert same(out2, want), k


def test_fixture_checksum(cuda, fixtures):
    from paper_1406_2628_b200 import mergepath as mp
    a, b = fixtures["checksum/a"], fixtures["checksum/b"]
    want = fixtures["checksum/sum"].tolist()
    assert mp.parallel_merge_checksum(a, b, 4, key_type=key_type("el")) == want[0]
    assert mp.segmented_parallel_merge_checksum(to_dev(a, "el", cuda), to_dev(b, "el", cuda),
                                                4, 48, key_type=key_type("el")) == want[1]


# ------------------------------------------------------------ KATs on device
def test_kats_on_device(cuda, kats):
    from paper_1406_2628_b200 import mergepath as mp
    kt = key_type("el")
    for c in kats["diagonal_search"]:
        a, b = element_array(c["a"]), element_array(c["b"])
        cnt = [0]
        pt = mp.diagonal_search(a, b, c["d"], comparisons=cnt, key_type=kt)
        assert [pt.a_off, pt.b_off] == c["want"], c["src"]
        if "comparisons" in c:
            assert cnt[0] == c["comparisons"]
    for c in kats["partition"]:
        pts = mp.partition(element_array(c["a"]), element_array(c["b"]), c["p"], key_type=kt)
        assert [[p.a_off, p.b_off] for p in pts] == c["want"], c["src"]
    for c in kats["stable_merge"]:
        a = element_array(c["a"], c["a_tag_base"])
        b = element_array(c["b"], c["b_tag_base"])
        lo, hi = c.get("p_range", [1, 1])
        for p in range(lo, hi + 1):
            out = mp.parallel_merge(a, b, p, key_type=kt)
            assert out["tag"].tolist() == c["want_tags"], c["src"]
    for c in kats["invalid_argument"]:
        a = element_array([1, 2])
        with pytest.raises(ValueError):
            op = getattr(mp, c["op"])
            if c["op"] in ("partition", "parallel_merge"):
                op(a, a, c["p"], key_type=kt)
            elif c["op"] in ("segmented_parallel_merge", "plan_segments"):
                op(a, a, c["p"], c["C"], key_type=kt)
            elif c["op"] == "parallel_merge_sort":
                op(a, c["p"], key_type=kt)
            else:
                op(a, c["p"], c["C"], key_type=kt)


# ------------------------------------------------------------ vs the C restatement
SHAPES = [(0, 0), (0, 1), (1, 0), (1, 1), (3839, 1), (1, 3840), (3840, 3840), (3841, 3839),
          (5000, 17), (17, 5000), (123457, 98765), (1 << 17, 1 << 17)]


@pytest.mark.parametrize("S", KEYS)
def test_random_merges_vs_oracle(cuda, port, S):
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(7)
    for na, nb in SHAPES:
        for dup in (4, 1 << 30):
            a = _rand_sorted(S, rng, na, dup)
            b = _rand_sorted(S, rng, nb, dup)
            if S == "el":
                b["tag"] += np.uint32(1 << 24)
            want, _, _, _ = port.merge(S, a, b)
            got = mp.parallel_merge(to_dev(a, S, cuda), to_dev(b, S, cuda), 8,
                                    key_type=key_type(S))
            assert same(from_dev(got, S), want), (S, na, nb, dup)


@pytest.mark.parametrize("S", ("u32", "f32", "u64", "i64"))
def test_random_merges_with_values_vs_oracle(cuda, port, S):
    torch = _torch()
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(11)
    for na, nb in SHAPES:
        a = _rand_sorted(S, rng, na, 16)
        b = _rand_sorted(S, rng, nb, 16)
        av = np.arange(na, dtype=np.uint32)
        bv = np.arange(nb, dtype=np.uint32) | np.uint32(1 << 31)
        want, wantv, _, _ = port.merge(S, a, b, av=av, bv=bv)
        got, gotv = mp.parallel_merge(to_dev(a, S, cuda), to_dev(b, S, cuda), 1,
                                      a_vals=torch.from_numpy(av).to(cuda),
                                      b_vals=torch.from_numpy(bv).to(cuda), key_type=key_type(S))
        assert same(from_dev(got, S), want), (S, na, nb)
        assert np.array_equal(gotv.cpu().numpy(), wantv), (S, na, nb)


def test_unaligned_views_exercise_edge_copies(cuda, port):
    """Sub-views at every 4-byte offset: the bulk-copy interior shrinks and
    the head/tail copies by ordinary loads take over."""
    torch = _torch()
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(3)
    base_a = np.sort(rng.integers(0, 1000, 20000).astype(np.uint32))
    base_b = np.sort(rng.integers(0, 1000, 20000).astype(np.uint32))
    da, db = torch.from_numpy(base_a).to(cuda), torch.from_numpy(base_b).to(cuda)
    for oa in range(4):
        for ob in range(4):
            for la, lb in ((19000, 17), (5, 7), (3, 0), (7777, 7779)):
                a, b = base_a[oa:oa + la], base_b[ob:ob + lb]
                want, _, _, _ = port.merge("u32", a, b)
                out_full = torch.empty(la + lb + 3, dtype=torch.uint32, device=cuda)
                out = out_full[(oa + ob) % 4:(oa + ob) % 4 + la + lb]
                mp.parallel_merge_into(da[oa:oa + la], db[ob:ob + lb], out, 2)
                assert np.array_equal(out.cpu().numpy(), want), (oa, ob, la, lb)


@pytest.mark.parametrize("S", KEYS)
def test_random_sorts_vs_oracle(cuda, port, S):
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(13)
    for n in (0, 1, 2, 2047, 2048, 2049, 4095, 4096, 4097, 10001, 65537, 300000):
        for dup in (3, 1 << 30):
            d = _rand_unsorted(S, rng, n, dup)
            want, _, _ = port.merge_sort(S, d)
            got = mp.parallel_merge_sort(to_dev(d, S, cuda), 4, key_type=key_type(S))
            assert same(from_dev(got, S), want), (S, n, dup)


@pytest.mark.parametrize("S", ("u32", "i32", "f32", "u64", "i64"))
def test_sort_with_values_is_stable(cuda, port, S):
    torch = _torch()
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(17)
    for n in (1, 100, 2048, 5000, 123456):
        d = _rand_unsorted(S, rng, n, 7)
        v = np.arange(n, dtype=np.uint32)
        want, wantv, _ = port.merge_sort(S, d, vals=v)
        got, gotv = mp.parallel_merge_sort(to_dev(d, S, cuda), 2,
                                           vals=torch.from_numpy(v).to(cuda),
                                           key_type=key_type(S))
        assert same(from_dev(got, S), want) and np.array_equal(gotv.cpu().numpy(), wantv), (S, n)


def test_checksum_vs_oracle(cuda, port):
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(19)
    for S in ("u32", "i32", "u64", "i64", "el", "f32"):
        for na, nb in ((0, 0), (10, 0), (1000, 2000), (70001, 50000)):
            a, b = _rand_sorted(S, rng, na, 50), _rand_sorted(S, rng, nb, 50)
            out, _, _, _ = port.merge(S, a, b)
            want = port.checksum(S, out)
            got = mp.parallel_merge_checksum(to_dev(a, S, cuda), to_dev(b, S, cuda), 4,
                                             key_type=key_type(S))
            assert got == want, (S, na, nb)


def test_device_generator_matches_oracle(cuda, port):
    torch = _torch()
    from paper_1406_2628_b200 import _native as N
    for kind, dt in ((0, torch.uint32), (1, torch.int32), (2, torch.uint64), (3, torch.uint64),
                     (4, torch.uint64)):
        out = torch.empty(100003, dtype=dt, device=cuda)
        N.check(N.lib.mp_generate(kind, 9, 12345, out.numel(), out.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream))
        assert np.array_equal(out.cpu().numpy(), port.generate(kind, 9, 12345, 100003)), kind


# ------------------------------------------------------------ BASELINE configs
def test_config1_bit_exact_and_partition(cuda, port):
    """Config 1: u32 2^20 + 2^20, seeds 1/2, p = 8: bit-exact output and the
    9 partition points equal the reference's partition(in, 8)."""
    torch = _torch()
    from oracle import bindings as B
    from paper_1406_2628_b200 import mergepath as mp
    a = port.radix_sort(port.generate(0, 1, 0, 1 << 20))
    b = port.radix_sort(port.generate(0, 2, 0, 1 << 20))
    if B.REF_LIB.exists():
        R = B.ref()
        want, _, _ = R.merge("u32", a, b, p=8)
        oa, ob, _ = R.partition("u32", a, b, 8)
    else:
        want, _, _, _ = port.merge("u32", a, b, p=8)
        oa, _ = port.partition("u32", a, b, 8)
    da, db = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    got = mp.parallel_merge(da, db, 8)
    assert np.array_equal(got.cpu().numpy(), want)
    pts = mp.partition(da, db, 8)
    assert [p.a_off for p in pts] == oa.tolist()
    assert mp.parallel_merge(a, b, 8).tobytes() == want.tobytes()  # host entry


def test_config5_shape_totalorder_merge(cuda, port):
    """Config 5 inputs (f32 Normal(0,1) and Exp(1) from the device generator,
    sorted by IEEE totalOrder with our sort) at 2^22 + 2^22: the merge of the
    same bytes equals the oracle's, -0.0/+0.0 included."""
    torch = _torch()
    from paper_1406_2628_b200 import _native as N
    n = 1 << 22
    st = torch.cuda.current_stream().cuda_stream
    a = torch.empty(n, dtype=torch.float32, device=cuda)
    b = torch.empty(n, dtype=torch.float32, device=cuda)
    N.check(N.lib.mp_generate(5, 1, 0, n, a.data_ptr(), st))
    N.check(N.lib.mp_generate(6, 2, 0, n, b.data_ptr(), st))
    a[::97] = -0.0  # signed zeros on both sides
    b[::89] = 0.0
    b[1::89] = -0.0
    for x in (a, b):
        N.check(N.lib.mp_sort(N.KEY_F32, x.data_ptr(), None, n, None, 0, st))
    ha = a.cpu().numpy().view(np.uint32)
    hb = b.cpu().numpy().view(np.uint32)
    order = lambda u: np.where(u & 0x80000000, ~u, u | 0x80000000)  # noqa: E731
    assert np.all(np.diff(order(ha).astype(np.int64)) >= 0)
    af = a.cpu().numpy()
    assert abs(float(af.mean())) < 0.01 and abs(float(af.std()) - 1) < 0.01
    assert abs(float(b.cpu().numpy().mean()) - 1) < 0.05  # 2/89 of B zeroed above
    from paper_1406_2628_b200 import mergepath as mp
    got = mp.parallel_merge(a, b, 8)
    want, _, _, _ = port.merge("f32", ha, hb)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want)


def _sorted_dev(kind, seed, n, dev):
    torch = _torch()
    from paper_1406_2628_b200 import _native as N
    dt = {0: torch.uint32, 1: torch.int32, 2: torch.uint64, 3: torch.uint64, 4: torch.uint64}[kind]
    x = torch.empty(n, dtype=dt, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), st))
    N.check(N.lib.mp_sort(N.KEY_U32 if kind == 0 else N.KEY_I32 if kind == 1 else N.KEY_U64,
                          x.data_ptr(), None, n, None, 0, st))
    return x


def test_config2_full_size_properties(cuda):
    """Config 2: i32 2^28 + 2^28 in [0,1024): sorted, and per-key counts of
    the output equal the sum of the inputs' (multiset equality).  For bare
    keys these two properties determine the merged bytes."""
    torch = _torch()
    from paper_1406_2628_b200 import mergepath as mp
    n = 1 << 28
    a = _sorted_dev(1, 1, n, cuda)
    b = _sorted_dev(1, 2, n, cuda)
    assert bool((a[1:] >= a[:-1]).all()) and bool((b[1:] >= b[:-1]).all())
    out = mp.parallel_merge(a, b, 8)
    assert bool((out[1:] >= out[:-1]).all())
    ca = torch.bincount(a, minlength=1024)
    cb = torch.bincount(b, minlength=1024)
    co = torch.bincount(out, minlength=1024)
    assert torch.equal(ca + cb, co)
    del out
    # the p-way partition points split the output at equal-size boundaries
    pts = mp.partition(a, b, 8)
    for i, p in enumerate(pts):
        assert p.d == (i * 2 * n) // 8


@pytest.mark.parametrize("variant", ["3a", "3b"])
def test_config3_full_size_stability(cuda, variant):
    """Config 3: u64 keys + u32 values (source index, bit 31 marks B),
    |A| = 2^29, |B| = 2^25.  Properties that pin the unique stable merge:
    keys sorted; A-origin values appear as 0,1,2,... and B-origin values as
    0,1,2,... (each input in order); keys match their source; on equal keys
    no B element precedes an A element."""
    torch = _torch()
    from paper_1406_2628_b200 import mergepath as mp
    na, nb = 1 << 29, 1 << 25
    if variant == "3a":
        a = _sorted_dev(2, 1, na, cuda)
        b = _sorted_dev(2, 2, nb, cuda)
    else:
        a = _sorted_dev(4, 1, na, cuda)
        b = _sorted_dev(3, 2, nb, cuda)
    av = torch.arange(na, dtype=torch.int32, device=cuda).view(torch.uint32)
    # j | 0x80000000 as a bit pattern == j - 2^31 as int32
    bv = (torch.arange(nb, dtype=torch.int32, device=cuda)
          + torch.iinfo(torch.int32).min).view(torch.uint32)
    out, outv = mp.parallel_merge(a, b, 8, a_vals=av, b_vals=bv)
    del av, bv
    ok = out.view(torch.int64)  # compare u64 through signed view with offset
    s = (ok ^ torch.iinfo(torch.int64).min)
    assert bool((s[1:] >= s[:-1]).all())
    del s
    v = outv.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    from_b = v >= (1 << 31)
    ia = v[~from_b]
    ib = v[from_b] - (1 << 31)
    assert ia.numel() == na and ib.numel() == nb
    assert torch.equal(ia, torch.arange(na, device=cuda))
    assert torch.equal(ib, torch.arange(nb, device=cuda))
    del ia, ib
    # tie rule: equal adjacent keys never go B then A
    eq = ok[1:] == ok[:-1]
    assert not bool((eq & from_b[:-1] & ~from_b[1:]).any())
    if variant == "3b":  # B entirely below A: output = B then A
        assert bool(from_b[:nb].all()) and not bool(from_b[nb:].any())


def test_config4_sort_full_size(cuda):
    """Config 4 on one GPU: 2^30 u32 keys, 16384-key block sort + 16 rounds
    (8 fused pairs); equals torch.sort of the same keys (bare keys: sorted
    order is unique)."""
    torch = _torch()
    from paper_1406_2628_b200 import _native as N
    n = 1 << 30
    x = torch.empty(n, dtype=torch.uint32, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    N.check(N.lib.mp_generate(0, 4, 0, n, x.data_ptr(), st))
    ref = torch.sort(x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values
    torch.cuda.empty_cache()  # torch.sort's temporaries (tens of GB) back to the driver
    N.check(N.lib.mp_sort(N.KEY_U32, x.data_ptr(), None, n, None, 0, st))
    got = x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    assert torch.equal(got, ref)


def test_config4_sort_full_size_vs_reference(cuda):
    """Config 4 at full size byte for byte against the REFERENCE's own
    parallel_merge_sort (oracle/_ref, sort.hpp:132-148, on this host's
    cores) on the same 2^30 keys -- and the host-span drop-in path
    (mp_sort_host from pageable memory) gives the same bytes."""
    torch = _torch()
    B = _ref_or_skip()
    from paper_1406_2628_b200 import _native as N
    n = 1 << 30
    x = torch.empty(n, dtype=torch.uint32, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    N.check(N.lib.mp_generate(0, 4, 0, n, x.data_ptr(), st))
    hx = x.cpu().numpy()
    N.check(N.lib.mp_sort(N.KEY_U32, x.data_ptr(), None, n, None, 0, st))
    got = x.cpu().numpy()
    del x
    want, _ = B.ref().merge_sort("u32", hx, p=B.host_cores())
    assert got.tobytes() == want.tobytes()
    ho = np.empty_like(hx)
    N.check(N.lib.mp_sort_host(N.KEY_U32, hx.ctypes.data, None, n, ho.ctypes.data, None, 0))
    assert ho.tobytes() == want.tobytes()


@pytest.mark.parametrize("kind", ["u32", "i32", "f32"])
def test_mid_size_sorts_with_fused_round_pairs(cuda, kind):
    """Sizes past the in-kernel-search threshold take the fused round pairs
    by default (K4q/K4r/K5e at 16384-output tiles): ragged sizes (short
    last groups of 1-3 runs), uniform keys and heavy duplicates, against
    torch.sort of the order image (bare keys: the sorted bytes are unique)."""
    torch = _torch()
    from paper_1406_2628_b200 import _native as N
    st = torch.cuda.current_stream().cuda_stream
    kt = {"u32": N.KEY_U32, "i32": N.KEY_I32, "f32": N.KEY_F32}[kind]
    g = torch.Generator(device=cuda)
    g.manual_seed(1406)
    for n, span in ((30_000_001, 1 << 32), (50_331_655, 1 << 32), (41_943_040 + 8191, 977)):
        raw = torch.randint(0, span, (n,), device=cuda, generator=g, dtype=torch.int64)
        if kind == "f32":
            f = (raw - span // 2).to(torch.float32) / 3.0
            f[::97] = -0.0
            x = f.view(torch.int32)
        else:
            x = (raw - (span // 2 if kind == "i32" else 0)).to(torch.int64)
            x = (x & 0xFFFFFFFF).to(torch.int64)
            x = torch.where(x >= 2**31, x - 2**32, x).to(torch.int32)
        u = x.to(torch.int64) & 0xFFFFFFFF
        if kind == "i32":
            key = u ^ 0x80000000
        elif kind == "f32":
            key = torch.where(u >= 2**31, (~u) & 0xFFFFFFFF, u | 0x80000000)
        else:
            key = u
        want = u[torch.sort(key, stable=True).indices]
        y = x.clone()
        N.check(N.lib.mp_sort(kt, y.data_ptr(), None, n, None, 0, st))
        got = y.to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(got, want), (kind, n)


# ------------------------------------------------------------ helpers
def _rand_sorted(S, rng, n, dup):
    from oracle.bindings import ELEMENT_DTYPE
    r = max(2, min(dup, 1 << 62))
    if S == "el":
        e = np.zeros(n, dtype=ELEMENT_DTYPE)
        e["key"] = np.sort(rng.integers(-r, r, n))
        e["tag"] = np.arange(n, dtype=np.uint32)
        return e
    if S == "f32":
        x = (rng.integers(-r, r, n) / 7.0).astype(np.float32)
        x[rng.random(n) < 0.05] = -0.0
        u = x.view(np.uint32)
        key = np.where(u & 0x80000000, ~u, u | 0x80000000)
        return u[np.argsort(key, kind="stable")]
    dt = {"u32": np.uint32, "i32": np.int32, "u64": np.uint64, "i64": np.int64}[S]
    if np.dtype(dt).kind == "u":
        return np.sort(rng.integers(0, min(r, np.iinfo(dt).max), n).astype(dt))
    return np.sort(rng.integers(-min(r, np.iinfo(dt).max), min(r, np.iinfo(dt).max), n).astype(dt))


def _rand_unsorted(S, rng, n, dup):
    x = _rand_sorted(S, rng, n, dup)
    perm = rng.permutation(n)
    x = x[perm]
    if S == "el":
        x["tag"] = np.arange(n, dtype=np.uint32)
    return x




@pytest.mark.parametrize("S", KEYS)
def test_large_merges_vs_oracle(cuda, port, S):
    """Merges >= 2^20 keys (full-size kernel grids); shapes cover CTA-range
    edges, one-sided windows, ragged tails."""
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(29)
    for na, nb, dup in ((1 << 20, 1 << 20, 1 << 30), (1_000_003, 48_571, 16),
                        (3, 1_500_001, 1 << 30), (2_000_000, 0, 8), (777_777, 777_778, 2)):
        a = _rand_sorted(S, rng, na, dup)
        b = _rand_sorted(S, rng, nb, dup)
        if S == "el":
            b["tag"] += np.uint32(1 << 24)
        want, _, _, _ = port.merge(S, a, b)
        got = mp.parallel_merge(to_dev(a, S, cuda), to_dev(b, S, cuda), 8, key_type=key_type(S))
        assert same(from_dev(got, S), want), (S, na, nb, dup)


def test_large_merge_unaligned_inputs(cuda, port):
    torch = _torch()
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(31)
    base_a = np.sort(rng.integers(0, 1 << 20, 1_300_000).astype(np.uint32))
    base_b = np.sort(rng.integers(0, 1 << 20, 1_300_000).astype(np.uint32))
    da, db = torch.from_numpy(base_a).to(cuda), torch.from_numpy(base_b).to(cuda)
    for oa, ob in ((1, 3), (2, 0), (3, 2)):
        a, b = base_a[oa:oa + 1_200_001], base_b[ob:ob + 1_100_000]
        want, _, _, _ = port.merge("u32", a, b)
        got = mp.parallel_merge(da[oa:oa + 1_200_001], db[ob:ob + 1_100_000], 4)
        assert np.array_equal(got.cpu().numpy(), want), (oa, ob)


def test_host_pipeline_many_chunks(cuda):
    """mp_merge_host's chunked PCIe pipeline (1 MiB chunks, read once per
    process, hence the subprocess): page-widened H2D copies at unaligned
    host offsets, ragged and empty sides, with and without values, against a
    stable numpy merge (ties to A)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1406_2628_b200 import _native as N
rng = np.random.default_rng(9)
bad = []
for kt, dt in ((0, np.uint32), (1, np.int32), (3, np.uint64), (4, np.int64)):
    for na, nb, dup, off in ((3_000_001, 2_500_003, 1 << 30, 1), (1_234_567, 0, 50, 3),
                             (5, 4_000_000, 7, 2), (2_000_000, 2_000_000, 1 << 20, 0)):
        ba = np.sort(rng.integers(0, dup, na + off).astype(dt))
        bb = np.sort(rng.integers(0, dup, nb + off).astype(dt))
        a, b = ba[off:], bb[off:]  # host pointers off the allocation start
        av = np.arange(na, dtype=np.uint32)
        bv = np.arange(nb, dtype=np.uint32) | np.uint32(1 << 31)
        cat = np.concatenate([a, b])
        perm = np.argsort(cat, kind="stable")
        for vals in (False, True):
            out = np.empty(na + nb, dtype=dt)
            outv = np.empty(na + nb, dtype=np.uint32) if vals else None
            p = lambda x: x.ctypes.data if x is not None else None
            N.check(N.lib.mp_merge_host(kt, p(a), p(av) if vals else None, na, p(b),
                                        p(bv) if vals else None, nb, p(out), p(outv), 0))
            ok = np.array_equal(out, cat[perm])
            if vals:
                ok = ok and np.array_equal(outv, np.concatenate([av, bv])[perm])
            if not ok:
                bad.append((kt, na, nb, vals))
print("BAD", bad)
sys.exit(1 if bad else 0)
'''
    from pathlib import Path
    env = dict(os.environ, MP_HOST_CHUNK_MB="1")
    r = subprocess.run([sys.executable, "-c", code, str(Path(__file__).resolve().parents[1])],
                       env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


_FUSED_SORT_CHECK = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import torch
from test_gpu_parity import _fused_round_cases
_fused_round_cases(torch.device("cuda", 0), sys.argv[2])
print("FUSED OK")
'''


@pytest.mark.parametrize("S", ("u32", "i32", "f32"))
@pytest.mark.parametrize("engine,quad", [("warp", "0"), ("warp", "1"), ("merge", "0"),
                                        ("merge", "1")])
def test_fused_round_sorts_vs_oracle(cuda, S, engine, quad):
    """Bare 32-bit sorts through each block sort -- K3w (default, 16384-key
    runs, warp bitonic levels + Merge Path passes) and the stable K3
    (MP_BLOCK_SORT=merge, 2048-key runs) -- then plain rounds or fused
    two-round passes (MP_SORT_QUAD=1, mp_quad.cuh) at every size.  The
    switches are read once per process, hence the subprocess."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _FUSED_SORT_CHECK, root, S], capture_output=True,
                       text=True, timeout=900,
                       env=dict(os.environ, MP_SORT_QUAD=quad, MP_BLOCK_SORT=engine))
    assert r.returncode == 0 and "FUSED OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def _fused_round_cases(cuda, S):
    """Sizes straddle run and group boundaries (runs of 16384 and 2048,
    groups of 4 runs) so the short last group has 1, 2 or 3 runs; inputs
    include heavy duplicates, all-equal, descending and (f32) signed zeros /
    NaNs."""
    from oracle import bindings
    from paper_1406_2628_b200 import mergepath as mp
    port = bindings.port()
    rng = np.random.default_rng(29)
    sizes = (511, 512, 513, 4095, 4096, 4097, 8191, 8193, 200_003, 1_000_000)
    for R in (16384, 2048):
        sizes += (4 * R - 1, 4 * R, 4 * R + 1, 5 * R + 7, 6 * R, 7 * R + 3, 16 * R + 1,
                  16 * R + 9 * R, 64 * R - 5)
    for n in sizes:
        for kind in ("dup3", "uniform", "equal", "desc"):
            if kind == "dup3":
                d = _rand_unsorted(S, rng, n, 3)
            elif kind == "uniform":
                d = _rand_unsorted(S, rng, n, 1 << 30)
            elif kind == "equal":
                d = _rand_unsorted(S, rng, n, 1)
            else:
                d = np.sort(_rand_unsorted(S, rng, n, 1 << 20))[::-1].copy()
            if S == "f32" and kind == "uniform":
                d.view(np.uint32)[::97] = 0x80000000  # -0.0
                d.view(np.uint32)[1::89] = 0x7FC00001  # NaN payloads
                d.view(np.uint32)[2::101] = 0xFFC00000
            want, _, _ = port.merge_sort(S, d)
            got = mp.parallel_merge_sort(to_dev(d, S, cuda), 4, key_type=key_type(S))
            assert same(from_dev(got, S), want), (S, n, kind)


def test_beyond_2_32_elements(cuda):
    """64-bit indexing end to end: a sort of 2^32 + 1001 u32 keys and a
    merge with |A| + |B| > 2^32, verified on the device in 2^28-element
    chunks (sortedness across chunk seams, per-chunk multiset fingerprint of
    the low 16 bits and the key sum)."""
    torch = _torch()
    from paper_1406_2628_b200 import _native as N
    free, _ = torch.cuda.mem_get_info()
    if free < (80 << 30):
        pytest.skip("needs ~60 GiB of device memory")
    st = torch.cuda.current_stream().cuda_stream
    C = 1 << 28

    def fingerprint(x):
        h = torch.zeros(65536, dtype=torch.int64, device=cuda)
        s = 0
        for i in range(0, x.numel(), C):
            v = x[i:i + C].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            h += torch.bincount(v & 0xFFFF, minlength=65536)
            s += int(v.sum())
        return h, s

    def sorted_u32(x):
        prev = None
        for i in range(0, x.numel(), C):
            v = x[i:i + C].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            if not bool((v[1:] >= v[:-1]).all()) or (prev is not None and int(v[0]) < prev):
                return False
            prev = int(v[-1])
        return True

    n = (1 << 32) + 1001
    x = torch.empty(n, dtype=torch.uint32, device=cuda)
    N.check(N.lib.mp_generate(0, 9, 0, n, x.data_ptr(), st))
    h0, s0 = fingerprint(x)
    N.check(N.lib.mp_sort(N.KEY_U32, x.data_ptr(), None, n, None, 0, st))
    torch.cuda.synchronize()
    assert sorted_u32(x)
    h1, s1 = fingerprint(x)
    assert s1 == s0 and torch.equal(h1, h0)
    na, nb = (1 << 31) + 3, (1 << 31) + 7
    a = x[:na].clone()
    del x
    b = torch.empty(nb, dtype=torch.uint32, device=cuda)
    N.check(N.lib.mp_generate(0, 2, 0, nb, b.data_ptr(), st))
    N.check(N.lib.mp_sort(N.KEY_U32, b.data_ptr(), None, nb, None, 0, st))
    out = torch.empty(na + nb, dtype=torch.uint32, device=cuda)
    N.check(N.lib.mp_merge(N.KEY_U32, a.data_ptr(), None, na, b.data_ptr(), None, nb,
                           out.data_ptr(), None, st))
    torch.cuda.synchronize()
    assert out.numel() > (1 << 32) and sorted_u32(out)
    ha, sa = fingerprint(a)
    hb, sb = fingerprint(b)
    ho, so = fingerprint(out)
    assert so == sa + sb and torch.equal(ho, ha + hb)


def _ref_or_skip():
    from oracle import bindings as B
    if not B.REF_LIB.exists():
        pytest.skip("oracle/_ref (the reference library) not built")
    return B


@pytest.mark.parametrize("config", ["2", "3a", "3b"])
def test_full_size_bit_exact_vs_reference(cuda, config):
    """BASELINE configs 2 and 3 at full size, byte for byte against the
    REFERENCE itself (oracle/_ref: parallel_merge_into on this host's cores)
    on the same input bytes: keys, and for config 3 the {key, value}
    records (values = source index, bit 31 marks B)."""
    torch = _torch()
    B = _ref_or_skip()
    from paper_1406_2628_b200 import mergepath as mp
    R = B.ref()
    team = R.team(B.host_cores())
    if config == "2":
        n = 1 << 28
        a = _sorted_dev(1, 1, n, cuda)
        b = _sorted_dev(1, 2, n, cuda)
        got = mp.parallel_merge(a, b, 8).cpu().numpy()
        want, _, _ = R.merge("i32", a.cpu().numpy(), b.cpu().numpy(), team=team)
        team.close()
        assert np.array_equal(got, want)
        return
    na, nb = 1 << 29, 1 << 25
    ka, kb = ((2, 2) if config == "3a" else (4, 3))
    a = _sorted_dev(ka, 1, na, cuda)
    b = _sorted_dev(kb, 2, nb, cuda)
    av = torch.arange(na, dtype=torch.int32, device=cuda).view(torch.uint32)
    bv = (torch.arange(nb, dtype=torch.int32, device=cuda)
          + torch.iinfo(torch.int32).min).view(torch.uint32)
    out, outv = mp.parallel_merge(a, b, 8, a_vals=av, b_vals=bv)
    ra = np.zeros(na, dtype=B.KV_DTYPE)
    ra["key"], ra["val"] = a.cpu().numpy(), av.cpu().numpy()
    rb = np.zeros(nb, dtype=B.KV_DTYPE)
    rb["key"], rb["val"] = b.cpu().numpy(), bv.cpu().numpy()
    del a, b, av, bv
    want, _, _ = R.merge("kv", ra, rb, team=team)
    team.close()
    del ra, rb
    assert np.array_equal(out.cpu().numpy(), want["key"])
    assert np.array_equal(outv.cpu().numpy(), want["val"])


def test_config5_full_size_bit_exact_vs_reference(cuda):
    """Config 5 on one GPU at full size (f32, |A| = |B| = 2^31, A ~ Normal,
    B ~ Exp, IEEE totalOrder), byte for byte against the reference's
    parallel merge with a totalOrder comparator on the same bytes."""
    torch = _torch()
    B = _ref_or_skip()
    from paper_1406_2628_b200 import _native as N
    st = torch.cuda.current_stream().cuda_stream
    n = 1 << 31
    ab = []
    for kind, seed in ((5, 1), (6, 2)):
        x = torch.empty(n, dtype=torch.float32, device=cuda)
        N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), st))
        N.check(N.lib.mp_sort(N.KEY_F32, x.data_ptr(), None, n, None, 0, st))
        ab.append(x)
    a, b = ab
    out = torch.empty(2 * n, dtype=torch.float32, device=cuda)
    N.check(N.lib.mp_merge(N.KEY_F32, a.data_ptr(), None, n, b.data_ptr(), None, n,
                           out.data_ptr(), None, st))
    torch.cuda.synchronize()
    ha, hb = a.cpu().numpy(), b.cpu().numpy()
    del a, b
    got = out.cpu().numpy()
    del out
    R = B.ref()
    team = R.team(B.host_cores())
    want, _, _ = R.merge("f32", ha, hb, team=team)
    team.close()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("S,n", [("u32", (1 << 26) + 12345), ("f32", (1 << 26) + 7),
                                 ("u64", (1 << 25) + 999)])
def test_host_sort_pipelined(cuda, S, n):
    """mp_sort_host over PCIe in chunks (each chunk sorted on the device
    while the next is copied in, then the remaining rounds): sizes of >= 4
    chunks, duplicates; u64 carries values to check stability."""
    from paper_1406_2628_b200 import _native as N
    rng = np.random.default_rng(31)
    kt = key_type(S)
    if S == "u64":
        x = rng.integers(0, 1 << 20, n, dtype=np.uint64)
        v = np.arange(n, dtype=np.uint32)
        out = np.empty_like(x)
        outv = np.empty_like(v)
        N.check(N.lib.mp_sort_host(kt, x.ctypes.data, v.ctypes.data, n, out.ctypes.data,
                                   outv.ctypes.data, 0))
        perm = np.argsort(x, kind="stable")
        assert np.array_equal(out, x[perm]) and np.array_equal(outv, v[perm])
        return
    x = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    x[::5] = 77
    if S == "f32":
        x[1::97] = 0x80000000  # -0.0 among the keys
    out = np.empty_like(x)
    N.check(N.lib.mp_sort_host(kt, x.ctypes.data, None, n, out.ctypes.data, None, 0))
    if S == "u32":
        assert np.array_equal(out, np.sort(x))
    else:
        img = np.where(x & 0x80000000, ~x, x | 0x80000000).astype(np.uint32)
        assert np.array_equal(out, x[np.argsort(img, kind="stable")])


def test_concurrent_calls_from_threads(cuda, port):
    """Merges and sorts issued concurrently from several host threads, each
    on its own stream (the library's scratch pool, host pipeline and launch
    counter are shared), including host-buffer calls; all bit-exact."""
    import threading
    torch = _torch()
    from paper_1406_2628_b200 import _native as N
    rng = np.random.default_rng(61)
    cases = []
    for k in range(6):
        na, nb = int(rng.integers(1, 3_000_000)), int(rng.integers(1, 3_000_000))
        a = np.sort(rng.integers(0, 1 << 20, na).astype(np.int32))
        b = np.sort(rng.integers(0, 1 << 20, nb).astype(np.int32))
        x = rng.integers(0, 1 << 32, 1_000_003, dtype=np.uint64).astype(np.uint32)
        cases.append((a, b, x))
    errors = []

    def work(k):
        try:
            a, b, x = cases[k]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
                out = torch.empty(len(a) + len(b), dtype=torch.int32, device="cuda")
                for _ in range(3):
                    N.check(N.lib.mp_merge(N.KEY_I32, da.data_ptr(), None, len(a), db.data_ptr(),
                                           None, len(b), out.data_ptr(), None, st.cuda_stream))
                dx = torch.from_numpy(x).cuda()
                N.check(N.lib.mp_sort(N.KEY_U32, dx.data_ptr(), None, len(x), None, 0,
                                      st.cuda_stream))
                st.synchronize()
                ho = np.empty(len(a) + len(b), dtype=np.int32)
                N.check(N.lib.mp_merge_host(N.KEY_I32, a.ctypes.data, None, len(a),
                                            b.ctypes.data, None, len(b), ho.ctypes.data, None, 0))
                want = np.sort(np.concatenate([a, b]), kind="stable")
                assert np.array_equal(out.cpu().numpy(), want), "device merge"
                assert np.array_equal(ho, want), "host merge"
                assert np.array_equal(dx.cpu().numpy(), np.sort(x)), "sort"
        except Exception as e:  # pragma: no cover
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def _extreme_pool(S):
    """Key values at the edges of each type's order."""
    if S == "f32":
        bits = [0x00000000, 0x80000000, 0x00000001, 0x80000001, 0x7F7FFFFF, 0xFF7FFFFF,
                0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000, 0x7FFFFFFF, 0xFFFFFFFF,
                0x3F800000, 0xBF800000, 0x007FFFFF, 0x807FFFFF]
        return np.array(bits, dtype=np.uint32)
    dt = {"u32": np.uint32, "i32": np.int32, "u64": np.uint64, "i64": np.int64}[S]
    info = np.iinfo(dt)
    vals = [info.min, info.min + 1, info.max, info.max - 1, 0, 1]
    if info.min < 0:
        vals += [-1, -2]
    if np.dtype(dt).itemsize == 4:
        vals += [0x7FFFFFFF if info.min < 0 else 0x80000000]
    else:
        vals += [(1 << 62)]
    return np.array(vals, dtype=dt)


def _order_sorted(S, x):
    if S == "f32":
        u = x.view(np.uint32)
        key = np.where(u & 0x80000000, ~u, u | 0x80000000)
        return u[np.argsort(key, kind="stable")]
    return np.sort(x, kind="stable")


@pytest.mark.parametrize("S", ("u32", "i32", "f32", "u64", "i64"))
def test_extreme_keys_merge_and_sort(cuda, port, S):
    """Keys at the type's extremes (min/max, sign boundaries; f32 +-0, +-inf,
    NaNs with payloads, denormals, FLT_MAX) drawn with heavy repetition,
    merged and sorted through the device, bit-exact vs the oracle; plus
    all-equal inputs at the maximum and the minimum key."""
    from paper_1406_2628_b200 import mergepath as mp
    rng = np.random.default_rng(71)
    pool = _extreme_pool(S)
    for n in (1, 7, 4095, 4097, 8193, 70_001):
        a = _order_sorted(S, pool[rng.integers(0, len(pool), n)])
        b = _order_sorted(S, pool[rng.integers(0, len(pool), n + 3)])
        want, _, _, _ = port.merge(S, a, b)
        got = mp.parallel_merge(to_dev(a, S, cuda), to_dev(b, S, cuda), 4, key_type=key_type(S))
        assert same(from_dev(got, S), want), (S, n, "merge")
        d = pool[rng.integers(0, len(pool), n)]
        want_s, _, _ = port.merge_sort(S, d)
        got_s = mp.parallel_merge_sort(to_dev(d, S, cuda), 4, key_type=key_type(S))
        assert same(from_dev(got_s, S), want_s), (S, n, "sort")
    for v in (pool.max() if S != "f32" else pool[-5], pool.min() if S != "f32" else pool[7]):
        d = np.full(10_007, v, dtype=pool.dtype)
        want_s, _, _ = port.merge_sort(S, d)
        got_s = mp.parallel_merge_sort(to_dev(d, S, cuda), 4, key_type=key_type(S))
        assert same(from_dev(got_s, S), want_s)


@pytest.mark.parametrize("fuse_tiles,k4_warp", [("0", "0"), ("2", "0"), ("0", "1000000")])
def test_split_search_paths_vs_oracle(cuda, fuse_tiles, k4_warp):
    """Merges and sorts up to a few waves of CTAs search their own split
    points in-kernel (SearchMap / RoundSearchMap, no K1/K4 launch), and
    somewhat larger sort rounds run K4 with a warp per boundary.  Re-run the
    random merge / sort / checksum parity tests with the in-kernel search off
    (MP_MERGE_FUSE_TILES=0: K1/K4 + K2 at every size), with a 2-tile
    threshold (the shapes straddle it) and with the warp K4 for every round,
    in a subprocess because the switches are read once per process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-m", "pytest", str(root / "tests" / "test_gpu_parity.py"),
                        "-q", "-x", "-p", "no:cacheprovider", "-k",
                        "random_merges or random_sorts or sort_with_values or checksum_vs"],
                       capture_output=True, text=True, timeout=1200, cwd=str(root),
                       env=dict(os.environ, MP_MERGE_FUSE_TILES=fuse_tiles,
                                MP_K4_WARP_TILES=k4_warp))
    assert r.returncode == 0 and " passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("S", ["i32", "u64"])
def test_pageable_host_spans_staged(cuda, port, S):
    """Host calls on pageable memory (numpy arrays, i.e. what a std::vector
    caller passes) go through the pinned staging slots and the copy pool:
    several chunks (1 MiB chunk override in a subprocess is not needed --
    the sizes span many 64 MiB chunks for u64 with values), unaligned
    sub-views, values; results equal the oracle and the pinned call."""
    import torch
    from paper_1406_2628_b200 import _native as N
    rng = np.random.default_rng(77)
    kt = key_type(S)
    dt = np.int32 if S == "i32" else np.uint64
    na, nb = (40_000_001, 27_000_013) if S == "i32" else (12_000_007, 9_000_001)
    a = np.sort(rng.integers(0, 1 << 20, na + 3).astype(dt))[3:]  # unaligned view
    b = np.sort(rng.integers(0, 1 << 20, nb).astype(dt))
    av = np.arange(na, dtype=np.uint32)
    bv = np.arange(nb, dtype=np.uint32) | np.uint32(1 << 31)
    out = np.empty(na + nb + 1, dtype=dt)[1:]
    outv = np.empty(na + nb, dtype=np.uint32)
    N.check(N.lib.mp_merge_host(kt, a.ctypes.data, av.ctypes.data, na, b.ctypes.data,
                                bv.ctypes.data, nb, out.ctypes.data, outv.ctypes.data, 0))
    want, wantv, _, _ = port.merge(S, a, b, av=av, bv=bv)
    assert np.array_equal(out, want) and np.array_equal(outv, wantv)
    # the pinned path gives the same bytes
    pa = torch.from_numpy(a.copy()).pin_memory()
    pb = torch.from_numpy(b.copy()).pin_memory()
    po = torch.empty(na + nb, dtype=pa.dtype).pin_memory()
    N.check(N.lib.mp_merge_host(kt, pa.data_ptr(), None, na, pb.data_ptr(), None, nb,
                                po.data_ptr(), None, 0))
    assert np.array_equal(po.numpy(), want)
    # the sort from pageable memory (chunked H2D staging + chunked D2H drain)
    x = rng.integers(0, 1 << 20, 3 * (1 << 24) + 5).astype(dt)
    v = np.arange(len(x), dtype=np.uint32)
    xo = np.empty_like(x)
    vo = np.empty_like(v)
    N.check(N.lib.mp_sort_host(kt, x.ctypes.data, v.ctypes.data, len(x), xo.ctypes.data,
                               vo.ctypes.data, 0))
    perm = np.argsort(x, kind="stable")
    assert np.array_equal(xo, x[perm]) and np.array_equal(vo, v[perm].astype(np.uint32))
