"""mergebench_b200 merge / sort on the GPU (§8f rows 1 and 3): key files
streamed into HBM, every repetition verified against std::merge / std::sort
before its row is reported, the reference's row schema and statistics, and
the key-file device load/store paths."""
from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
TOOL = ROOT / "paper_1406_2628_b200" / "bin" / "mergebench_b200"
pytestmark = pytest.mark.gpu

ROW_KEYS = {"op", "variant", "n", "p", "cache_elems", "reps", "median_seconds", "mean_seconds",
            "speedup_vs_p1", "partition_comparisons", "merge_steps", "merge_rounds", "verified"}


def _run(*args):
    r = subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True, timeout=600)
    return r


def _gen(tmp_path, dist, na, nb, seed=3):
    a, b = tmp_path / f"{dist}_a.bin", tmp_path / f"{dist}_b.bin"
    r = _run("gen", "--dist", dist, "--na", na, "--nb", nb, "--seed", seed, "--out-a", a,
             "--out-b", b)
    assert r.returncode == 0, r.stderr
    return a, b


@pytest.mark.parametrize("dist", ["uniform", "all_equal", "disjoint_ranges", "interleaved"])
@pytest.mark.parametrize("residency", ["device", "host", "file"])
def test_merge_rows_verified(cuda, port, tmp_path, dist, residency):
    a, b = _gen(tmp_path, dist, 300_001, 199_999)
    r = _run("merge", "--a", a, "--b", b, "--threads", "1,4,8", "--reps", "3",
             "--residency", residency)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["meta"]["na"] == 300_001 and rep["meta"]["residency"] == residency
    rows = rep["rows"]
    assert [x["p"] for x in rows] == [1, 4, 8]
    for x in rows:
        assert set(x) == ROW_KEYS and x["verified"] and x["n"] == 500_000
        assert x["merge_steps"] == 500_000 and x["speedup_vs_p1"] > 0
    assert rows[0]["partition_comparisons"] == 0  # p=1: no interior search
    # the reference's own statistics on the same keys (partition_comparisons
    # of a p-way search, core.hpp:99-146)
    from test_keyfile import read_keys
    A, B = read_keys(a), read_keys(b)
    for x in rows[1:]:
        _, want = port.partition("i64", A, B, x["p"])
        assert x["partition_comparisons"] == want


def test_merge_segmented_register_csv(cuda, tmp_path):
    a, b = _gen(tmp_path, "uniform", 1 << 18, (1 << 18) + 5)
    r = _run("merge", "--a", a, "--b", b, "--variant", "segmented", "--threads", "1,2",
             "--sink", "register", "--format", "csv", "--reps", "3")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[0].startswith("op,variant,n,p,cache_elems")
    assert len(lines) == 1 + 3 * 2  # default caches 3N/{2,5,10} x threads
    assert all(line.endswith(",true") and ",segmented," in line for line in lines[1:])


@pytest.mark.parametrize("residency", ["device", "host", "file"])
def test_sort_rows_verified(cuda, tmp_path, residency):
    rng = np.random.default_rng(5)
    x = rng.integers(-2**62, 2**62, 123_457, dtype=np.int64)
    x[::7] = 42  # duplicates
    f = tmp_path / "keys.bin"
    from test_keyfile import write_keys
    write_keys(f, x, True)
    for variant in ("plain", "cache_efficient"):
        r = _run("sort", "--in", f, "--variant", variant, "--threads", "1,3", "--reps", "3",
                 "--residency", residency)
        assert r.returncode == 0, r.stderr
        rows = json.loads(r.stdout)["rows"]
        assert len(rows) == 2 and all(row["verified"] for row in rows)
        assert all(row["merge_rounds"] is not None for row in rows)


def test_keyfile_device_load_store(cuda, tmp_path):
    import torch
    from paper_1406_2628_b200 import _native as N
    from test_keyfile import read_keys, write_keys
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(1)
    for n in (0, 1, 1000, (32 << 20) // 8 * 2 + 12345):  # crosses two staging chunks
        x = rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64)
        f = tmp_path / f"k{n}.bin"
        write_keys(f, x, True)
        d = torch.empty(max(n, 1), dtype=torch.int64, device=cuda)
        got = C.c_uint64()
        N.check(N.lib.mp_keyfile_load(str(f).encode(), d.data_ptr(), n, C.byref(got), 0, st))
        assert got.value == n and np.array_equal(d[:n].cpu().numpy(), x)
        g = tmp_path / f"s{n}.bin"
        N.check(N.lib.mp_keyfile_store(str(g).encode(), d.data_ptr(), n, 0, st))
        assert g.read_bytes() == f.read_bytes()
    t = tmp_path / "k.txt"
    write_keys(t, np.array([3, -1, 7]), False)
    d = torch.empty(3, dtype=torch.int64, device=cuda)
    got = C.c_uint64()
    N.check(N.lib.mp_keyfile_load(str(t).encode(), d.data_ptr(), 3, C.byref(got), 0, st))
    assert d.cpu().tolist() == [3, -1, 7]
    with pytest.raises(ValueError, match="capacity"):
        N.check(N.lib.mp_keyfile_load(str(t).encode(), d.data_ptr(), 2, C.byref(got), 0, st))


def test_keyfile_merge_file_to_file(cuda, port, tmp_path):
    """mp_keyfile_merge: two sorted key files -> one, through the host
    pipeline with the files mapped (ingest overlapped with the merge).  The
    output file is byte-identical to write_keys(oracle merge): binary inputs
    spanning several pipeline chunks with heavy duplicates (ties to A are
    invisible in bare keys, but every chunk boundary lands inside a run of
    equal keys), a text input, empty inputs, and a missing file."""
    from paper_1406_2628_b200 import _native as N
    from test_keyfile import read_keys, write_keys
    rng = np.random.default_rng(7)
    cases = [
        (np.sort(rng.integers(-50, 50, 9_000_001)), np.sort(rng.integers(-50, 50, 7_654_321)), True, True),
        (np.sort(rng.integers(-2**62, 2**62, 3_000_000)), np.sort(rng.integers(-2**62, 2**62, 17)), True, False),
        (np.sort(rng.integers(0, 1000, 1001)), np.zeros(0, dtype=np.int64), False, True),
        (np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.int64), True, True),
    ]
    for k, (a, b, bin_a, bin_b) in enumerate(cases):
        fa, fb, fo, fw = (tmp_path / f"{k}_{x}" for x in ("a", "b", "out", "want"))
        write_keys(fa, a, bin_a)
        write_keys(fb, b, bin_b)
        got = C.c_uint64()
        N.check(N.lib.mp_keyfile_merge(str(fa).encode(), str(fb).encode(), str(fo).encode(),
                                       C.byref(got), 0))
        assert got.value == len(a) + len(b)
        want, _, _, _ = port.merge("i64", a.astype(np.int64), b.astype(np.int64))
        write_keys(fw, want, True)
        assert fo.read_bytes() == fw.read_bytes(), k
        assert np.array_equal(read_keys(fo), want)
    with pytest.raises(OSError):
        N.check(N.lib.mp_keyfile_merge(str(tmp_path / "missing").encode(), str(fb).encode(),
                                       str(fo).encode(), None, 0))
    before = fa.read_bytes()
    with pytest.raises(ValueError, match="one of the inputs"):  # would truncate a mapped input
        N.check(N.lib.mp_keyfile_merge(str(fa).encode(), str(fb).encode(), str(fa).encode(),
                                       None, 0))
    assert fa.read_bytes() == before
    with pytest.raises(ValueError, match="is the input"):
        N.check(N.lib.mp_keyfile_sort(str(fa).encode(), str(fa).encode(), None, 0))


def test_keyfile_sort_file_to_file(cuda, port, tmp_path):
    """mp_keyfile_sort: key file in, sorted key file out (mapped files through
    mp_sort_host's pipeline), byte-identical to write_keys(oracle sort)."""
    from paper_1406_2628_b200 import _native as N
    from test_keyfile import write_keys
    rng = np.random.default_rng(11)
    for k, (x, binary) in enumerate([(rng.integers(-2**62, 2**62, 5_000_003), True),
                                     (rng.integers(-3, 3, 70_001), False),
                                     (np.zeros(0, dtype=np.int64), True)]):
        fi, fo, fw = (tmp_path / f"{k}_{s}" for s in ("in", "out", "want"))
        write_keys(fi, x, binary)
        got = C.c_uint64()
        N.check(N.lib.mp_keyfile_sort(str(fi).encode(), str(fo).encode(), C.byref(got), 0))
        assert got.value == len(x)
        want, _, _ = port.merge_sort("i64", x.astype(np.int64))
        write_keys(fw, want, True)
        assert fo.read_bytes() == fw.read_bytes(), k
