"""Key files (§8f row 3) and the mergebench_b200 CLI contract (§8f row 1)
on the CPU: byte-identity with files written by the REFERENCE's dataio
(tests/golden/keyfiles/, recorded by make_keyfile_golden.py), the readers'
format detection and error mapping (dataio.cpp:33-98), and the tool's
gen / report subcommands and exit codes (mergebench.cpp; SPEC.md bench-cli:
0 ok, 1 usage, 2 I/O, 3 validation, 4 mismatch).  Device paths are in
tests/test_gpu_mergebench.py."""
from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden" / "keyfiles"
TOOL = ROOT / "paper_1406_2628_b200" / "bin" / "mergebench_b200"
CASES = json.loads((GOLD / "index.json").read_text())


def _N():
    from paper_1406_2628_b200 import _native as N
    return N


def read_keys(path) -> np.ndarray:
    N = _N()
    n, b = C.c_uint64(), C.c_int()
    N.check(N.lib.mp_keyfile_count(str(path).encode(), C.byref(n), C.byref(b)))
    out = np.zeros(max(n.value, 1), dtype=np.int64)
    got = C.c_uint64()
    N.check(N.lib.mp_keyfile_read(str(path).encode(), out.ctypes.data, n.value, C.byref(got)))
    return out[:got.value]


def write_keys(path, keys, binary) -> None:
    N = _N()
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    N.check(N.lib.mp_keyfile_write(str(path).encode(), keys.ctypes.data if len(keys) else None,
                                   len(keys), int(binary)))


def stem(c):
    return f"gen_{c['dist']}_{c['na']}_{c['nb']}_{c['seed']}"


@pytest.mark.parametrize("case", CASES, ids=stem)
def test_reference_files_round_trip(tmp_path, case):
    """Read the reference's binary and text files; writing the keys back
    gives byte-identical files."""
    for side, n in (("a", case["na"]), ("b", case["nb"])):
        kb = read_keys(GOLD / f"{stem(case)}_{side}.bin")
        kt = read_keys(GOLD / f"{stem(case)}_{side}.text")
        assert len(kb) == n and np.array_equal(kb, kt)
        assert np.all(kb[:-1] <= kb[1:])
        for fmt, binary in (("bin", 1), ("text", 0)):
            p = tmp_path / f"x.{fmt}"
            write_keys(p, kb, binary)
            assert p.read_bytes() == (GOLD / f"{stem(case)}_{side}.{fmt}").read_bytes()


@pytest.mark.parametrize("case", CASES, ids=stem)
@pytest.mark.parametrize("fmt", ["bin", "text"])
def test_tool_gen_matches_reference_bytes(tmp_path, case, fmt):
    """`mergebench_b200 gen` reproduces the reference generator's files."""
    a, b = tmp_path / f"a.{fmt}", tmp_path / f"b.{fmt}"
    r = subprocess.run([str(TOOL), "gen", "--dist", case["dist"], "--na", str(case["na"]),
                        "--nb", str(case["nb"]), "--seed", str(case["seed"]), "--out-a", str(a),
                        "--out-b", str(b), "--format", fmt], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert a.read_bytes() == (GOLD / f"{stem(case)}_a.{fmt}").read_bytes()
    assert b.read_bytes() == (GOLD / f"{stem(case)}_b.{fmt}").read_bytes()


def test_reader_format_detection_and_errors(tmp_path):
    p = tmp_path / "t.txt"
    p.write_text("5\n\n-3\n  12  \n9223372036854775807\n-9223372036854775808\n")
    assert read_keys(p).tolist() == [5, -3, 12, 2**63 - 1, -2**63]
    p.write_text("1\n2\nx3\n")
    with pytest.raises(ValueError, match="line 3"):  # std::invalid_argument
        read_keys(p)
    p.write_text("1 2\n")
    with pytest.raises(ValueError, match="line 1"):
        read_keys(p)
    with pytest.raises(OSError):  # std::runtime_error: cannot open
        read_keys(tmp_path / "missing.bin")
    q = tmp_path / "trunc.bin"
    write_keys(q, np.arange(10), True)
    q.write_bytes(q.read_bytes()[:-8])  # header says 10, 9 present
    with pytest.raises(OSError, match="truncated"):
        read_keys(q)
    q.write_bytes(b"MPKB0001\x05")  # header cut short
    with pytest.raises(OSError, match="truncated"):
        read_keys(q)
    e = tmp_path / "empty.bin"
    write_keys(e, np.zeros(0, dtype=np.int64), True)
    assert e.read_bytes() == b"MPKB0001" + bytes(8) and len(read_keys(e)) == 0
    (tmp_path / "empty.txt").write_text("")
    assert len(read_keys(tmp_path / "empty.txt")) == 0
    N = _N()
    small = np.zeros(2, dtype=np.int64)
    got = C.c_uint64()
    with pytest.raises(ValueError, match="capacity"):
        N.check(N.lib.mp_keyfile_read(str(GOLD / "gen_uniform_300_200_1_a.bin").encode(),
                                      small.ctypes.data, 2, C.byref(got)))


def _run(*args):
    return subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True)


def test_tool_usage_and_validation_exit_codes(tmp_path):
    assert _run().returncode == 1
    assert _run("bogus").returncode == 1
    assert _run("cachesim").returncode == 1
    assert _run("gen", "--na", "3").returncode == 1  # missing required options
    assert _run("gen", "--na", "3", "--nb", "3", "--out-a", tmp_path / "a", "--out-b",
                tmp_path / "b", "--dist", "gaussian").returncode == 1
    a = GOLD / "gen_uniform_300_200_1_a.bin"
    assert _run("merge", "--a", a, "--b", a, "--reps", "2").returncode == 1
    assert _run("merge", "--a", a, "--b", a, "--nope", "1").returncode == 1
    # I/O: missing input file -> 2; unsorted input -> 3 (both before any GPU use)
    assert _run("merge", "--a", tmp_path / "none.bin", "--b", a).returncode == 2
    u = tmp_path / "unsorted.txt"
    u.write_text("3\n1\n2\n")
    r = _run("merge", "--a", u, "--b", a)
    assert r.returncode == 3 and "not sorted" in r.stderr
    assert _run("gen", "--na", "1", "--nb", "1", "--out-a", tmp_path / "no/such/dir/a",
                "--out-b", tmp_path / "b").returncode == 2


def test_tool_report_rerender(tmp_path):
    """report: re-render a saved JSON report as CSV / JSON (the reference's
    column order, %.9g floats, empty cells for null)."""
    rep = {"meta": {"tool": "mergebench_b200", "op": "merge"}, "rows": [
        {"op": "merge", "variant": "regular", "n": 2097152, "p": 1, "cache_elems": 0, "reps": 5,
         "median_seconds": 0.000123456789012, "mean_seconds": 0.000125, "verified": True,
         "speedup_vs_p1": 1.0, "partition_comparisons": 0, "merge_steps": 2097152,
         "merge_rounds": None},
        {"op": "merge", "variant": "regular", "n": 2097152, "p": 8, "cache_elems": 0, "reps": 5,
         "median_seconds": 1.5e-05, "mean_seconds": 1.6e-05, "verified": True,
         "speedup_vs_p1": 8.23045267, "partition_comparisons": 147, "merge_steps": 2097152,
         "merge_rounds": None}]}
    f = tmp_path / "r.json"
    f.write_text(json.dumps(rep))
    r = _run("report", "--in", f)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[0] == ("op,variant,n,p,cache_elems,reps,median_seconds,mean_seconds,"
                        "speedup_vs_p1,partition_comparisons,merge_steps,merge_rounds,verified")
    assert lines[1] == "merge,regular,2097152,1,0,5,0.000123456789,0.000125,1,0,2097152,,true"
    assert lines[2] == "merge,regular,2097152,8,0,5,1.5e-05,1.6e-05,8.23045267,147,2097152,,true"
    r = _run("report", "--in", f, "--format", "json", "--out", tmp_path / "o.json")
    assert r.returncode == 0
    assert json.loads((tmp_path / "o.json").read_text()) == rep
    (tmp_path / "bad.json").write_text("{\"meta\": {}}")
    assert _run("report", "--in", tmp_path / "bad.json").returncode == 3
    (tmp_path / "bad2.json").write_text("{not json")
    assert _run("report", "--in", tmp_path / "bad2.json").returncode == 3
    assert _run("report", "--in", tmp_path / "nope.json").returncode == 2
