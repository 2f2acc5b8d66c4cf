"""The reference's OWN test suites, compiled unchanged against the drop-in
headers (include/mergepath/*.hpp) and linked to libmergepath_b200.so.

oracle/Makefile (target ref_tests, run by __graft_entry__.build() where
/root/reference exists) builds, into oracle/_ref/:
  ref_unit_tests  -- proj/tests/test_core.cpp, test_parallel.cpp,
                     test_sort.cpp (29 doctest cases) on tests/cpp/doctest.h
  ref_acceptance  -- proj/tests/acceptance.cpp (criteria 1-10 gate, 11 is
                     informational) with the reference's cachesim/dataio
The binaries travel to the GPU box prebuilt; /root/reference does not.
"""
from __future__ import annotations

import os
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref"

pytestmark = pytest.mark.gpu


def _run(name: str, timeout: int):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = str(ROOT / "paper_1406_2628_b200") + ":" + env.get(
        "LD_LIBRARY_PATH", "")
    return subprocess.run([str(exe)], capture_output=True, text=True, timeout=timeout,
                          env=env)


def test_reference_unit_tests_pass_on_dropin(cuda):
    r = _run("ref_unit_tests", 600)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-2000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m and int(m.group(1)) == 29 and int(m.group(3)) == 0


def test_reference_acceptance_gating_criteria_pass_on_dropin(cuda):
    r = _run("ref_acceptance", 1800)
    print(r.stdout)
    print(r.stderr[-2000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion")]
    assert len(lines) == 11
    for ln in lines:
        num = int(ln.split()[1])
        if num <= 10:  # 11 = wall-clock speedup of p=4 vs p=1: informational
            assert " PASS" in ln, ln
    assert r.returncode == 0
