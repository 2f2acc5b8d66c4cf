"""The C ABI boundary on the CPU container: the library loads, exports every
symbol include/mergepath_b200.h declares, host-only helpers answer, argument
validation follows the reference, and compute calls fail loudly (no CPU
fallback) when there is no GPU."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mergepath_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(mp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1406_2628_b200 import _native as N
    syms = declared_symbols()
    assert len(syms) >= 14
    bound = {name for name, _, _ in N.SIGNATURES}
    assert set(syms) == bound, "ctypes binding out of sync with the header"
    lib = C.CDLL(str(N.LIB_PATH))
    for s in syms:
        assert hasattr(lib, s), s


def test_exports_via_nm():
    import shutil
    import subprocess
    from paper_1406_2628_b200 import _native as N
    if not shutil.which("nm"):
        pytest.skip("nm missing")
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (mp_[a-z0-9_]+)$", out, re.M))
    assert set(declared_symbols()) <= exported


def test_host_helpers():
    from paper_1406_2628_b200 import _native as N
    assert N.lib.mp_abi_version() >= 100
    assert [N.lib.mp_key_size(k) for k in range(6)] == [4, 4, 4, 8, 8, 16]
    assert N.lib.mp_key_size(99) == 0
    assert N.lib.mp_sort_scratch_bytes(0, 0, 1) == 0
    b = N.lib.mp_sort_scratch_bytes(0, 0, 1 << 30)
    assert b >= (1 << 32)  # one N-sized ping-pong buffer of u32
    assert N.lib.mp_sort_scratch_bytes(0, 1, 1 << 20) > N.lib.mp_sort_scratch_bytes(0, 0, 1 << 20)


def test_invalid_arguments_without_gpu():
    from paper_1406_2628_b200 import _native as N
    a = np.arange(4, dtype=np.uint32)
    # p == 0 is rejected before any device work (core.hpp:139-140)
    assert N.lib.mp_partition(0, a.ctypes.data, 4, a.ctypes.data, 4, 0, a.ctypes.data,
                              None, None) == N.MP_ERR_INVALID
    assert b"positive" in N.lib.mp_last_error()
    assert N.lib.mp_merge(0, None, None, 4, None, None, 0, None, None,
                          None) == N.MP_ERR_INVALID
    assert N.lib.mp_generate(9, 0, 0, 1, None, None) == N.MP_ERR_INVALID
    assert N.lib.mp_merge_host(42, a.ctypes.data, None, 4, a.ctypes.data, None, 4,
                               a.ctypes.data, None, 0) == N.MP_ERR_UNSUPPORTED


def test_compute_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1406_2628_b200 import _native as N
    from paper_1406_2628_b200 import mergepath as mp
    a = np.arange(4, dtype=np.uint32)
    out = np.zeros(8, dtype=np.uint32)
    rc = N.lib.mp_merge_host(0, a.ctypes.data, None, 4, a.ctypes.data, None, 4,
                             out.ctypes.data, None, 0)
    assert rc == N.MP_ERR_CUDA
    with pytest.raises(N.MergePathError):
        mp.parallel_merge(a, a, 2)


def test_python_api_validation_is_host_side():
    from paper_1406_2628_b200 import mergepath as mp
    a = np.arange(4, dtype=np.uint32)
    with pytest.raises(ValueError):
        mp.parallel_merge(a, a, 0)
    with pytest.raises(ValueError):
        mp.segmented_parallel_merge(a, a, 2, 2)
    with pytest.raises(ValueError):
        mp.segmented_parallel_merge(a, a, 0, 48)
    with pytest.raises(ValueError):
        mp.plan_segments(a, a, 2, 0)
    with pytest.raises(ValueError):
        mp.partition(a, a, 0)
    with pytest.raises(ValueError):
        mp.parallel_merge_sort(a, 0)
    with pytest.raises(ValueError):
        mp.cache_efficient_parallel_sort(a, 2, 2)
    with pytest.raises(ValueError):
        mp.cache_efficient_parallel_sort(a, 0, 48)
    with pytest.raises(TypeError):
        mp.parallel_merge(a, a.astype(np.int32), 1)


def test_sort_plan_kats(kats):
    from paper_1406_2628_b200 import mergepath as mp
    for c in kats["sort_plan"]:
        v = mp.SortVariant.plain if c["variant"] == "plain" else mp.SortVariant.cache_efficient
        plan = mp.make_sort_plan(v, c["n"], c["C"])
        for key in ("block_size", "blocks", "tree_levels"):
            if key in c:
                assert getattr(plan, key) == c[key], c["src"]
    gp = mp.gpu_sort_plan(1 << 30)
    assert gp.block_size == 2048 and gp.tree_levels == 19
    gp = mp.gpu_sort_plan(1 << 30, bare32=True)  # config 4: 16384-key runs, 16 rounds
    assert gp.block_size == 16384 and gp.tree_levels == 16


def test_custom_comparator_rejected():
    """A comparator the kernels do not implement raises instead of being
    ignored (the C++ drop-in rejects it at compile time, b200_backend.hpp)."""
    import operator
    from paper_1406_2628_b200 import mergepath as mp
    a = np.arange(4, dtype=np.uint32)
    desc = lambda x, y: x > y  # noqa: E731
    for call in (lambda c: mp.parallel_merge(a, a, 2, comp=c),
                 lambda c: mp.parallel_merge_into(a, a, np.empty(8, np.uint32), 2, comp=c),
                 lambda c: mp.segmented_parallel_merge(a, a, 2, 30, comp=c),
                 lambda c: mp.parallel_merge_checksum(a, a, 2, comp=c),
                 lambda c: mp.parallel_merge_sort(a, 2, comp=c),
                 lambda c: mp.cache_efficient_parallel_sort(a, 2, 30, comp=c)):
        with pytest.raises(TypeError):
            call(desc)
        with pytest.raises(TypeError):
            call(mp.TOTAL_ORDER_LESS)  # the f32 order on u32 keys
    f = np.zeros(2, dtype=np.float32)
    with pytest.raises(TypeError):
        mp.parallel_merge(f, f, 1, comp=operator.lt)  # std::less<float>: -0 == +0
    # the allow-listed names pass the check (then fail loudly without a GPU)
    mp._check_comp(mp.LESS, N_KEY("u32"))
    mp._check_comp(operator.lt, N_KEY("i64"))
    mp._check_comp(mp.TOTAL_ORDER_LESS, N_KEY("f32"))
    mp._check_comp(mp.KEY_LESS, N_KEY("element"))


def N_KEY(name):
    from paper_1406_2628_b200 import _native as N
    return {"u32": N.KEY_U32, "i64": N.KEY_I64, "f32": N.KEY_F32,
            "element": N.KEY_ELEMENT}[name]
