"""The single-process multi-GPU C ABI (mp_multi_merge / mp_multi_sort over
a {device, keys, vals, len} shard table) on the GPU box.

* tests/cpp/test_multi_gpu.cpp -- a C++ caller with no Python in the path --
  merges u64 keys (+ u32 values) and sorts u32 keys (+ values, stability
  visible) over 1..7 shards, blocking and stream-ordered, ragged and empty
  shards, against std::merge / std::stable_sort.  On the one-GPU lease every
  shard lives on device 0 (distinct streams, same-device "peers"); with more
  GPUs visible it also runs with one shard per GPU.
* f32 totalOrder and i64 keys through ctypes, against the C restatement.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu
BIN = ROOT / "paper_1406_2628_b200" / "bin" / "test_multi_gpu"


def test_cpp_caller_one_gpu(cuda):
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "OK: 0 failure(s)" in r.stdout


def test_cpp_caller_all_gpus(cuda):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("one GPU visible: covered by test_cpp_caller_one_gpu")
    r = subprocess.run([str(BIN)] + [str(d) for d in range(n)], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def _shards(torch, x, cuts, dev):
    keep = [x[cuts[g]:cuts[g + 1]].clone() for g in range(len(cuts) - 1)]
    return keep, [(dev.index or 0, t.data_ptr() if t.numel() else None, None, t.numel())
                  for t in keep]


@pytest.mark.parametrize("S", ["f32", "i64"])
def test_multi_sort_and_merge_key_types(cuda, port, S):
    import torch
    from paper_1406_2628_b200 import _native as N
    rng = np.random.default_rng(97)
    n = 777_777
    if S == "f32":
        x = rng.standard_normal(n).astype(np.float32)
        x[::50] = -0.0
        x[1::50] = 0.0
        kt, t = N.KEY_F32, torch.from_numpy(x).to(cuda)
    else:
        x = rng.integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
        kt, t = N.KEY_I64, torch.from_numpy(x).to(cuda)
    cuts = [0, 100_000, 100_000, 400_000, n]
    keep, tab = _shards(torch, t, cuts, cuda)
    arr = N.shards_array(tab)
    N.check(N.lib.mp_multi_sort(kt, arr, len(tab), None))
    got = torch.cat(keep).cpu().numpy()
    want, _, _ = port.merge_sort(S, x.view(np.uint32) if S == "f32" else x)
    assert got.view(want.dtype).tobytes() == want.tobytes()
    # merge the sorted halves back through mp_multi_merge into 3 output shards
    h = n // 2
    a, b = torch.from_numpy(want[:h].copy()).to(cuda), torch.from_numpy(want[h:].copy()).to(cuda)
    if S == "f32":
        a, b = a.view(torch.float32), b.view(torch.float32)
    ka, ta = _shards(torch, a, [0, h // 3, h], cuda)
    kb, tb = _shards(torch, b, [0, 5, n - h], cuda)
    out = torch.empty(n, dtype=a.dtype, device=cuda)
    ko, to = _shards(torch, out, [0, 1, n // 2, n], cuda)
    N.check(N.lib.mp_multi_merge(kt, N.shards_array(ta), 2, N.shards_array(tb), 2,
                                 N.shards_array(to), 3, None))
    m, _, _, _ = port.merge(S, want[:h], want[h:])
    assert torch.cat(ko).cpu().numpy().view(m.dtype).tobytes() == m.tobytes()


def test_multi_sort_values_with_empty_first_shard(cuda, port):
    """Values ride along when ANY shard carries them -- an empty first shard
    has no value pointer (regression found by tools/stress_multi.py)."""
    import torch
    from paper_1406_2628_b200 import _native as N
    rng = np.random.default_rng(5)
    x = rng.integers(0, 7, 301).astype(np.uint32)
    v = np.arange(301, dtype=np.uint32)
    want, wantv, _ = port.merge_sort("u32", x, vals=v)
    cuts = [0, 0, 2, 150, 301]
    keys = [torch.from_numpy(x[cuts[g]:cuts[g + 1]].copy()).to(cuda) for g in range(4)]
    vals = [torch.from_numpy(v[cuts[g]:cuts[g + 1]].copy()).to(cuda) for g in range(4)]
    tab = [(0, k.data_ptr() if k.numel() else None, w.data_ptr() if w.numel() else None,
            k.numel()) for k, w in zip(keys, vals)]
    N.check(N.lib.mp_multi_sort(N.KEY_U32, N.shards_array(tab), 4, None))
    assert np.array_equal(torch.cat(keys).cpu().numpy(), want)
    assert np.array_equal(torch.cat(vals).cpu().numpy(), wantv)
    # the same table through the merge: A = the sorted first half, B = the rest
    h = 150
    a_k = [torch.from_numpy(want[:h].copy()).to(cuda)]
    b_k = [torch.from_numpy(want[h:].copy()).to(cuda)]
    a_v = [torch.from_numpy(np.arange(h, dtype=np.uint32)).to(cuda)]
    b_v = [torch.from_numpy(np.arange(301 - h, dtype=np.uint32) | np.uint32(1 << 31)).to(cuda)]
    out_k = [torch.empty(0, dtype=torch.uint32, device=cuda),
             torch.empty(301, dtype=torch.uint32, device=cuda)]
    out_v = [torch.empty(0, dtype=torch.uint32, device=cuda),
             torch.empty(301, dtype=torch.uint32, device=cuda)]
    N.check(N.lib.mp_multi_merge(
        N.KEY_U32, N.shards_array([(0, a_k[0].data_ptr(), a_v[0].data_ptr(), h)]), 1,
        N.shards_array([(0, b_k[0].data_ptr(), b_v[0].data_ptr(), 301 - h)]), 1,
        N.shards_array([(0, None, None, 0), (0, out_k[1].data_ptr(), out_v[1].data_ptr(), 301)]),
        2, None))
    m, mv, _, _ = port.merge("u32", want[:h], want[h:], av=a_v[0].cpu().numpy(),
                             bv=b_v[0].cpu().numpy())
    assert np.array_equal(out_k[1].cpu().numpy(), m) and np.array_equal(out_v[1].cpu().numpy(), mv)


def test_python_multi_sort_and_merge(cuda, port):
    """multigpu.multi_sort / multi_merge (the shard-table ABI from Python),
    with values and per-shard streams."""
    import torch
    from paper_1406_2628_b200 import multigpu as mg
    rng = np.random.default_rng(8)
    x = rng.integers(0, 1000, 500_003).astype(np.int32)
    v = np.arange(len(x), dtype=np.uint32)
    want, wantv, _ = port.merge_sort("i32", x, vals=v)
    cuts = [0, 7, 250_000, 250_001, len(x)]
    ks = [torch.from_numpy(x[cuts[g]:cuts[g + 1]].copy()).to(cuda) for g in range(4)]
    vs = [torch.from_numpy(v[cuts[g]:cuts[g + 1]].copy()).to(cuda) for g in range(4)]
    streams = [torch.cuda.Stream(cuda) for _ in range(4)]
    mg.multi_sort(ks, vals=vs, streams=streams)
    for s in streams:
        s.synchronize()
    assert np.array_equal(torch.cat(ks).cpu().numpy(), want)
    assert np.array_equal(torch.cat(vs).cpu().numpy(), wantv)
    h = 123_456
    a = [torch.from_numpy(want[:h].copy()).to(cuda)]
    b = [torch.from_numpy(want[h:h + 1000].copy()).to(cuda),
         torch.from_numpy(want[h + 1000:].copy()).to(cuda)]
    out = [torch.empty(n, dtype=torch.int32, device=cuda) for n in (1, len(want) - 1)]
    mg.multi_merge(a, b, out)
    m, _, _, _ = port.merge("i32", want[:h], want[h:])
    assert np.array_equal(torch.cat(out).cpu().numpy(), m)
