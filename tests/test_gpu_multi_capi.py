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
