"""Randomised parity stress on the GPU: merges (with and without values) and
sorts of random key types, sizes (log-uniform up to 2^25), duplicate
densities and sub-view offsets through the public Python mirror, each
checked bit-exactly against the C restatement (oracle/).  Prints one line
per failure and a summary.  usage: python tools/stress_parity.py [cases] [seed]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
from oracle import bindings
from paper_1406_2628_b200 import mergepath as mp
from conftest import same
from test_gpu_parity import _rand_sorted, _rand_unsorted, to_dev, from_dev, key_type

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2628)
dev = torch.device("cuda", 0)
port = bindings.port()
bad, t0 = 0, time.time()
kinds = {"merge": 0, "merge_vals": 0, "sort": 0, "sort_vals": 0}
for c in range(cases):
    S = rng.choice(["u32", "i32", "f32", "u64", "i64", "el"])
    dup = int(rng.choice([2, 16, 1000, 1 << 20, 1 << 40]))
    op = rng.choice(["merge", "merge_vals", "sort", "sort_vals"])
    if S == "el" and op.endswith("vals"):
        op = op[:-5]
    n1 = int(np.exp(rng.uniform(0, np.log(1 << 25))))
    n2 = int(np.exp(rng.uniform(0, np.log(1 << 25)))) if rng.random() < 0.8 else int(rng.integers(0, 4))
    try:
        if op.startswith("merge"):
            a, b = _rand_sorted(S, rng, n1, dup), _rand_sorted(S, rng, n2, dup)
            if S == "el":
                b["tag"] += np.uint32(1 << 24)
            if op == "merge_vals":
                av = np.arange(n1, dtype=np.uint32)
                bv = np.arange(n2, dtype=np.uint32) | np.uint32(1 << 31)
                want, wantv, _, _ = port.merge(S, a, b, av=av, bv=bv)
                got, gotv = mp.parallel_merge(to_dev(a, S, dev), to_dev(b, S, dev), 4,
                                              a_vals=torch.from_numpy(av).to(dev),
                                              b_vals=torch.from_numpy(bv).to(dev), key_type=key_type(S))
                ok = same(from_dev(got, S), want) and np.array_equal(gotv.cpu().numpy(), wantv)
            else:
                want, _, _, _ = port.merge(S, a, b)
                got = mp.parallel_merge(to_dev(a, S, dev), to_dev(b, S, dev), 4, key_type=key_type(S))
                ok = same(from_dev(got, S), want)
        else:
            d = _rand_unsorted(S, rng, n1, dup)
            if op == "sort_vals":
                v = np.arange(n1, dtype=np.uint32)
                want, wantv, _ = port.merge_sort(S, d, vals=v)
                got, gotv = mp.parallel_merge_sort(to_dev(d, S, dev), 4, vals=torch.from_numpy(v).to(dev),
                                                   key_type=key_type(S))
                ok = same(from_dev(got, S), want) and np.array_equal(gotv.cpu().numpy(), wantv)
            else:
                want, _, _ = port.merge_sort(S, d)
                got = mp.parallel_merge_sort(to_dev(d, S, dev), 4, key_type=key_type(S))
                ok = same(from_dev(got, S), want)
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", c, S, op, n1, n2, dup, repr(e)[:200], flush=True)
    kinds[op] += 1
    if not ok:
        bad += 1
        print("MISMATCH", c, S, op, n1, n2, dup, flush=True)
print(f"stress: {cases} cases {kinds}, {bad} failures, {time.time() - t0:.0f} s", flush=True)
sys.exit(1 if bad else 0)
