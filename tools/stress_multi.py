"""Randomised parity stress of the multi-GPU building blocks on the GPU:
mp_merge_pieces (random piece splits incl. empty pieces, random output
ranges, values), mp_multi_merge and mp_multi_sort (random shard tables on
the visible devices, blocking and stream-ordered), random key types and
duplicate densities, each checked bit-exactly against the C restatement
(oracle/).  usage: python tools/stress_multi.py [cases] [seed]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
from oracle import bindings
from paper_1406_2628_b200 import _native as N
from conftest import same
from test_gpu_parity import _rand_sorted, _rand_unsorted, to_dev, from_dev, key_type

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1406)
G = torch.cuda.device_count()
port = bindings.port()
bad, t0 = 0, time.time()
kinds = {"pieces": 0, "multi_merge": 0, "multi_sort": 0}


def cuts(n, k):
    c = np.sort(rng.integers(0, n + 1, k - 1)) if k > 1 else np.array([], dtype=np.int64)
    return np.concatenate([[0], c, [n]]).astype(np.int64)


def shards(x, S, c, vals=None):
    keep, tab = [], []
    for g in range(len(c) - 1):
        d = int(rng.integers(0, G))
        dev = torch.device("cuda", d)
        part = x[c[g]:c[g + 1]]
        t = to_dev(part, S, dev)  # (an empty part keeps the key dtype)
        v = (torch.from_numpy(vals[c[g]:c[g + 1]].copy()).to(dev) if vals is not None else None)
        keep += [t, v]
        tab.append((d, t.data_ptr() if len(part) else None,
                    v.data_ptr() if v is not None and len(part) else None, len(part)))
    return keep, tab


for c in range(cases):
    S = str(rng.choice(["u32", "i32", "f32", "u64", "i64", "el"]))
    dup = int(rng.choice([2, 16, 1000, 1 << 20, 1 << 40]))
    op = str(rng.choice(list(kinds)))
    vals = S != "el" and rng.random() < 0.5
    n1 = int(np.exp(rng.uniform(0, np.log(1 << 22))))
    n2 = int(np.exp(rng.uniform(0, np.log(1 << 22)))) if rng.random() < 0.85 else int(rng.integers(0, 3))
    kt = key_type(S)
    try:
        if op in ("pieces", "multi_merge"):
            a, b = _rand_sorted(S, rng, n1, dup), _rand_sorted(S, rng, n2, dup)
            if S == "el":
                b["tag"] += np.uint32(1 << 24)
            av = np.arange(n1, dtype=np.uint32) if vals else None
            bv = (np.arange(n2, dtype=np.uint32) | np.uint32(1 << 31)) if vals else None
            want, wantv, _, _ = port.merge(S, a, b, av=av, bv=bv)
            n = n1 + n2
            if op == "pieces":
                torch.cuda.set_device(0)
                ka, ta = shards(a, S, cuts(n1, int(rng.integers(1, 17))), av)
                kb, tb = shards(b, S, cuts(n2, int(rng.integers(1, 17))), bv)
                o0 = int(rng.integers(0, n + 1))
                o1 = int(rng.integers(o0, n + 1))
                out = to_dev(want[:max(o1 - o0, 1)], S, torch.device("cuda", 0)).clone()
                outv = torch.zeros(max(o1 - o0, 1), dtype=torch.uint32, device="cuda:0") if vals else None
                pa = N.pieces_array([(p[1], p[2], p[3]) for p in ta])
                pb = N.pieces_array([(p[1], p[2], p[3]) for p in tb])
                N.check(N.lib.mp_merge_pieces(kt, pa, len(ta), pb, len(tb), o0, o1, out.data_ptr(),
                                              outv.data_ptr() if vals else None,
                                              torch.cuda.current_stream().cuda_stream))
                torch.cuda.synchronize()
                ok = o1 == o0 or (same(from_dev(out, S)[:o1 - o0], want[o0:o1]) and
                                  (not vals or np.array_equal(outv.cpu().numpy()[:o1 - o0], wantv[o0:o1])))
            else:
                ka, ta = shards(a, S, cuts(n1, int(rng.integers(1, 17))), av)
                kb, tb = shards(b, S, cuts(n2, int(rng.integers(1, 17))), bv)
                oc = cuts(n, int(rng.integers(1, 9)))
                zeros = np.zeros(n, dtype=want.dtype)
                ko, to = shards(zeros, S, oc, np.zeros(n, dtype=np.uint32) if vals else None)
                N.check(N.lib.mp_multi_merge(kt, N.shards_array(ta), len(ta), N.shards_array(tb),
                                             len(tb), N.shards_array(to), len(to), None))
                got = np.concatenate([from_dev(k, S) for k in ko[0::2]]) if n else want
                ok = same(got[:n], want)
                if vals and n:
                    gv = np.concatenate([v.cpu().numpy() for v in ko[1::2]])
                    ok = ok and np.array_equal(gv, wantv)
        else:
            d = _rand_unsorted(S, rng, n1, dup)
            v = np.arange(n1, dtype=np.uint32) if vals else None
            want, wantv, _ = port.merge_sort(S, d, vals=v)
            kx, tx = shards(d, S, cuts(n1, int(rng.integers(1, 17))), v)
            N.check(N.lib.mp_multi_sort(kt, N.shards_array(tx), len(tx), None))
            got = np.concatenate([from_dev(k, S) for k in kx[0::2]]) if n1 else want
            ok = same(got[:n1], want)
            if vals and n1:
                gv = np.concatenate([x.cpu().numpy() for x in kx[1::2]])
                ok = ok and np.array_equal(gv, wantv)
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", c, S, op, n1, n2, dup, vals, repr(e)[:300], flush=True)
    kinds[op] += 1
    if not ok:
        bad += 1
        print("MISMATCH", c, S, op, n1, n2, dup, vals, flush=True)
print(f"stress_multi: {cases} cases {kinds} on {G} GPU(s), {bad} failures, "
      f"{time.time() - t0:.0f} s", flush=True)
sys.exit(1 if bad else 0)
