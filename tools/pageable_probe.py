"""Host-span calls on pinned vs pageable memory (the drop-in's natural
callers pass std::vector = pageable memory): config-2 merge through
mp_merge_host and the config-4 sort through mp_sort_host, wall clock per
call, plus a byte check of the two results.  One JSON line per case."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1406_2628_b200 import _native as N  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream


def gen(kind, seed, n, dt, sort_kt=None):
    x = torch.empty(n, dtype=dt, device=dev)
    N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), st))
    if sort_kt is not None:
        N.check(N.lib.mp_sort(sort_kt, x.data_ptr(), None, n, None, 0, st))
    return x.cpu()


def timeit(f, reps=5):
    f()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t)
    return sorted(ts)[len(ts) // 2]


n = 1 << 28
a = gen(1, 1, n, torch.int32, N.KEY_I32)
b = gen(1, 2, n, torch.int32, N.KEY_I32)
res = {}
for mem in ("pinned", "pageable"):
    if mem == "pinned":
        ha, hb = a.pin_memory(), b.pin_memory()
        ho = torch.empty(2 * n, dtype=torch.int32).pin_memory()
        pa, pb, po = ha.data_ptr(), hb.data_ptr(), ho.data_ptr()
        keep = (ha, hb, ho)
    else:
        na_, nb_ = a.numpy().copy(), b.numpy().copy()
        no = np.empty(2 * n, dtype=np.int32)
        pa, pb, po = na_.ctypes.data, nb_.ctypes.data, no.ctypes.data
        keep = (na_, nb_, no)
    sec = timeit(lambda: N.check(N.lib.mp_merge_host(N.KEY_I32, pa, None, n, pb, None, n, po,
                                                     None, 0)))
    out = keep[2].numpy() if mem == "pinned" else keep[2]
    res[mem] = out.copy()
    print(json.dumps({"case": "config2 merge mp_merge_host", "memory": mem, "ms": sec * 1e3,
                      "elements_per_s": 2 * n / sec}), flush=True)
print(json.dumps({"case": "config2 merge", "pageable_equals_pinned":
                  bool(np.array_equal(res["pinned"], res["pageable"]))}))
del res, a, b
m = 1 << 30
x = gen(0, 4, m, torch.uint32)
res = {}
for mem in ("pinned", "pageable"):
    if mem == "pinned":
        hx = x.pin_memory()
        ho = torch.empty(m, dtype=torch.uint32).pin_memory()
        px, po = hx.data_ptr(), ho.data_ptr()
        out = ho
    else:
        nx = x.numpy().copy()
        no = np.empty(m, dtype=np.uint32)
        px, po = nx.ctypes.data, no.ctypes.data
        out = no
    sec = timeit(lambda: N.check(N.lib.mp_sort_host(N.KEY_U32, px, None, m, po, None, 0)),
                 reps=3)
    res[mem] = (out.numpy() if mem == "pinned" else out).copy()
    print(json.dumps({"case": "config4 sort mp_sort_host", "memory": mem, "ms": sec * 1e3,
                      "keys_per_s": m / sec}), flush=True)
print(json.dumps({"case": "config4 sort", "pageable_equals_pinned":
                  bool(np.array_equal(res["pinned"], res["pageable"]))}))
