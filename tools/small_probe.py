"""Latency of small device-resident merges and sorts (the one-wave regime
where CTAs search their own split points; MP_MERGE_FUSE_TILES=0 turns that
off for an A/B).  CUDA events around 50 back-to-back calls."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1406_2628_b200 import _native as N

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
res = {}
for n in [int(x) for x in __import__("os").environ.get("SIZES", "65536,262144,1048576,4194304").split(",")]:
    x = torch.randint(0, 2**31 - 1, (n,), dtype=torch.int64, device=dev).to(torch.int32)
    y = torch.empty_like(x)
    sb = N.lib.mp_sort_scratch_bytes(N.KEY_U32, 0, n)
    scr = torch.empty(max(sb, 16), dtype=torch.uint8, device=dev)
    a = torch.sort(x[: n // 2])[0]
    b = torch.sort(x[n // 2:])[0]
    o = torch.empty(n, dtype=torch.int32, device=dev)

    def sort():
        N.check(N.lib.mp_sort_to(N.KEY_U32, x.data_ptr(), None, y.data_ptr(), None, n,
                                 scr.data_ptr(), sb, st.cuda_stream))

    def merge():
        N.check(N.lib.mp_merge(N.KEY_U32, a.data_ptr(), None, a.numel(), b.data_ptr(), None,
                               b.numel(), o.data_ptr(), None, st.cuda_stream))
    for name, fn in (("sort", sort), ("merge", merge)):
        for _ in range(5):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[f"{name}_{n}_us"] = round(e0.elapsed_time(e1) / 50 * 1000, 2)
    assert torch.equal(y, torch.sort(x)[0])
print(json.dumps(res))
