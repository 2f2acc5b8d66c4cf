"""Sort timing on the legacy default stream vs a created stream."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0)
n = 1 << 30
x = torch.empty(n, dtype=torch.uint32, device=dev)
N.check(N.lib.mp_generate(0, 4, 0, n, x.data_ptr(), 0))
out = torch.empty_like(x)
scr = torch.empty(N.lib.mp_sort_scratch_bytes(0, 0, n), dtype=torch.uint8, device=dev)
for name, s in (("legacy", torch.cuda.default_stream()), ("created", torch.cuda.Stream())):
    with torch.cuda.stream(s):
        st = s.cuda_stream
        f = lambda: N.check(N.lib.mp_sort_to(0, x.data_ptr(), None, out.data_ptr(), None, n, scr.data_ptr(), scr.numel(), st))
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(5): f()
        e1.record(s); torch.cuda.synchronize()
        print(json.dumps({"stream": name, "ms": e0.elapsed_time(e1) / 5}))
