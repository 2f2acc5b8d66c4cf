"""u32 keys + u32 values merge timing (2^27 + 2^27), for tile-shape A/B."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
n = 1 << 27
def gen(seed):
    x = torch.empty(n, dtype=torch.uint32, device=dev)
    N.check(N.lib.mp_generate(0, seed, 0, n, x.data_ptr(), st))
    N.check(N.lib.mp_sort(0, x.data_ptr(), None, n, None, 0, st)); return x
a, b = gen(1), gen(2)
av = torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32); bv = av.clone()
out = torch.empty(2 * n, dtype=torch.uint32, device=dev); outv = torch.empty_like(out)
f = lambda: N.check(N.lib.mp_merge(0, a.data_ptr(), av.data_ptr(), n, b.data_ptr(), bv.data_ptr(), n, out.data_ptr(), outv.data_ptr(), st))
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"lib": os.environ.get("MP_NATIVE_LIB", "default")[-12:], "ms": round(ms, 4), "GBps": round(2 * n * 16 / ms / 1e6)}))
