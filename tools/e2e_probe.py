"""e2e host-buffer merge: wall time per call vs chunk size, plus a per-stage
breakdown of one call (H2D, merge, D2H alone)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
n = 1 << 28
def gen(seed):
    x = torch.empty(n, dtype=torch.int32, device=dev)
    N.check(N.lib.mp_generate(1, seed, 0, n, x.data_ptr(), st))
    N.check(N.lib.mp_sort(1, x.data_ptr(), None, n, None, 0, st)); return x
a, b = gen(1), gen(2)
ha, hb = a.cpu().pin_memory(), b.cpu().pin_memory()
ho = torch.empty(2 * n, dtype=torch.int32).pin_memory()
f = lambda: N.check(N.lib.mp_merge_host(1, ha.data_ptr(), None, n, hb.data_ptr(), None, n, ho.data_ptr(), None, 0))
f(); f()
ts = []
for _ in range(5):
    t = time.perf_counter(); f(); ts.append(time.perf_counter() - t)
print(json.dumps({"chunk_mb": os.environ.get("MP_HOST_CHUNK_MB", "16"), "ms": [round(x * 1e3, 2) for x in ts],
                  "elements_per_s": 2 * n / min(ts)}))
