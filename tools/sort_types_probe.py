"""Device-resident sort rates per key type at 2^28 keys (and u32 + values):
where the stable path (K3 + plain rounds) stands against the bare 32-bit path
(K3w + fused round pairs)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
n = int(os.environ.get("N", 1 << 28))
def run(name, kt, width, vals):
    x = torch.empty(n * width // 4, dtype=torch.int32, device=dev)
    gk = {4: 0, 8: 2}[width]
    N.check(N.lib.mp_generate(gk, 4, 0, n, x.data_ptr(), st))
    v = torch.arange(n, dtype=torch.int32, device=dev) if vals else None
    out = torch.empty_like(x); ov = torch.empty_like(v) if vals else None
    scr = torch.empty(N.lib.mp_sort_scratch_bytes(kt, 1 if vals else 0, n), dtype=torch.uint8, device=dev)
    f = lambda: N.check(N.lib.mp_sort_to(kt, x.data_ptr(), v.data_ptr() if vals else None, out.data_ptr(),
                                         ov.data_ptr() if vals else None, n, scr.data_ptr(), scr.numel(), st))
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"case": name, "n": n, "ms": round(ms, 3), "keys_per_s": n / ms * 1e3,
                      "bytes_per_key": width + (4 if vals else 0)}))
run("u32 bare", N.KEY_U32, 4, False)
run("u32 + u32 values", N.KEY_U32, 4, True)
run("u64 bare", N.KEY_U64, 8, False)
run("u64 + u32 values", N.KEY_U64, 8, True)
