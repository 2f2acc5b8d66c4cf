"""Block-sort A/B (env MP_BLOCK_SORT=warp|bare|merge, MP_SORT_QUAD=1 in separate
processes): correctness vs torch.sort and sort timings."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
res = {"block_sort": os.environ.get("MP_BLOCK_SORT", "default"), "quad": os.environ.get("MP_SORT_QUAD", "0")}
for kt, dt, kind in ((0, torch.uint32, 0), (1, torch.int32, 1), (2, torch.float32, 5)):
    n = 1 << 30 if kt == 0 else (1 << 26) + 12345
    x = torch.empty(n, dtype=dt, device=dev)
    N.check(N.lib.mp_generate(kind, 4, 0, n, x.data_ptr(), st))
    if kt == 2:
        x[::1001] = -0.0
        x[1::1003] = 0.0
    out = torch.empty_like(x)
    scr = torch.empty(N.lib.mp_sort_scratch_bytes(kt, 0, n), dtype=torch.uint8, device=dev)
    f = lambda: N.check(N.lib.mp_sort_to(kt, x.data_ptr(), None, out.data_ptr(), None, n, scr.data_ptr(), scr.numel(), st))
    f(); torch.cuda.synchronize()
    if kt == 0:
        ref = torch.sort(x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values
        ok = torch.equal(out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, ref)
    elif kt == 1:
        ok = torch.equal(out, torch.sort(x).values)
    else:
        u = x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        img = torch.where(u >= 0x80000000, u ^ 0xFFFFFFFF, u | 0x80000000)
        ok = torch.equal((out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF), torch.gather(u, 0, torch.sort(img).indices))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): f()
    e1.record(); torch.cuda.synchronize()
    res[f"kt{kt}"] = {"n": n, "ok": bool(ok), "ms": round(e0.elapsed_time(e1) / 3, 3)}
print(json.dumps(res))
