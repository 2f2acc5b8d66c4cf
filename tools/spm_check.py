"""Quick A/B of the two merge engines on the GPU (correctness + timing)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
def gen(kind, seed, n, dt):
    x = torch.empty(n, dtype=dt, device=dev)
    N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), st))
    return x
for kind, kt, dt, n in ((1, 1, torch.int32, 1 << 28), (0, 0, torch.uint32, 1 << 28), (2, 3, torch.uint64, 1 << 27)):
    a, b = gen(kind, 1, n, dt), gen(kind, 2, n, dt)
    for x in (a, b):
        N.check(N.lib.mp_sort(kt, x.data_ptr(), None, n, None, 0, st))
    out = torch.empty(2 * n, dtype=dt, device=dev)
    ref = torch.empty_like(out)
    # reference engine: tiles (via env is static; call the two-phase API = tiles)
    ws = torch.empty(N.lib.mp_merge_workspace_bytes(kt, n, n), dtype=torch.uint8, device=dev)
    N.check(N.lib.mp_merge_plan(kt, a.data_ptr(), n, b.data_ptr(), n, ws.data_ptr(), st))
    N.check(N.lib.mp_merge_execute(kt, a.data_ptr(), None, n, b.data_ptr(), None, n, ref.data_ptr(), None, ws.data_ptr(), st))
    torch.cuda.synchronize()
    N.check(N.lib.mp_merge(kt, a.data_ptr(), None, n, b.data_ptr(), None, n, out.data_ptr(), None, st))
    torch.cuda.synchronize()
    ok = torch.equal(out.view(torch.uint8), ref.view(torch.uint8))
    def timeit(fn, reps=20):
        for _ in range(3): fn()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    t_spm = timeit(lambda: N.lib.mp_merge(kt, a.data_ptr(), None, n, b.data_ptr(), None, n, out.data_ptr(), None, st))
    def tiles():
        N.lib.mp_merge_plan(kt, a.data_ptr(), n, b.data_ptr(), n, ws.data_ptr(), st)
        N.lib.mp_merge_execute(kt, a.data_ptr(), None, n, b.data_ptr(), None, n, ref.data_ptr(), None, ws.data_ptr(), st)
    t_tiles = timeit(tiles)
    byts = 2 * n * a.element_size() * 2
    print(json.dumps({"kt": kt, "n": 2 * n, "equal": ok, "spm_ms": t_spm, "tiles_ms": t_tiles,
                      "spm_GBps": byts / t_spm / 1e6, "tiles_GBps": byts / t_tiles / 1e6}))
