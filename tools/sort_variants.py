"""A/B sort-round thread shapes (variant libraries) on config 4."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
vd = os.path.join(os.path.dirname(N.LIB_PATH), "variants")
libs = {"default": N.lib}
for f in sorted(os.listdir(vd)):
    if f.startswith(sys.argv[1] if len(sys.argv) > 1 else "libmergepath_b200_svt"):
        L = C.CDLL(os.path.join(vd, f))
        for name, res, args in N.SIGNATURES:
            g = getattr(L, name); g.restype = res; g.argtypes = args
        libs[f] = L
n = 1 << 30
x = torch.empty(n, dtype=torch.uint32, device=dev)
N.check(N.lib.mp_generate(0, 4, 0, n, x.data_ptr(), st))
ref = torch.sort(x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values
for name, L in libs.items():
    out = torch.empty_like(x)
    scr = torch.empty(L.mp_sort_scratch_bytes(0, 0, n), dtype=torch.uint8, device=dev)
    f = lambda: L.mp_sort_to(0, x.data_ptr(), None, out.data_ptr(), None, n, scr.data_ptr(), scr.numel(), st)
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ok = torch.equal(out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, ref)
    print(json.dumps({"lib": name, "ms": e0.elapsed_time(e1) / 5, "ok": ok}))
