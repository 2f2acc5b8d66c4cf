"""A/B plain-merge thread shapes (variant libraries): configs 2, 3a, random u32."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
vd = os.path.join(os.path.dirname(N.LIB_PATH), "variants")
libs = {"default": N.lib}
for f in sorted(os.listdir(vd)):
    if f.startswith("libmergepath_b200_mvt"):
        L = C.CDLL(os.path.join(vd, f))
        for name, res, args in N.SIGNATURES:
            g = getattr(L, name); g.restype = res; g.argtypes = args
        libs[f] = L
def gen(kind, seed, n, dt):
    x = torch.empty(n, dtype=dt, device=dev)
    N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), st)); return x
cases = [("cfg2", 1, 1, torch.int32, 1 << 28, 1 << 28, False), ("u32rand", 0, 0, torch.uint32, 1 << 28, 1 << 28, False),
         ("cfg3a", 2, 3, torch.uint64, 1 << 29, 1 << 25, True)]
for name, kind, kt, dt, na, nb, vals in cases:
    a, b = gen(kind, 1, na, dt), gen(kind, 2, nb, dt)
    for x in (a, b): N.check(N.lib.mp_sort(kt, x.data_ptr(), None, x.numel(), None, 0, st))
    av = torch.arange(na, dtype=torch.int32, device=dev) if vals else None
    bv = torch.arange(nb, dtype=torch.int32, device=dev) if vals else None
    outv = torch.empty(na + nb, dtype=torch.int32, device=dev) if vals else None
    p = lambda t: t.data_ptr() if t is not None else None
    ref = torch.empty(na + nb, dtype=dt, device=dev)
    N.check(N.lib.mp_merge(kt, a.data_ptr(), p(av), na, b.data_ptr(), p(bv), nb, ref.data_ptr(), p(outv), st))
    res = {"case": name}
    for ln, L in libs.items():
        out = torch.empty_like(ref)
        f = lambda: L.mp_merge(kt, a.data_ptr(), p(av), na, b.data_ptr(), p(bv), nb, out.data_ptr(), p(outv), st)
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        res[ln.replace("libmergepath_b200_", "")] = (round(e0.elapsed_time(e1) / 20, 4),
                                                     torch.equal(out.view(torch.uint8), ref.view(torch.uint8)))
    print(json.dumps(res))
