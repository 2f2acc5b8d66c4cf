"""A/B the tile size of the K1+K2 merge engine (variant libraries)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
os.environ["MP_MERGE_ENGINE"] = "tiles"
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
libs = {"256": N.lib}
vd = os.path.join(os.path.dirname(N.LIB_PATH), "variants")
for nt in ("512", "1024"):
    L = C.CDLL(os.path.join(vd, f"libmergepath_b200_nt{nt}.so"))
    for name, res, args in N.SIGNATURES:
        f = getattr(L, name); f.restype = res; f.argtypes = args
    libs[nt] = L
def gen(kind, seed, n, dt):
    x = torch.empty(n, dtype=dt, device=dev)
    N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), st)); return x
for kind, kt, dt, n in ((1, 1, torch.int32, 1 << 28), (0, 0, torch.uint32, 1 << 28), (2, 3, torch.uint64, 1 << 27)):
    a, b = gen(kind, 1, n, dt), gen(kind, 2, n, dt)
    for x in (a, b): N.check(N.lib.mp_sort(kt, x.data_ptr(), None, n, None, 0, st))
    ref = torch.empty(2 * n, dtype=dt, device=dev)
    N.check(N.lib.mp_merge(kt, a.data_ptr(), None, n, b.data_ptr(), None, n, ref.data_ptr(), None, st))
    res = {"kt": kt}
    for nt, L in libs.items():
        out = torch.empty_like(ref)
        f = lambda: L.mp_merge(kt, a.data_ptr(), None, n, b.data_ptr(), None, n, out.data_ptr(), None, st)
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res[nt] = (round(ms, 4), torch.equal(out.view(torch.uint8), ref.view(torch.uint8)))
    print(json.dumps(res))
