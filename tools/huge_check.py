"""64-bit indexing check: sort of 2^32 + 1000 u32 keys and merge with
|A| + |B| > 2^32 (i32), verified by properties on the device."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
res = {}
n = (1 << 32) + 1000
x = torch.empty(n, dtype=torch.uint32, device=dev)
N.check(N.lib.mp_generate(0, 9, 0, n, x.data_ptr(), st))
h0 = torch.bincount((x.view(torch.int32) & 0xFFFF).long(), minlength=65536)  # multiset fingerprint
t = time.time()
N.check(N.lib.mp_sort(0, x.data_ptr(), None, n, None, 0, st)); torch.cuda.synchronize()
res["sort_s"] = round(time.time() - t, 3)
xi = x.view(torch.int32).long() & 0xFFFFFFFF
res["sort_sorted"] = bool((xi[1:] >= xi[:-1]).all())
res["sort_same_multiset"] = bool(torch.equal(torch.bincount((x.view(torch.int32) & 0xFFFF).long(), minlength=65536), h0))
del xi
na, nb = (1 << 31) + 3, (1 << 31) + 7
a = x[:na].view(torch.int32).clone(); del x
b = torch.empty(nb, dtype=torch.int32, device=dev)
N.check(N.lib.mp_generate(1, 2, 0, nb, b.data_ptr(), st)); N.check(N.lib.mp_sort(1, b.data_ptr(), None, nb, None, 0, st))
a = torch.sort(a).values  # i32 order
out = torch.empty(na + nb, dtype=torch.int32, device=dev)
N.check(N.lib.mp_merge(1, a.data_ptr(), None, na, b.data_ptr(), None, nb, out.data_ptr(), None, st)); torch.cuda.synchronize()
res["merge_sorted"] = bool((out[1:] >= out[:-1]).all())
res["merge_sum"] = bool(out.long().sum() == a.long().sum() + b.long().sum())
print(json.dumps(res))
