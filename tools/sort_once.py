"""One 2^30-key u32 sort (for ncu launch lists / captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
n = int(os.environ.get("N", 1 << 30))
x = torch.empty(n, dtype=torch.uint32, device=dev)
N.check(N.lib.mp_generate(0, 4, 0, n, x.data_ptr(), st))
out = torch.empty_like(x)
scr = torch.empty(N.lib.mp_sort_scratch_bytes(0, 0, n), dtype=torch.uint8, device=dev)
for _ in range(int(os.environ.get("REPS", 1))):
    N.check(N.lib.mp_sort_to(0, x.data_ptr(), None, out.data_ptr(), None, n, scr.data_ptr(), scr.numel(), st))
torch.cuda.synchronize()
print("ok")
