"""Time mp_sort at a given size (argv[1] = log2-ish n spec like 2^31+5)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0); st = torch.cuda.current_stream().cuda_stream
n = eval(sys.argv[1].replace("^", "**"))
x = torch.empty(n, dtype=torch.uint32, device=dev)
N.check(N.lib.mp_generate(0, 9, 0, n, x.data_ptr(), st)); torch.cuda.synchronize()
for rep in range(3):
    t = time.time()
    N.check(N.lib.mp_sort(0, x.data_ptr(), None, n, None, 0, st)); torch.cuda.synchronize()
    print(sys.argv[1], "rep", rep, "sort s", round(time.time() - t, 3), flush=True)
