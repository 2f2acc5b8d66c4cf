"""Does the ALU-bound block sort overlap with HBM-bound merges on a B200?

Times (CUDA events): (a) one 2^30-key u32 sort (mp_sort_to); (b) a chain of
M merges of 2^28 + 2^28 u32 keys (mp_merge, HBM-bound K1 + K2); (c) both at
once on two streams (the merges on a high-priority stream).  If (c) is well
below (a) + (b), the sort's block-sort phase can hide under HBM-bound work.
usage: python tools/overlap_probe.py [M]"""
import sys
import torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1406_2628_b200 import _native as N

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = torch.device("cuda", 0)
n = 1 << 30
x = torch.randint(0, 2**31 - 1, (n,), dtype=torch.int64, device=dev).to(torch.int32)
y = torch.empty_like(x)
sb = N.lib.mp_sort_scratch_bytes(N.KEY_U32, 0, n)
scr = torch.empty(sb, dtype=torch.uint8, device=dev)
a = torch.sort(torch.randint(0, 2**31 - 1, (1 << 28,), dtype=torch.int64, device=dev))[0].to(torch.int32)
b = torch.sort(torch.randint(0, 2**31 - 1, (1 << 28,), dtype=torch.int64, device=dev))[0].to(torch.int32)
o = torch.empty(1 << 29, dtype=torch.int32, device=dev)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
s1 = torch.cuda.Stream(dev)
s2 = torch.cuda.Stream(dev, priority=int(__import__("os").environ.get("PRIO", "-1")))


def sort(st):
    N.check(N.lib.mp_sort_to(N.KEY_U32, x.data_ptr(), None, y.data_ptr(), None, n,
                             scr.data_ptr(), sb, st.cuda_stream))


def merges(st):
    for _ in range(M):
        N.check(N.lib.mp_merge(N.KEY_U32, a.data_ptr(), None, a.numel(), b.data_ptr(), None,
                               b.numel(), o.data_ptr(), None, st.cuda_stream))


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    s2.wait_event(e0)
    fn()
    ev = torch.cuda.Event()
    ev.record(s2)
    s1.wait_stream(s2)
    e1.record(s1)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for _ in range(2):
    ta = timed(lambda: sort(s1))
    tb = timed(lambda: merges(s2))
    tc = timed(lambda: (merges(s2), sort(s1)))
    print(f"sort {ta:.2f} ms, {M} merges {tb:.2f} ms, sum {ta + tb:.2f}, concurrent {tc:.2f} ms "
          f"(saved {ta + tb - tc:.2f})", flush=True)
