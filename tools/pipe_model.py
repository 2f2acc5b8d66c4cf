"""Replicates mp_merge_host's chunk pipeline in Python to find where the
e2e time goes: (a) copies only with the pipeline's dependencies, (b) + the
merge per chunk, (c) event timestamps of each stage per chunk."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1406_2628_b200 import _native as N
dev = torch.device("cuda", 0)
n = 1 << 28
st0 = torch.cuda.current_stream().cuda_stream
def gen(seed):
    x = torch.empty(n, dtype=torch.int32, device=dev)
    N.check(N.lib.mp_generate(1, seed, 0, n, x.data_ptr(), st0))
    N.check(N.lib.mp_sort(1, x.data_ptr(), None, n, None, 0, st0)); return x
a, b = gen(1), gen(2)
ha, hb = a.cpu().pin_memory(), b.cpu().pin_memory()
ho = torch.empty(2 * n, dtype=torch.int32).pin_memory()
A, B = ha.numpy(), hb.numpy()
slots = int(os.environ.get("SLOTS", "4"))
Q = int(os.environ.get("Q_MB", "64")) << 18  # elements
bufa = [torch.empty(Q, dtype=torch.int32, device=dev) for _ in range(slots)]
bufb = [torch.empty(Q, dtype=torch.int32, device=dev) for _ in range(slots)]
bufo = [torch.empty(Q, dtype=torch.int32, device=dev) for _ in range(slots)]
ws = [torch.empty(N.lib.mp_merge_workspace_bytes(1, Q, Q) // 8 + 8, dtype=torch.int64, device=dev) for _ in range(slots)]
sh, sc, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def split(d):
    lo, hi = max(0, d - n), min(d, n)
    while lo < hi:
        m = (lo + hi) // 2
        if B[d - 1 - m] < A[m]: hi = m
        else: lo = m + 1
    return lo
bounds = list(range(0, 2 * n, Q)) + [2 * n]
splits = [split(d) for d in bounds]
def run(merge=True, trace=None, dep=True, split_h2d=True, src2=None):
    evd = [None] * slots
    for k in range(len(bounds) - 1):
        s = k % slots
        d0, d1 = bounds[k], bounds[k + 1]
        a0, a1 = splits[k], splits[k + 1]
        b0, b1 = d0 - a0, d1 - a1
        with torch.cuda.stream(sh):
            if evd[s] is not None: sh.wait_event(evd[s])
            e_h0 = torch.cuda.Event(enable_timing=True); e_h0.record()
            if src2 is not None:
                o = (d0 // 2) % (n - Q); h = (d1 - d0) // 2
                bufa[s][:h].copy_(src2[0][o:o + h], non_blocking=True)
                bufb[s][:d1 - d0 - h].copy_(src2[1][o + h:o + d1 - d0], non_blocking=True)
            elif split_h2d:
                bufa[s][:a1 - a0].copy_(ha[a0:a1], non_blocking=True)
                bufb[s][:b1 - b0].copy_(hb[b0:b1], non_blocking=True)
            else:
                o = (d0 // 2) % (n - Q); bufa[s][:d1 - d0].copy_(ha[o:o + d1 - d0], non_blocking=True)
            e_h = torch.cuda.Event(enable_timing=True); e_h.record()
        with torch.cuda.stream(sc):
            sc.wait_event(e_h)
            if merge:
                N.check(N.lib.mp_merge(1, bufa[s].data_ptr(), None, a1 - a0, bufb[s].data_ptr(), None, b1 - b0,
                                       bufo[s].data_ptr(), None, sc.cuda_stream))
            e_c = torch.cuda.Event(enable_timing=True); e_c.record()
        with torch.cuda.stream(sd):
            if dep: sd.wait_event(e_c)
            ho[d0:d1].copy_(bufo[s][:d1 - d0], non_blocking=True)
            evd[s] = torch.cuda.Event(enable_timing=True); evd[s].record()
        if trace is not None: trace.append((e_h0, e_h, e_c, evd[s]))
def timeit(fn):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(3):
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return round(best * 1e3, 2)
res = {"Q_MB": Q >> 18, "slots": slots, "copies_only_ms": timeit(lambda: run(False)),
       "copies_nodep_ms": timeit(lambda: run(False, dep=False)),
       "copies_onecopy_ms": timeit(lambda: run(False, split_h2d=False)),
       "two_from_a_ms": timeit(lambda: run(False, src2=(ha, ha))),
       "two_from_b_ms": timeit(lambda: run(False, src2=(hb, hb))),
       "two_from_ab_ms": timeit(lambda: run(False, src2=(ha, hb))),
       "with_merge_ms": timeit(lambda: run(True))}
tr = []
run(True, tr); torch.cuda.synchronize()
t0 = tr[0][0]
res["trace_ms"] = [[round(t0.elapsed_time(e), 2) for e in row] for row in tr[:6] + tr[-3:]]
print(json.dumps(res))
