"""Measure host<->device copy bandwidth on this box (pinned host memory):
H2D alone, D2H alone, and both directions concurrently (duplex)."""
import time, torch, json
dev = torch.device("cuda", 0)
n = 1 << 30  # bytes
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device=dev)
d_out = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best
h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
def duplex():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
dup = t(duplex)
print(json.dumps({"h2d_GBps": n/h2d/1e9, "d2h_GBps": n/d2h/1e9, "duplex_each_GBps": n/dup/1e9, "duplex_total_GBps": 2*n/dup/1e9}))

# the same copies split over two streams per direction (two DMA engines?)
s3, s4 = torch.cuda.Stream(), torch.cuda.Stream()
hh = n // 2
def h2d2():
    with torch.cuda.stream(s1): d_in[:hh].copy_(h_in[:hh], non_blocking=True)
    with torch.cuda.stream(s3): d_in[hh:].copy_(h_in[hh:], non_blocking=True)
def d2h2():
    with torch.cuda.stream(s2): h_out[:hh].copy_(d_out[:hh], non_blocking=True)
    with torch.cuda.stream(s4): h_out[hh:].copy_(d_out[hh:], non_blocking=True)
def dup2():
    h2d2(); d2h2()
a, b, c = t(h2d2), t(d2h2), t(dup2)
print(json.dumps({"two_streams_h2d_GBps": n/a/1e9, "two_streams_d2h_GBps": n/b/1e9,
                  "two_streams_duplex_each_GBps": n/c/1e9}))
