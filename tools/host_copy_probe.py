"""Host memory copy bandwidth with T threads (numpy copies release the GIL):
pageable -> pageable, the staging step a pageable host-span call needs, and
pinned H2D/D2H for comparison.  Prints one JSON line per measurement."""
import json
import threading
import time

import numpy as np

N = 1 << 30  # bytes per copy


def par_copy(dst, src, T):
    n = len(src)
    cuts = [k * n // T for k in range(T + 1)]
    th = [threading.Thread(target=lambda a, b: np.copyto(dst[a:b], src[a:b]),
                           args=(cuts[k], cuts[k + 1])) for k in range(T)]
    for t in th:
        t.start()
    for t in th:
        t.join()


src = np.ones(N, dtype=np.uint8)
dst = np.empty(N, dtype=np.uint8)
dst[:] = 0
for T in (1, 2, 4, 8, 12, 16):
    par_copy(dst, src, T)
    t = time.perf_counter()
    for _ in range(3):
        par_copy(dst, src, T)
    dt = (time.perf_counter() - t) / 3
    print(json.dumps({"copy": "pageable->pageable", "threads": T, "GBps": N / dt / 1e9}))
# two concurrent copies (in-staging and out-draining at once), T each
src2 = np.ones(N, dtype=np.uint8)
dst2 = np.empty(N, dtype=np.uint8)
dst2[:] = 0
for T in (4, 8):
    t = time.perf_counter()
    a = threading.Thread(target=par_copy, args=(dst, src, T))
    b = threading.Thread(target=par_copy, args=(dst2, src2, T))
    a.start(); b.start(); a.join(); b.join()
    dt = time.perf_counter() - t
    print(json.dumps({"copy": "2 concurrent pageable->pageable", "threads_each": T,
                      "GBps_each": N / dt / 1e9}))
try:
    import torch
    h = torch.empty(N, dtype=torch.uint8).pin_memory()
    d = torch.empty(N, dtype=torch.uint8, device="cuda")
    for name, f in (("pinned H2D", lambda: d.copy_(h, non_blocking=True)),
                    ("pinned D2H", lambda: h.copy_(d, non_blocking=True))):
        f(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        print(json.dumps({"copy": name, "GBps": 3 * N / (time.perf_counter() - t) / 1e9}))
    # pinned <-> pageable memcpy (the staging hop)
    hp = h.numpy()
    for T in (4, 8, 16):
        t = time.perf_counter()
        par_copy(hp, src, T)
        dt = time.perf_counter() - t
        print(json.dumps({"copy": "pageable->pinned", "threads": T, "GBps": N / dt / 1e9}))
except Exception as e:  # pragma: no cover
    print(json.dumps({"error": str(e)}))
