"""Cost of page-locking pageable host memory per call (cudaHostRegister +
cudaHostUnregister) vs the driver's pageable copies, on this box."""
import ctypes, json, time
import numpy as np
import torch
cudart = ctypes.CDLL("libcudart.so") if False else None
rt = torch.cuda.cudart()
dev = torch.device("cuda", 0)
torch.cuda.init()
res = {}
for mb in (64, 256, 1024):
    n = mb << 20
    h = np.ones(n, dtype=np.uint8)  # pageable, touched
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    ptr = h.ctypes.data
    t = time.perf_counter(); rt.cudaHostRegister(ptr, n, 0); t1 = time.perf_counter()
    ht = torch.from_numpy(h)
    d.copy_(ht, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    rt.cudaHostUnregister(ptr); t3 = time.perf_counter()
    d.copy_(ht); torch.cuda.synchronize(); t4 = time.perf_counter()
    res[f"{mb}MB"] = {"register_ms": round((t1 - t) * 1e3, 2), "h2d_pinned_ms": round((t2 - t1) * 1e3, 2),
                      "unregister_ms": round((t3 - t2) * 1e3, 2), "h2d_pageable_ms": round((t4 - t3) * 1e3, 2)}
print(json.dumps(res))
