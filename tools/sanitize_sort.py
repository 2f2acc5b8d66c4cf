"""Small sorts and merges for compute-sanitizer (memcheck / racecheck): the
fused passes forced at every size (MP_SORT_QUAD=1), ragged sizes, every bare
key type, one merge with values."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1406_2628_b200 import mergepath as mp
dev = torch.device("cuda", 0)
rng = np.random.default_rng(5)
for n in (70_001, 262_144 + 33, 1_000_003):
    for dt in (np.uint32, np.int32, np.float32):
        x = rng.integers(0, 1 << 31, n).astype(dt)
        t = torch.from_numpy(x.view(np.int32) if dt != np.int32 else x).to(dev)
        kt = {np.uint32: "u32", np.int32: "i32", np.float32: "f32"}[dt]
        got = mp.parallel_merge_sort(t if dt == np.int32 else t.view({np.uint32: torch.uint32, np.float32: torch.float32}[dt]), 4)
        ref = np.sort(x)
        assert np.array_equal(got.cpu().numpy().view(dt), ref), (n, kt)
a = np.sort(rng.integers(0, 1000, 300_001).astype(np.int32)); b = np.sort(rng.integers(0, 1000, 200_003).astype(np.int32))
out = mp.parallel_merge(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), 8)
assert np.array_equal(out.cpu().numpy(), np.sort(np.concatenate([a, b]), kind="stable"))
torch.cuda.synchronize()
print("sanitize workload ok")
