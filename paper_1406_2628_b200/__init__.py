"""paper_1406_2628_b200 -- B200-native Merge Path merge and merge sort.

Hot path (BASELINE.json north_star): Merge Path partition -> merge and the
bottom-up merge sort built on it, as hand-written sm_100a kernels behind the
C ABI in include/mergepath_b200.h (libmergepath_b200.so, built in-tree).

    from paper_1406_2628_b200 import mergepath as mp
    out = mp.parallel_merge(a, b, p=8)        # a, b: sorted CUDA tensors
    s = mp.parallel_merge_sort(keys, p=8)

The multi-GPU layer (one process per GPU, torch.distributed) lives in
paper_1406_2628_b200.multigpu.
"""
from . import _native  # noqa: F401  (fails loudly if the .so is missing)
from . import mergepath  # noqa: F401

__all__ = ["mergepath"]


def kernel_sources_sha256() -> str:
    """SHA-256 over the kernel sources (csrc/*.cu, *.cuh, except the key-file
    I/O header, which holds no device code): profiles stamped with it
    (profiles/traffic_config*.json) are only used while it matches."""
    import hashlib
    from pathlib import Path
    h = hashlib.sha256()
    for p in sorted((Path(__file__).resolve().parent / "csrc").glob("*.cu*")):
        if p.name == "mp_keyfile.cuh":
            continue
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()
