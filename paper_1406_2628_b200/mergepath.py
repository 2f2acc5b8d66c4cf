"""Python mirror of the reference's mergepath API, running on the B200.

Same operation names, argument meaning and error behaviour as the reference
C++ templates (cited per function); every call goes through the C ABI of
libmergepath_b200.so.  Inputs may be

  * CUDA torch tensors  -> the device entry points, asynchronous on the
                           current torch stream, results stay in HBM;
  * host numpy arrays   -> the *_host entry points (staged through the GPU).

Key type comes from the dtype (uint32, int32, float32 [IEEE totalOrder],
uint64, int64) or, for the reference's 16-byte `element`, from
ELEMENT_DTYPE / key_type=KEY_ELEMENT.  Worker count `p` and cache size `C`
are validated exactly like the reference (p == 0 and C < 3 raise
ValueError, the analogue of std::invalid_argument) but never change the
merged bytes, which are identical for every p and C.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native as N

try:  # torch is plumbing only (device memory + streams)
    import torch
except ImportError:  # pragma: no cover
    torch = None

ELEMENT_DTYPE = np.dtype([("key", "<i8"), ("tag", "<u4"), ("pad", "<u4")])

_NP_KEYS = {np.dtype(np.uint32): N.KEY_U32, np.dtype(np.int32): N.KEY_I32,
            np.dtype(np.float32): N.KEY_F32, np.dtype(np.uint64): N.KEY_U64,
            np.dtype(np.int64): N.KEY_I64, ELEMENT_DTYPE: N.KEY_ELEMENT}


def _torch_keys():
    if torch is None:
        return {}
    return {torch.uint32: N.KEY_U32, torch.int32: N.KEY_I32,
            torch.float32: N.KEY_F32, torch.uint64: N.KEY_U64,
            torch.int64: N.KEY_I64}


# --------------------------------------------------------------------------
# reference data types (core.hpp:63-75, parallel.hpp:29-46, sort.hpp:29-42)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class PartitionPoint:
    a_off: int = 0
    b_off: int = 0

    @property
    def d(self) -> int:
        return self.a_off + self.b_off


@dataclass
class WindowStats:
    a_consumed: int = 0
    b_consumed: int = 0


@dataclass
class MergeStats:
    partition_comparisons: int = 0
    merge_steps: int = 0
    windows: list = field(default_factory=list)


@dataclass
class SegmentPlan:
    cache_elems: int = 0
    window_len: int = 0
    p_eff: int = 0
    iterations: int = 0
    starting_points: list = field(default_factory=list)


class SortVariant(Enum):
    plain = 0
    cache_efficient = 1


@dataclass
class SortPlan:
    variant: SortVariant = SortVariant.plain
    block_size: int = 0
    blocks: int = 0
    tree_levels: int = 0


@dataclass
class SortStats:
    merge_rounds: int = 0


SORT_BASE_RUN = 32  # sort.hpp:29 (the reference CPU plan)


# --------------------------------------------------------------------------
# argument plumbing
# --------------------------------------------------------------------------
class _Arr:
    """A key (or value) array: pointer, length, key type, residency."""

    def __init__(self, x, key_type=None, values=False):
        self.obj = x
        if torch is not None and isinstance(x, torch.Tensor):
            if not x.is_cuda:
                x = x.numpy()
                self.obj = x
            else:
                if not x.is_contiguous():
                    raise ValueError("tensor must be contiguous")
                self.device = True
                self.ptr = x.data_ptr()
                if values:
                    if x.dtype not in (torch.int32, torch.uint32):
                        raise ValueError("values must be uint32")
                    self.kt, self.n = None, x.numel()
                    return
                self.kt = key_type if key_type is not None else _torch_keys().get(x.dtype)
                if self.kt is None:
                    raise TypeError(f"unsupported key dtype {x.dtype}")
                self.n = x.numel() * x.element_size() // N.KEY_SIZES[self.kt]
                return
        x = np.ascontiguousarray(x)
        self.obj = x
        self.device = False
        self.ptr = x.ctypes.data if x.size else None
        if values:
            if x.dtype not in (np.uint32, np.int32):
                raise ValueError("values must be uint32")
            self.kt, self.n = None, x.size
            return
        self.kt = key_type if key_type is not None else _NP_KEYS.get(x.dtype)
        if self.kt is None:
            raise TypeError(f"unsupported key dtype {x.dtype}")
        self.n = x.nbytes // N.KEY_SIZES[self.kt]


def _stream_ptr(dev_arr: _Arr) -> int:
    return torch.cuda.current_stream(dev_arr.obj.device).cuda_stream


def _pair(a, b, key_type):
    A = _Arr(a, key_type)
    B = _Arr(b, key_type)
    if A.kt != B.kt:
        raise TypeError("A and B must have the same key type")
    if A.device != B.device:
        raise ValueError("A and B must both be CUDA tensors or both host arrays")
    return A, B


def _check_p(p: int) -> None:
    if p == 0:  # parallel.hpp:54-57, core.hpp:139-140
        raise ValueError("merge: worker count must be positive")


# --------------------------------------------------------------------------
# comparators: the reference templates take any Comp; the device kernels
# implement exactly one order per key type (b200_backend.hpp key_traits).
# The Python mirror accepts the same allow-list by name and rejects every
# other comparator, as the C++ drop-in does at compile time.
# --------------------------------------------------------------------------
LESS = "less"                          # std::less<T> on u32/i32/u64/i64
TOTAL_ORDER_LESS = "total_order_less"  # IEEE totalOrder on f32
KEY_LESS = "key_less"                  # mergepath::key_less on element (core.hpp:52)

_COMP_FOR = {N.KEY_U32: LESS, N.KEY_I32: LESS, N.KEY_U64: LESS, N.KEY_I64: LESS,
             N.KEY_F32: TOTAL_ORDER_LESS, N.KEY_ELEMENT: KEY_LESS}


def _check_comp(comp, kt) -> None:
    """None selects the key type's own order.  Otherwise comp must name that
    order (LESS / TOTAL_ORDER_LESS / KEY_LESS, or operator.lt for the
    integer keys); a custom callable (e.g. descending) has no kernel and
    raises TypeError instead of being ignored."""
    if comp is None:
        return
    import operator
    want = _COMP_FOR[kt]
    if comp == want or (comp is operator.lt and want == LESS):
        return
    raise TypeError(f"comparator {comp!r} is not supported for this key type on the B200 "
                    f"backend (supported: None or {want!r})")


def _window_of(cache_elems: int) -> int:  # parallel.hpp:59-63
    if cache_elems < 3:
        raise ValueError("merge: cache capacity must be at least 3")
    return cache_elems // 3


def _device_index(A: _Arr) -> int:
    return A.obj.device.index if A.device else 0


def _empty_like_keys(A: _Arr, n: int):
    if A.device:
        if A.kt == N.KEY_ELEMENT:
            return torch.empty(n * 2, dtype=torch.int64, device=A.obj.device)
        return torch.empty(n, dtype=A.obj.dtype, device=A.obj.device)
    if A.kt == N.KEY_ELEMENT:
        return np.zeros(n, dtype=ELEMENT_DTYPE)
    return np.empty(n, dtype=A.obj.dtype)


def _empty_vals(A: _Arr, n: int):
    if A.device:
        return torch.empty(n, dtype=torch.uint32, device=A.obj.device)
    return np.empty(n, dtype=np.uint32)


# --------------------------------------------------------------------------
# core.hpp: diagonal_search / partition / diagonal_of
# --------------------------------------------------------------------------
def _host_device() -> int:
    """GPU used for host-array calls: MERGEPATH_DEVICE, else 0 (as the C++
    drop-in, b200_backend.hpp)."""
    return int(os.environ.get("MERGEPATH_DEVICE", "0"))


def diagonal_of(n: int, p: int, i: int) -> int:
    """core.hpp:90-92"""
    return i * n // p


def _search(A: _Arr, B: _Arr, diags: list[int], counter: list | None):
    count = len(diags)
    if count == 0:
        return []
    if not A.device:  # host arrays: the ABI stages them (mp_diagonal_search_host)
        d_h = np.asarray(diags, dtype=np.uint64)
        o_h = np.zeros(count, dtype=np.uint64)
        c_h = C.c_uint64(0)
        N.check(N.lib.mp_diagonal_search_host(A.kt, A.ptr, A.n, B.ptr, B.n, d_h.ctypes.data,
                                              count, o_h.ctypes.data, C.byref(c_h),
                                              _host_device()))
        if counter is not None:
            counter[0] += int(c_h.value)
        return [PartitionPoint(int(o), d - int(o))
                for o, d in zip(o_h, [min(x, A.n + B.n) for x in diags])]
    dev = torch.device("cuda", _device_index(A))
    d_t = torch.tensor(diags, dtype=torch.int64, device=dev)
    o_t = torch.empty(count, dtype=torch.int64, device=dev)
    c_t = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(N.lib.mp_diagonal_search(A.kt, A.ptr, A.n, B.ptr, B.n, d_t.data_ptr(), count,
                                     o_t.data_ptr(), c_t.data_ptr(), stream))
    offs = o_t.cpu().tolist()
    if counter is not None:
        counter[0] += int(c_t.item())
    return [PartitionPoint(o, d - o) for o, d in zip(offs, [min(x, A.n + B.n) for x in diags])]


def diagonal_search(a, b, d: int, comparisons: list | None = None, key_type=None):
    """core.hpp:120-132: the point where the merge path crosses diagonal d.
    `comparisons` (a one-element list) accumulates the comparison count."""
    A, B = _pair(a, b, key_type)
    if d > A.n + B.n:  # core.hpp:104 (contract violation in the reference)
        raise ValueError("diagonal out of range")
    return _search(A, B, [d], comparisons)[0]


def partition(a, b, p: int, comparisons: list | None = None, key_type=None):
    """core.hpp:134-146: p+1 points on the equispaced diagonals i*N/p."""
    if p == 0:
        raise ValueError("partition: p must be positive")
    A, B = _pair(a, b, key_type)
    n = A.n + B.n
    return _search(A, B, [diagonal_of(n, p, i) for i in range(p + 1)], comparisons)


# --------------------------------------------------------------------------
# parallel.hpp: merges
# --------------------------------------------------------------------------
def _merge(A: _Arr, B: _Arr, out, a_vals, b_vals, out_vals):
    O = _Arr(out, A.kt)
    if O.n != A.n + B.n:  # parallel.hpp:155-156 (abort in the reference)
        raise ValueError("output size must equal |A| + |B|")
    if O.device != A.device:
        raise ValueError("output residency must match the inputs")
    vals = a_vals is not None or b_vals is not None or out_vals is not None
    if vals and (a_vals is None or b_vals is None or out_vals is None):
        raise ValueError("values must be given for A, B and out")
    AV = _Arr(a_vals, values=True) if vals else None
    BV = _Arr(b_vals, values=True) if vals else None
    OV = _Arr(out_vals, values=True) if vals else None
    if vals and (AV.n != A.n or BV.n != B.n or OV.n != O.n):
        raise ValueError("value arrays must match their key arrays")
    vp = (lambda x: x.ptr if x is not None else None)
    if A.device:
        N.check(N.lib.mp_merge(A.kt, A.ptr, vp(AV), A.n, B.ptr, vp(BV), B.n, O.ptr, vp(OV),
                               _stream_ptr(A)))
    else:
        N.check(N.lib.mp_merge_host(A.kt, A.ptr, vp(AV), A.n, B.ptr, vp(BV), B.n, O.ptr,
                                    vp(OV), _host_device()))


def _merge_stats(A, B, p, stats):
    if stats is None:
        return
    stats.merge_steps += A.n + B.n
    # the reference counts the searches of workers with a non-empty segment
    n = A.n + B.n
    diags = [diagonal_of(n, p, w) for w in range(p) if diagonal_of(n, p, w) != diagonal_of(n, p, w + 1)]
    cnt = [0]
    _search(A, B, diags, cnt)
    stats.partition_comparisons += cnt[0]


def parallel_merge_into(a, b, out, p: int = 1, comp=None, stats: MergeStats | None = None,
                        a_vals=None, b_vals=None, out_vals=None, key_type=None):
    """parallel.hpp:151-171: stable merge of A and B into `out`."""
    _check_p(p)
    A, B = _pair(a, b, key_type)
    _check_comp(comp, A.kt)
    _merge(A, B, out, a_vals, b_vals, out_vals)
    _merge_stats(A, B, p, stats)


def parallel_merge(a, b, p: int = 1, comp=None, stats: MergeStats | None = None,
                   a_vals=None, b_vals=None, key_type=None):
    """parallel.hpp:173-179.  Returns the merged keys, or (keys, values)
    when values are given."""
    _check_p(p)
    A, B = _pair(a, b, key_type)
    _check_comp(comp, A.kt)
    out = _empty_like_keys(A, A.n + B.n)
    out_vals = _empty_vals(A, A.n + B.n) if a_vals is not None else None
    _merge(A, B, out, a_vals, b_vals, out_vals)
    _merge_stats(A, B, p, stats)
    return (out, out_vals) if out_vals is not None else out


def _segment_plan(A: _Arr, B: _Arr, p: int, cache_elems: int):
    """Window starts + the reference's two comparison counters, computed on
    the device by mp_segment_plan (window k starts on diagonal k*L,
    test_parallel.cpp:120-137)."""
    iters = int(N.lib.mp_segment_iterations(A.n, B.n, cache_elems))
    L = cache_elems // 3
    if iters == 0:
        return [], 0, 0
    if A.device:
        st = torch.empty(iters, dtype=torch.int64, device=A.obj.device)
        cnt = torch.zeros(2, dtype=torch.int64, device=A.obj.device)
        N.check(N.lib.mp_segment_plan(A.kt, A.ptr, A.n, B.ptr, B.n, p, cache_elems,
                                      st.data_ptr(), cnt.data_ptr(), cnt.data_ptr() + 8,
                                      _stream_ptr(A)))
        sa = st.cpu().tolist()
        plan_cmp, merge_cmp = cnt.cpu().tolist()
    else:
        st = np.zeros(iters, dtype=np.uint64)
        pc, mc = C.c_uint64(0), C.c_uint64(0)
        N.check(N.lib.mp_segment_plan_host(A.kt, A.ptr, A.n, B.ptr, B.n, p, cache_elems,
                                           st.ctypes.data, None, C.byref(pc), C.byref(mc), _host_device()))
        sa = st.tolist()
        plan_cmp, merge_cmp = pc.value, mc.value
    starts = [PartitionPoint(int(x), k * L - int(x)) for k, x in enumerate(sa)]
    return starts, plan_cmp, merge_cmp


def plan_segments(a, b, p: int, cache_elems: int, comparisons: list | None = None,
                  key_type=None) -> SegmentPlan:
    """parallel.hpp:258-292: window geometry and every window's starting
    point; `comparisons` accumulates the reference's search count."""
    _check_p(p)
    L = _window_of(cache_elems)
    A, B = _pair(a, b, key_type)
    starts, plan_cmp, _ = _segment_plan(A, B, p, cache_elems)
    if comparisons is not None:
        comparisons[0] += plan_cmp
    return SegmentPlan(cache_elems, L, min(p, L), len(starts), starts)


def _segmented_stats(A, B, p, cache_elems, stats):
    if stats is None:
        return
    starts, _, merge_cmp = _segment_plan(A, B, p, cache_elems)
    stats.merge_steps += A.n + B.n
    stats.partition_comparisons += merge_cmp
    ends = starts[1:] + [PartitionPoint(A.n, B.n)]
    for s, e in zip(starts, ends):
        stats.windows.append(WindowStats(e.a_off - s.a_off, e.b_off - s.b_off))


def segmented_parallel_merge_into(a, b, out, p: int, cache_elems: int, comp=None,
                                  stats: MergeStats | None = None, a_vals=None,
                                  b_vals=None, out_vals=None, key_type=None):
    """parallel.hpp:200-225.  One CTA tile *is* an SPM window staged in
    shared memory; the merged bytes equal the regular merge's."""
    _check_p(p)
    _window_of(cache_elems)
    A, B = _pair(a, b, key_type)
    _check_comp(comp, A.kt)
    _merge(A, B, out, a_vals, b_vals, out_vals)
    _segmented_stats(A, B, p, cache_elems, stats)


def segmented_parallel_merge(a, b, p: int, cache_elems: int, comp=None,
                             stats: MergeStats | None = None, a_vals=None, b_vals=None,
                             key_type=None):
    """parallel.hpp:227-236."""
    _check_p(p)
    _window_of(cache_elems)
    A, B = _pair(a, b, key_type)
    _check_comp(comp, A.kt)
    out = _empty_like_keys(A, A.n + B.n)
    out_vals = _empty_vals(A, A.n + B.n) if a_vals is not None else None
    _merge(A, B, out, a_vals, b_vals, out_vals)
    _segmented_stats(A, B, p, cache_elems, stats)
    return (out, out_vals) if out_vals is not None else out


def _checksum(A: _Arr, B: _Arr) -> int:
    if A.device:
        s = torch.zeros(1, dtype=torch.int64, device=A.obj.device)
        N.check(N.lib.mp_merge_checksum(A.kt, A.ptr, A.n, B.ptr, B.n, s.data_ptr(),
                                        _stream_ptr(A)))
        return int(s.item()) & 0xFFFFFFFFFFFFFFFF
    s = C.c_uint64(0)
    N.check(N.lib.mp_merge_checksum_host(A.kt, A.ptr, A.n, B.ptr, B.n, C.byref(s), _host_device()))
    return s.value


def parallel_merge_checksum(a, b, p: int = 1, comp=None, stats=None, key_type=None) -> int:
    """parallel.hpp:181-198: register-sink merge (no output array)."""
    _check_p(p)
    A, B = _pair(a, b, key_type)
    _check_comp(comp, A.kt)
    s = _checksum(A, B)
    _merge_stats(A, B, p, stats)
    return s


def segmented_parallel_merge_checksum(a, b, p: int, cache_elems: int, comp=None,
                                      stats=None, key_type=None) -> int:
    """parallel.hpp:238-256."""
    _check_p(p)
    _window_of(cache_elems)
    A, B = _pair(a, b, key_type)
    _check_comp(comp, A.kt)
    s = _checksum(A, B)
    _segmented_stats(A, B, p, cache_elems, stats)
    return s


# --------------------------------------------------------------------------
# sort.hpp
# --------------------------------------------------------------------------
def make_sort_plan(variant: SortVariant, n: int, cache_elems: int) -> SortPlan:
    """sort.hpp:44-55: the reference's CPU plan (block 32 or C/3).  The GPU
    schedule (block-sorted runs + Merge Path rounds) is gpu_sort_plan()."""
    block = SORT_BASE_RUN if variant == SortVariant.plain else _window_of(cache_elems)
    blocks = 0 if n == 0 else (n + block - 1) // block
    levels = 0 if blocks <= 1 else (blocks - 1).bit_length()
    return SortPlan(variant, block, blocks, levels)


GPU_SORT_RUN = 2048       # stable K3 block sort (values, 64-bit keys, element)
GPU_SORT_RUN_BARE = 16384  # K3w block sort (bare u32 / i32 / f32 keys)


def gpu_sort_plan(n: int, bare32: bool = False) -> SortPlan:
    """The B200 schedule: block-sorted runs (16384 keys for bare 32-bit keys,
    2048 otherwise), then ceil(log2(n/run)) Merge Path rounds (large bare
    32-bit sorts run them as fused pairs: one HBM pass per two rounds)."""
    run = GPU_SORT_RUN_BARE if bare32 else GPU_SORT_RUN
    blocks = 0 if n == 0 else (n + run - 1) // run
    levels = 0 if blocks <= 1 else (blocks - 1).bit_length()
    return SortPlan(SortVariant.plain, run, blocks, levels)


def _sort(data, vals, key_type):
    D = _Arr(data, key_type)
    out = _empty_like_keys(D, D.n)
    out_vals = _empty_vals(D, D.n) if vals is not None else None
    V = _Arr(vals, values=True) if vals is not None else None
    if V is not None and V.n != D.n:
        raise ValueError("values must match keys")
    if D.device:
        O = _Arr(out, D.kt)
        N.check(N.lib.mp_sort_to(D.kt, D.ptr, V.ptr if V is not None else None, O.ptr,
                                 out_vals.data_ptr() if V is not None else None,
                                 D.n, None, 0, _stream_ptr(D)))
    else:
        O = _Arr(out, D.kt)
        N.check(N.lib.mp_sort_host(D.kt, D.ptr, V.ptr if V is not None else None, D.n,
                                   O.ptr, _Arr(out_vals, values=True).ptr if V is not None else None,
                                   _host_device()))
    return (out, out_vals) if out_vals is not None else out


def parallel_merge_sort(data, p: int = 1, comp=None, stats: SortStats | None = None,
                        vals=None, key_type=None):
    """sort.hpp:132-148: stable sort (w.r.t. input index).  `merge_rounds`
    reports the reference plan's round count (sort.hpp:142-146) so that
    drop-in callers see unchanged statistics."""
    _check_p(p)
    _check_comp(comp, _Arr(data, key_type).kt)
    res = _sort(data, vals, key_type)
    if stats is not None:
        n = _Arr(data, key_type).n
        stats.merge_rounds += make_sort_plan(SortVariant.plain, n, 0).tree_levels
    return res


def cache_efficient_parallel_sort(data, p: int, cache_elems: int, comp=None,
                                  stats: SortStats | None = None, vals=None, key_type=None):
    """sort.hpp:150-195: same bytes as the plain sort (test_sort.cpp:128-135)."""
    _check_p(p)
    _window_of(cache_elems)
    _check_comp(comp, _Arr(data, key_type).kt)
    res = _sort(data, vals, key_type)
    if stats is not None:
        n = _Arr(data, key_type).n
        stats.merge_rounds += make_sort_plan(SortVariant.cache_efficient, n,
                                             cache_elems).tree_levels
    return res
