"""numpy bindings of the two CPU checkers (test infrastructure only).

port(): oracle/liboracle.so -- the plain-C restatement in mp_oracle.c.
ref():  oracle/_ref/libmergepath_ref.so -- the unmodified reference library
        (built from /root/reference by oracle/Makefile; shipped prebuilt to
        the GPU box, where /root/reference does not exist).

Key suffixes: u32 i32 f32 u64 i64 el (+ kv for the reference's
{u64 key, u32 value} record used by config 3).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libmergepath_ref.so"

ELEMENT_DTYPE = np.dtype([("key", "<i8"), ("tag", "<u4"), ("pad", "<u4")])
KV_DTYPE = np.dtype([("key", "<u8"), ("val", "<u4"), ("pad", "<u4")])
DTYPES = {"u32": np.dtype(np.uint32), "i32": np.dtype(np.int32),
          "f32": np.dtype(np.uint32),  # raw float bits
          "u64": np.dtype(np.uint64), "i64": np.dtype(np.int64),
          "el": ELEMENT_DTYPE, "kv": KV_DTYPE}
SUFFIXES = ("u32", "i32", "f32", "u64", "i64", "el")

_u64p = C.POINTER(C.c_uint64)


def build() -> None:
    """Build liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-f", str(HERE / "Makefile")], check=True,
                   cwd=HERE.parent, stdout=subprocess.DEVNULL)


def _ptr(x):
    if x is None or x.size == 0:
        return C.c_void_p(None)
    return C.c_void_p(x.ctypes.data)


def _as(S, x):
    x = np.ascontiguousarray(x)
    if S == "f32" and x.dtype == np.float32:
        x = x.view(np.uint32)
    want = DTYPES[S]
    if x.dtype != want:
        raise TypeError(f"{S} expects {want}, got {x.dtype}")
    return x


class _Lib:
    def __init__(self, path: Path, prefix: str):
        if not path.exists():
            build()
        self.lib = C.CDLL(str(path))
        self.prefix = prefix

    def fn(self, name, S):
        return getattr(self.lib, f"{self.prefix}_{name}_{S}")


class Port(_Lib):
    """The C restatement (mp_oracle.c)."""

    def __init__(self):
        super().__init__(PORT_LIB, "orc")
        L = self.lib
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
        L.orc_radix_sort.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64]
        for S in SUFFIXES:
            f = getattr(L, f"orc_diagonal_search_{S}")
            f.restype = C.c_uint64
            f.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64, _u64p]
            getattr(L, f"orc_checksum_{S}").restype = C.c_uint64
            getattr(L, f"orc_checksum_{S}").argtypes = [C.c_void_p, C.c_uint64]

    def mix64(self, x: int) -> int:
        return self.lib.orc_mix64(x)

    def diagonal_search(self, S, a, b, d):
        a, b = _as(S, a), _as(S, b)
        c = C.c_uint64(0)
        r = self.fn("diagonal_search", S)(_ptr(a), len(a), _ptr(b), len(b), d, C.byref(c))
        return int(r), c.value

    def partition(self, S, a, b, p):
        a, b = _as(S, a), _as(S, b)
        offs = np.zeros(p + 1, dtype=np.uint64)
        c = C.c_uint64(0)
        rc = self.fn("partition", S)(_ptr(a), C.c_uint64(len(a)), _ptr(b), C.c_uint64(len(b)),
                                     C.c_uint64(p), _ptr(offs), C.byref(c))
        if rc:
            raise ValueError("partition: p must be positive")
        return offs, c.value

    def merge(self, S, a, b, p=1, av=None, bv=None):
        a, b = _as(S, a), _as(S, b)
        n = len(a) + len(b)
        out = np.empty(n, dtype=DTYPES[S])
        outv = np.empty(n, dtype=np.uint32) if av is not None else None
        cmp_, steps = C.c_uint64(0), C.c_uint64(0)
        rc = self.fn("parallel_merge", S)(
            _ptr(a), _ptr(av), C.c_uint64(len(a)), _ptr(b), _ptr(bv), C.c_uint64(len(b)),
            _ptr(out), _ptr(outv), C.c_uint64(p), C.byref(cmp_), C.byref(steps))
        if rc:
            raise ValueError("merge: worker count must be positive")
        return out, outv, cmp_.value, steps.value

    def segmented_merge(self, S, a, b, p, cache, av=None, bv=None):
        a, b = _as(S, a), _as(S, b)
        n = len(a) + len(b)
        L = max(cache // 3, 1)
        iters = (n + L - 1) // L
        out = np.empty(n, dtype=DTYPES[S])
        outv = np.empty(n, dtype=np.uint32) if av is not None else None
        wa = np.zeros(max(iters, 1), dtype=np.uint64)
        wb = np.zeros(max(iters, 1), dtype=np.uint64)
        cmp_, steps, it = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        rc = self.fn("segmented_merge", S)(
            _ptr(a), _ptr(av), C.c_uint64(len(a)), _ptr(b), _ptr(bv), C.c_uint64(len(b)),
            _ptr(out), _ptr(outv), C.c_uint64(p), C.c_uint64(cache), C.byref(cmp_),
            C.byref(steps), _ptr(wa), _ptr(wb), C.byref(it))
        if rc:
            raise ValueError("segmented merge: invalid argument")
        return out, outv, list(zip(wa[:iters].tolist(), wb[:iters].tolist())), cmp_.value, steps.value

    def plan_segments(self, S, a, b, p, cache):
        a, b = _as(S, a), _as(S, b)
        n = len(a) + len(b)
        L = max(cache // 3, 1)
        iters = (n + L - 1) // L
        sa = np.zeros(max(iters, 1), dtype=np.uint64)
        sb = np.zeros(max(iters, 1), dtype=np.uint64)
        wl, pe, it, c = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64(0)
        rc = self.fn("plan_segments", S)(
            _ptr(a), C.c_uint64(len(a)), _ptr(b), C.c_uint64(len(b)), C.c_uint64(p),
            C.c_uint64(cache), _ptr(sa), _ptr(sb), C.byref(wl), C.byref(pe), C.byref(it),
            C.byref(c))
        if rc:
            raise ValueError("plan_segments: invalid argument")
        return dict(window_len=wl.value, p_eff=pe.value, iterations=it.value,
                    starts=list(zip(sa[:iters].tolist(), sb[:iters].tolist())),
                    comparisons=c.value)

    def merge_sort(self, S, data, p=1, vals=None):
        data = _as(S, data)
        out = np.empty_like(data)
        outv = np.empty(len(data), dtype=np.uint32) if vals is not None else None
        r = C.c_uint64(0)
        rc = self.fn("merge_sort", S)(_ptr(data), _ptr(vals), C.c_uint64(len(data)),
                                      C.c_uint64(p), _ptr(out), _ptr(outv), C.byref(r))
        if rc:
            raise ValueError("sort: invalid argument")
        return out, outv, r.value

    def ce_sort(self, S, data, p, cache, vals=None):
        data = _as(S, data)
        out = np.empty_like(data)
        outv = np.empty(len(data), dtype=np.uint32) if vals is not None else None
        r = C.c_uint64(0)
        rc = self.fn("ce_sort", S)(_ptr(data), _ptr(vals), C.c_uint64(len(data)),
                                   C.c_uint64(p), C.c_uint64(cache), _ptr(out), _ptr(outv),
                                   C.byref(r))
        if rc:
            raise ValueError("sort: invalid argument")
        return out, outv, r.value

    def checksum(self, S, out):
        out = _as(S, out)
        return int(self.fn("checksum", S)(_ptr(out), len(out)))

    def generate(self, kind: int, seed: int, first: int, n: int):
        dt = {0: np.uint32, 1: np.int32, 2: np.uint64, 3: np.uint64, 4: np.uint64,
              5: np.float32, 6: np.float32}[kind]
        out = np.empty(n, dtype=dt)
        if self.lib.orc_generate(kind, seed, first, n, _ptr(out)):
            raise ValueError(kind)
        return out

    def radix_sort(self, keys, vals=None):
        """Ascending (stable) sort of generated inputs; keys in place."""
        kt = {np.dtype(np.uint32): 0, np.dtype(np.int32): 1, np.dtype(np.float32): 2,
              np.dtype(np.uint64): 3, np.dtype(np.int64): 4}[keys.dtype]
        if self.lib.orc_radix_sort(kt, _ptr(keys), _ptr(vals), len(keys)):
            raise ValueError(kt)
        return keys


class Ref(_Lib):
    """The unmodified reference library (oracle/_ref)."""

    def __init__(self):
        if not REF_LIB.exists() and not Path("/root/reference/proj").exists():
            raise FileNotFoundError(f"{REF_LIB} not built and reference absent")
        super().__init__(REF_LIB, "ref")
        L = self.lib
        L.ref_team_new.restype = C.c_void_p
        L.ref_team_new.argtypes = [C.c_uint64]
        L.ref_team_free.argtypes = [C.c_void_p]
        L.ref_team_lanes.restype = C.c_uint64
        L.ref_team_lanes.argtypes = [C.c_void_p]
        for S in SUFFIXES + ("kv",):
            f = getattr(L, f"ref_diagonal_search_{S}")
            f.restype = C.c_uint64
            f.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64, _u64p]
            getattr(L, f"ref_parallel_merge_{S}").argtypes = [
                C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                _u64p, _u64p]
        for nm in ("ref_merge_checksum_i64", "ref_merge_checksum_el"):
            getattr(L, nm).restype = C.c_uint64
            getattr(L, nm).argtypes = [C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.ref_segmented_checksum_el.restype = C.c_uint64
        L.ref_segmented_checksum_el.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64,
                                                C.c_void_p, C.c_uint64]
        L.ref_checksum_of_el.restype = C.c_uint64
        L.ref_checksum_of_el.argtypes = [C.c_void_p, C.c_uint64]

    # a persistent thread_team for timing (parallel.hpp:151-162 overload)
    def team(self, p: int):
        return _Team(self.lib, p)

    def diagonal_search(self, S, a, b, d):
        a, b = _as(S, a), _as(S, b)
        c = C.c_uint64(0)
        r = self.fn("diagonal_search", S)(_ptr(a), len(a), _ptr(b), len(b), d, C.byref(c))
        return int(r), c.value

    def partition(self, S, a, b, p):
        a, b = _as(S, a), _as(S, b)
        oa = np.zeros(p + 1, dtype=np.uint64)
        ob = np.zeros(p + 1, dtype=np.uint64)
        c = C.c_uint64(0)
        rc = self.fn("partition", S)(_ptr(a), C.c_uint64(len(a)), _ptr(b), C.c_uint64(len(b)),
                                     C.c_uint64(p), _ptr(oa), _ptr(ob), C.byref(c))
        if rc:
            raise ValueError("partition: p must be positive")
        return oa, ob, c.value

    def merge(self, S, a, b, p=1, team=None, out=None):
        a, b = _as(S, a), _as(S, b)
        if out is None:
            out = np.empty(len(a) + len(b), dtype=DTYPES[S])
        c, s = C.c_uint64(0), C.c_uint64(0)
        if team is not None:
            self.fn("parallel_merge", S)(team.h, _ptr(a), len(a), _ptr(b), len(b), _ptr(out),
                                         C.byref(c), C.byref(s))
        else:
            rc = self.fn("parallel_merge_p", S)(C.c_uint64(p), _ptr(a), C.c_uint64(len(a)),
                                                _ptr(b), C.c_uint64(len(b)), _ptr(out),
                                                C.byref(c), C.byref(s))
            if rc:
                raise ValueError("merge: worker count must be positive")
        return out, c.value, s.value

    def segmented_merge(self, S, a, b, p, cache):
        a, b = _as(S, a), _as(S, b)
        n = len(a) + len(b)
        L = max(cache // 3, 1)
        iters = (n + L - 1) // L
        out = np.empty(n, dtype=DTYPES[S])
        wa = np.zeros(max(iters, 1), dtype=np.uint64)
        wb = np.zeros(max(iters, 1), dtype=np.uint64)
        c, s, nw = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        rc = self.fn("segmented_merge", S)(
            C.c_uint64(p), C.c_uint64(cache), _ptr(a), C.c_uint64(len(a)), _ptr(b),
            C.c_uint64(len(b)), _ptr(out), C.byref(c), C.byref(s), _ptr(wa), _ptr(wb),
            C.byref(nw))
        if rc:
            raise ValueError("segmented merge: invalid argument")
        k = nw.value
        return out, list(zip(wa[:k].tolist(), wb[:k].tolist())), c.value, s.value

    def plan_segments(self, S, a, b, p, cache):
        a, b = _as(S, a), _as(S, b)
        n = len(a) + len(b)
        L = max(cache // 3, 1)
        iters = (n + L - 1) // L
        sa = np.zeros(max(iters, 1), dtype=np.uint64)
        sb = np.zeros(max(iters, 1), dtype=np.uint64)
        wl, pe, it, c = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64(0)
        rc = self.fn("plan_segments", S)(
            _ptr(a), C.c_uint64(len(a)), _ptr(b), C.c_uint64(len(b)), C.c_uint64(p),
            C.c_uint64(cache), _ptr(sa), _ptr(sb), C.byref(wl), C.byref(pe), C.byref(it),
            C.byref(c))
        if rc:
            raise ValueError("plan_segments: invalid argument")
        return dict(window_len=wl.value, p_eff=pe.value, iterations=it.value,
                    starts=list(zip(sa[:iters].tolist(), sb[:iters].tolist())),
                    comparisons=c.value)

    def merge_sort(self, S, data, p=1):
        data = _as(S, data)
        out = np.empty_like(data)
        r = C.c_uint64(0)
        rc = self.fn("merge_sort", S)(_ptr(data), C.c_uint64(len(data)), C.c_uint64(p),
                                      _ptr(out), C.byref(r))
        if rc:
            raise ValueError("sort: invalid argument")
        return out, r.value

    def ce_sort(self, S, data, p, cache):
        data = _as(S, data)
        out = np.empty_like(data)
        r = C.c_uint64(0)
        rc = self.fn("ce_sort", S)(_ptr(data), C.c_uint64(len(data)), C.c_uint64(p),
                                   C.c_uint64(cache), _ptr(out), C.byref(r))
        if rc:
            raise ValueError("sort: invalid argument")
        return out, r.value

    def merge_checksum_el(self, a, b, p):
        a, b = _as("el", a), _as("el", b)
        return int(self.lib.ref_merge_checksum_el(p, _ptr(a), len(a), _ptr(b), len(b)))

    def segmented_checksum_el(self, a, b, p, cache):
        a, b = _as("el", a), _as("el", b)
        return int(self.lib.ref_segmented_checksum_el(p, cache, _ptr(a), len(a), _ptr(b),
                                                      len(b)))

    def checksum_of_el(self, out):
        out = _as("el", out)
        return int(self.lib.ref_checksum_of_el(_ptr(out), len(out)))


class _Team:
    def __init__(self, lib, p):
        self.lib = lib
        self.h = lib.ref_team_new(p)

    def close(self):
        if self.h:
            self.lib.ref_team_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def ref_available() -> bool:
    return REF_LIB.exists() or Path("/root/reference/proj").exists()


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def sequential_merge(S, a, b, start, length):
    """core.hpp:148-180 through the port: returns (out, end) or raises
    ValueError on overrun (core.hpp:161-162)."""
    P = port()
    a, b = _as(S, a), _as(S, b)
    out = np.empty(max(length, 0), dtype=DTYPES[S])
    ea, eb, st = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    rc = P.fn("sequential_merge", S)(
        _ptr(a), C.c_void_p(None), C.c_uint64(len(a)), _ptr(b), C.c_void_p(None),
        C.c_uint64(len(b)), C.c_uint64(start[0]), C.c_uint64(start[1]), C.c_uint64(length),
        _ptr(out), C.c_void_p(None), C.byref(ea), C.byref(eb), C.byref(st))
    if rc:
        raise ValueError("sequential_merge: length overruns the path")
    return out, (ea.value, eb.value)
