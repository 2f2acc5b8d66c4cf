"""ctypes binding of the C ABI in include/mergepath_b200.h.

The library is loaded from the package directory (built in-tree by
paper_1406_2628_b200/build.py).  There is no fallback: if the shared library
is missing the import fails loudly, and every compute entry point fails with
a CUDA error when no GPU is present.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os as _os

# MP_NATIVE_LIB: load a differently-compiled build of the same library
# (tuning A/B runs, tools/variant_bench.sh); the product default is in-tree.
LIB_PATH = Path(_os.environ.get("MP_NATIVE_LIB") or
                Path(__file__).resolve().parent / "libmergepath_b200.so")

MP_OK, MP_ERR_INVALID, MP_ERR_CUDA, MP_ERR_OOM, MP_ERR_UNSUPPORTED, MP_ERR_IO = range(6)

KEY_U32, KEY_I32, KEY_F32, KEY_U64, KEY_I64, KEY_ELEMENT = range(6)
KEY_NAMES = {KEY_U32: "u32", KEY_I32: "i32", KEY_F32: "f32", KEY_U64: "u64",
             KEY_I64: "i64", KEY_ELEMENT: "element"}
KEY_SIZES = {KEY_U32: 4, KEY_I32: 4, KEY_F32: 4, KEY_U64: 8, KEY_I64: 8,
             KEY_ELEMENT: 16}

# (name, restype, argtypes) for every symbol include/mergepath_b200.h declares.
_u64, _i, _p = C.c_uint64, C.c_int, C.c_void_p
SIGNATURES = [
    ("mp_last_error", C.c_char_p, []),
    ("mp_abi_version", _i, []),
    ("mp_launch_count", _u64, []),
    ("mp_keyfile_count", _i, [C.c_char_p, _p, _p]),
    ("mp_keyfile_read", _i, [C.c_char_p, _p, _u64, _p]),
    ("mp_keyfile_write", _i, [C.c_char_p, _p, _u64, _i]),
    ("mp_keyfile_load", _i, [C.c_char_p, _p, _u64, _p, _i, _p]),
    ("mp_keyfile_store", _i, [C.c_char_p, _p, _u64, _i, _p]),
    ("mp_keyfile_merge", _i, [C.c_char_p, C.c_char_p, C.c_char_p, _p, _i]),
    ("mp_keyfile_sort", _i, [C.c_char_p, C.c_char_p, _p, _i]),
    ("mp_key_size", _u64, [_i]),
    ("mp_partition", _i, [_i, _p, _u64, _p, _u64, _u64, _p, _p, _p]),
    ("mp_diagonal_search", _i, [_i, _p, _u64, _p, _u64, _p, _u64, _p, _p, _p]),
    ("mp_merge", _i, [_i, _p, _p, _u64, _p, _p, _u64, _p, _p, _p]),
    ("mp_merge_workspace_bytes", _u64, [_i, _u64, _u64]),
    ("mp_merge_plan", _i, [_i, _p, _u64, _p, _u64, _p, _p]),
    ("mp_merge_execute", _i, [_i, _p, _p, _u64, _p, _p, _u64, _p, _p, _p, _p]),
    ("mp_merge_checksum", _i, [_i, _p, _u64, _p, _u64, _p, _p]),
    ("mp_sort_scratch_bytes", _u64, [_i, _i, _u64]),
    ("mp_sort", _i, [_i, _p, _p, _u64, _p, _u64, _p]),
    ("mp_sort_to", _i, [_i, _p, _p, _p, _p, _u64, _p, _u64, _p]),
    ("mp_segment_iterations", _u64, [_u64, _u64, _u64]),
    ("mp_segment_plan", _i, [_i, _p, _u64, _p, _u64, _u64, _u64, _p, _p, _p, _p]),
    ("mp_partition_host", _i, [_i, _p, _u64, _p, _u64, _u64, _p, _p, _i]),
    ("mp_diagonal_search_host", _i, [_i, _p, _u64, _p, _u64, _p, _u64, _p, _p, _i]),
    ("mp_segment_plan_host", _i, [_i, _p, _u64, _p, _u64, _u64, _u64, _p, _p, _p, _p, _i]),
    ("mp_merge_host", _i, [_i, _p, _p, _u64, _p, _p, _u64, _p, _p, _i]),
    ("mp_sort_host", _i, [_i, _p, _p, _u64, _p, _p, _i]),
    ("mp_merge_checksum_host", _i, [_i, _p, _u64, _p, _u64, _p, _i]),
    ("mp_merge_pieces", _i, [_i, _p, _i, _p, _i, _u64, _u64, _p, _p, _p]),
    ("mp_pieces_partition", _i, [_i, _p, _i, _p, _i, _p, _u64, _p, _p]),
    ("mp_multi_merge", _i, [_i, _p, _i, _p, _i, _p, _i, _p]),
    ("mp_multi_sort", _i, [_i, _p, _i, _p]),
    ("mp_peer_copy", _i, [_p, _p, _u64, _p]),
    ("mp_ipc_export", _i, [_p, _p, _p]),
    ("mp_ipc_import", _i, [_p, _u64, _p]),
    ("mp_ipc_close", _i, [_p]),
    ("mp_ipc_open_count", _u64, []),
    ("mp_release", _i, [_i]),
    ("mp_host_alloc", _p, [_u64]),
    ("mp_host_free", _i, [_p]),
    ("mp_signal", _i, [_p, _u64, _p]),
    ("mp_wait", _i, [_p, _u64, _p]),
    ("mp_generate", _i, [_i, _u64, _u64, _u64, _p, _p]),
]


class MergePathError(RuntimeError):
    """A non-OK status from the native library."""

    def __init__(self, status: int, message: str):
        super().__init__(f"mergepath status {status}: {message}")
        self.status = status


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    """Raise for a non-OK status: invalid arguments map to ValueError (the
    reference's std::invalid_argument), everything else to MergePathError."""
    if status == MP_OK:
        return
    msg = lib.mp_last_error().decode(errors="replace")
    if status == MP_ERR_INVALID:
        raise ValueError(msg)
    if status == MP_ERR_IO:
        raise OSError(msg)  # the reference's std::runtime_error (dataio.cpp)
    raise MergePathError(status, msg)


class Piece(C.Structure):
    """mp_piece: one contiguous (possibly peer-mapped) shard."""
    _fields_ = [("keys", C.c_void_p), ("vals", C.c_void_p), ("len", C.c_uint64)]


def pieces_array(pieces):
    """[(keys_ptr, vals_ptr_or_None, len)] -> ctypes mp_piece array."""
    arr = (Piece * max(1, len(pieces)))()
    for k, (kp, vp, n) in enumerate(pieces):
        arr[k].keys, arr[k].vals, arr[k].len = kp, vp, n
    return arr


class Shard(C.Structure):
    """mp_shard: a shard of a sequence on one GPU."""
    _fields_ = [("device", C.c_int), ("keys", C.c_void_p), ("vals", C.c_void_p),
                ("len", C.c_uint64)]


def shards_array(shards):
    """[(device, keys_ptr, vals_ptr_or_None, len)] -> ctypes mp_shard array."""
    arr = (Shard * max(1, len(shards)))()
    for k, (d, kp, vp, n) in enumerate(shards):
        arr[k].device, arr[k].keys, arr[k].vals, arr[k].len = d, kp, vp, n
    return arr
