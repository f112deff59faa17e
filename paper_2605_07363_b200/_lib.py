"""ctypes binding of the C ABI in ``include/misa_b200.h``.

The library is the only compute path of this package: if it is missing, or no
CUDA device is present, every entry point raises — there is no CPU fallback.
Return codes map to the reference's error convention: MISA_EINVAL -> ValueError
(``validation.py:8-51``), anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from ._build import LIB

MISA_OK = 0
MISA_EINVAL = -1
MISA_ECUDA = -2
MISA_EUNSUPPORTED = -3
FLAG_OVERFLOW = 1
FLAG_UNDERFLOW = 2

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_f32 = ctypes.c_float

# name -> argtypes (all return int except where noted)
SIGNATURES: dict[str, list] = {
    "misa_pool_keys": [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _i64, _vp],
    "misa_pool_append": [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _i64, _vp],
    "misa_route_scores": [_vp, _i64, _i32, _i32, _vp, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp, _vp],
    "misa_route_select": [_vp, _i32, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp],
    "misa_score_materialize": [_vp, _i64, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _i32,
                               _vp, _i64, _vp],
    "misa_score_materialize_split": [_vp, _i64, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp,
                                     _vp, _i32, _vp, _i64, _vp],
    "misa_score_materialize_paged": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp,
                                     _i32, _vp, _i32, _vp, _i64, _vp],
    "misa_score_filter": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _i32, _vp, _vp,
                          _i32, _vp, _vp],
    "misa_select_threshold": [_vp, _i64, _vp, _i64, _i32, _i32, _f32, _i64, _vp, _vp],
    "misa_select_topk": [_vp, _vp, _i32, _vp, _i64, _i32, _i64, _vp, _i64, _vp, _vp, _vp],
    "misa_select_dense": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _i64, _vp, _vp],
    "misa_select_dense_long": [_vp, _i64, _vp, _i64, _i32, _i64, _f32, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _i64,
                               _vp, _vp],
    "misa_refine_scores": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i64, _vp, _vp, _i32, _i64, _vp, _vp, _i64,
                           _vp],
    "misa_score_materialize_varlen": [_vp, _i64, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp,
                                      _vp, _vp, _i32, _vp, _i64, _vp],
    "misa_score_filter_varlen": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _vp,
                                 _i32, _vp, _vp, _i32, _vp, _vp],
    "misa_route_scores_varlen": [_vp, _i64, _i32, _i32, _vp, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i32,
                                 _vp, _vp],
    "misa_merge_topk": [_vp, _vp, _i32, _i64, _i64, _i32, _i32, _vp, _i64, _vp, _vp],
    "misa_list_kth": [_vp, _i64, _i64, _i32, _i32, _vp, _vp],
    "misa_list_prune": [_vp, _vp, _i64, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp],
    "misa_shard_map_indices": [_vp, _i64, _i32, _i32, _i32, _vp],
    "misa_select_topk_runs": [_vp, _vp, _i32, _vp, _i64, _i32, _i64, _vp, _i64, _vp, _vp, _vp],
    "misa_select_dense_runs": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _i64, _vp],
    "misa_refine_candidates": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i64, _vp, _vp, _i32, _i64, _vp, _vp,
                               _i32, _vp, _vp],
    "misa_score_filter_split": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _i32,
                                _vp, _vp, _i32, _vp, _vp],
    "misa_sort_rows": [_vp, _i64, _vp, _i64, _i32, _vp],
    "misa_sparse_attention": [_vp, _i64, _i32, _i32, _vp, _i64, _vp, _i64, _i32, _i32, _f32, _vp, _vp],
    "misa_relevance_dots": [_vp, _i64, _i32, _vp, _i32, _i32, _vp, _i64, _vp],
    "misa_pack_rows_f64": [_vp, _i64, _i32, _i64, _i64, _vp, _i32, _i64, _vp, _vp],
    "misa_quant_rows_fp8": [_vp, _i64, _i32, _vp, _vp, _vp],
}
EXTRA = {"misa_abi_version": ([], ctypes.c_int), "misa_last_error": ([], ctypes.c_char_p),
         "misa_sm_count": ([], ctypes.c_int)}

_lock = threading.Lock()
_handle: ctypes.CDLL | None = None


class MisaLibraryError(ImportError):
    pass


def load(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it was never built."""
    global _handle
    with _lock:
        if _handle is not None:
            return _handle
        path = path or LIB
        if not os.path.exists(path):
            raise MisaLibraryError(
                f"CUDA extension not built: {path} is missing. Run `python -m paper_2605_07363_b200._build` "
                "(or __graft_entry__.build()); this package has no CPU fallback.")
        lib = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        for name, (args, res) in EXTRA.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _handle = lib
        return lib


def last_error() -> str:
    msg = load().misa_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == MISA_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == MISA_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"misa_b200 error {rc}: {msg}")


# entry points that launch device work (counted for the bench's gpu_launches claim)
LAUNCHING = frozenset(n for n in SIGNATURES)
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(load(), name)(*args), name)
    if name in LAUNCHING:
        launch_count += 1
