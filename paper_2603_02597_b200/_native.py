"""ctypes binding of libgpubpe.so (the C ABI declared in include/gpubpe.h).

This is the binding a maintainer of the reference would add:
plain pointers and sizes; device pointers come from torch tensors, the stream
from torch.cuda.  ctypes releases the GIL for the duration of every call.

There is no fallback: if the shared library is missing or fails to load, every
product entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import DeviceError

import os

# GPUBPE_LIB selects an alternative in-tree build (tuning experiments only)
LIB_PATH = Path(__file__).resolve().parent / os.environ.get("GPUBPE_LIB", "libgpubpe.so")

OK, EINVAL, ECUDA, ENOMEM, ETABLE, ERANGE = 0, 1, 2, 3, 4, 5
F_NO_MEMO, F_STRICT, F_HOST_TABLES = 1, 2, 4
MODE_DEFAULT, MODE_GPT2_REGEX = 0, 1

# (name, restype, argtypes) for every entry point of include/gpubpe.h
_vp, _u32p, _u8p, _u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.c_void_p, ctypes.c_void_p
_u64, _int = ctypes.c_uint64, ctypes.c_int


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "n_bytes", "n_ids", "passes", "n_segments", "memo_hits", "short_merges",
        "medium_segments", "giant_segments", "giant_bytes", "engine_passes", "tiles",
        "overflow", "well_formed", "allocations")]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n in _STAT_NAMES}


_STAT_NAMES = tuple(n for n, _ in Stats._fields_)


def stats_dict(values) -> dict:
    """gpubpe_stats fields (a tuple in header order) as the device_stats dict."""
    return dict(zip(_STAT_NAMES, values))

SIGNATURES = {
    "gpubpe_ctx_create": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _u64,
                                 ctypes.c_uint32, ctypes.POINTER(_vp)]),
    "gpubpe_encode": (_int, [_vp, _vp, _u64, _vp, _u64, _u64, _u64, _vp, _vp, _vp]),
    "gpubpe_encode_host": (_int, [_vp, _vp, _u64, _vp, _u64, _u64, _u64, _vp, _vp,
                                  ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_float), _vp]),
    "gpubpe_encode_host_gather": (_int, [_vp, _vp, _vp, _u64, _u64, _u64, _vp, _vp,
                                         ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_float), _vp]),
    "gpubpe_host_alloc": (_int, [_int, _u64, ctypes.POINTER(_vp)]),
    "gpubpe_host_free": (None, [_vp]),
    "gpubpe_query": (_int, [_vp, _vp, ctypes.POINTER(Stats)]),
    "gpubpe_junction_bits": (_int, [_vp, _vp]),
    "gpubpe_set_pretok": (_int, [_vp, _vp, _u64]),
    "gpubpe_set_mode": (_int, [_vp, ctypes.c_uint32]),
    "gpubpe_set_vocab": (_int, [_vp, _vp, _vp, _vp, _u64]),
    "gpubpe_decode": (_int, [_vp, _vp, _u64, _vp, _u64, _vp, _u64, _vp, ctypes.POINTER(ctypes.c_uint64),
                             ctypes.POINTER(ctypes.c_uint64), _vp]),
    "gpubpe_merge_tokens": (_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "gpubpe_merge_tokens_ex": (_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, ctypes.c_int64, _vp]),
    "gpubpe_eval_pairs": (_int, [_vp, _vp, _u64, _vp, _vp]),
    "gpubpe_compact": (_int, [_vp, _u64, _u64, ctypes.c_uint32, _vp, _int, _vp]),
    "gpubpe_lookup_keys": (_int, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "gpubpe_parse_merges": (_int, [_int, _vp, _vp, _vp, _u64, _vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "gpubpe_launches_per_encode": (_int, []),
    "gpubpe_lookup_pairs": (_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "gpubpe_set_profiling": (_int, [_vp, _int]),
    "gpubpe_kernel_ms": (_int, [_vp, ctypes.POINTER(ctypes.c_float), _int]),
    "gpubpe_last_error": (ctypes.c_char_p, [_vp]),
    "gpubpe_ctx_destroy": (None, [_vp]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load and type the shared library (raises DeviceError if absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeviceError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            try:
                lib = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, ctx, what: str) -> None:
    if rc == OK:
        return
    msg = load().gpubpe_last_error(ctx).decode("utf-8", "replace") if ctx else ""
    if rc == EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise DeviceError(f"{what} failed (code {rc}): {msg}")
