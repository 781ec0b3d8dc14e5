"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/gpubpe.h declares (no compute calls here)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "gpubpe.h"


def declared_symbols() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"\b(gpubpe_[a-z_]+)\s*\(", text))


def test_header_declares_the_api():
    syms = declared_symbols()
    assert {"gpubpe_ctx_create", "gpubpe_encode", "gpubpe_query", "gpubpe_last_error",
            "gpubpe_ctx_destroy", "gpubpe_lookup_pairs", "gpubpe_launches_per_encode"} <= syms


def test_library_exports_every_declared_symbol():
    from paper_2603_02597_b200 import _native

    if not _native.LIB_PATH.exists():
        pytest.skip("libgpubpe.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing
    assert set(_native.SIGNATURES) == declared_symbols()
    _native.load()
    assert lib.gpubpe_launches_per_encode() == 1


def test_stats_struct_matches_header():
    from paper_2603_02597_b200 import _native

    text = HEADER.read_text()
    body = text[text.index("typedef struct gpubpe_stats"): text.index("} gpubpe_stats;")]
    fields = re.findall(r"uint64_t\s+(\w+);", body)
    assert fields == [f for f, _ in _native.Stats._fields_]


def test_device_api_refuses_without_cuda(tokenizer):
    import torch

    from paper_2603_02597_b200.errors import DeviceError
    import paper_2603_02597_b200 as bpe

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(DeviceError):
        bpe.tokenize_batch([b"hello"], tokenizer)


def test_signatures_match_header_arity():
    """Every ctypes signature in _native.py has as many arguments as the
    prototype in include/gpubpe.h."""
    from paper_2603_02597_b200 import _native

    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    protos = dict(re.findall(r"\b(gpubpe_[a-z_]+)\s*\(([^;{]*?)\)\s*;", text))
    assert set(protos) == set(_native.SIGNATURES)
    for name, args in protos.items():
        n = 0 if args.strip() in ("", "void") else args.count(",") + 1
        assert len(_native.SIGNATURES[name][1]) == n, name


def test_hostlist_reads_bytes_addresses_through_the_c_api():
    """device.bytes_ptrs_lens (csrc/hostlist.c): data addresses and lengths of a
    list of bytes via PyBytes_AS_STRING; anything but bytes is a TypeError."""
    from paper_2603_02597_b200.device import bytes_ptrs_lens

    parts = [b"hello", b"", bytes(range(256)) * 40, b"\xff\x00x"]
    ptrs, lens = bytes_ptrs_lens(parts)
    assert lens.tolist() == [len(p) for p in parts]
    for p, a, n in zip(parts, ptrs, lens):
        assert ctypes.string_at(int(a), int(n)) == p
    with pytest.raises(TypeError):
        bytes_ptrs_lens([b"a", "str"])
    with pytest.raises(TypeError):
        bytes_ptrs_lens([bytearray(b"a")])
    assert [x.size for x in bytes_ptrs_lens([])] == [0, 0]


def test_hostlist_split_views():
    """chunker._split_views (csrc/hostlist.c split_views): per-document views of
    one result array, equal to Python slicing, keeping the array alive; empty
    documents, zero documents and bad offsets."""
    from paper_2603_02597_b200.chunker import _split_views

    ids = np.arange(1000, dtype=np.uint32)
    offs = np.array([0, 0, 3, 3, 700, 1000, 1000], np.int64)
    views = _split_views(ids, offs)
    o = offs.tolist()
    assert len(views) == 6
    for v, a, b in zip(views, o, o[1:]):
        assert v.dtype == np.uint32 and v.base is ids and v.tolist() == ids[a:b].tolist()
    assert _split_views(ids, np.zeros(1, np.int64)) == []
    with pytest.raises(ValueError):
        _split_views(ids, np.array([0, 5, 3], np.int64))
    with pytest.raises(ValueError):
        _split_views(ids, np.array([0, 1001], np.int64))
    del ids
    assert views[4].tolist() == list(range(700, 1000))  # the views keep the array alive
