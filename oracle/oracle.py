"""CPU oracle for the GPT-2 byte-level BPE encode path.

TEST INFRASTRUCTURE ONLY -- the parity checker and the CPU baseline ("port").
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module.  The product package (paper_2603_02597_b200) never imports it; it
has no CPU fallback.

It restates the reference (paths relative to /root/reference/pkg):

* the byte <-> symbol bijection          src/lanebpe/byte_codec.py:26,37-55
* vocab.json / merges.txt parsing        src/lanebpe/byte_codec.py:80-88,
                                          src/lanebpe/merge_table.py:88-116
* per-byte base ids                      src/lanebpe/byte_codec.py:97-118
* the merge table + sequential engine +  bpe_oracle.c (merge_table.py:28-278,
  chunked batch pipeline                   engines.py:269-335, chunker.py:42-187)
* the naive rescan greedy loop           tests/reference.py:18-39 and
                                          tools/gen_golden.py:44-58 (pure Python,
                                          small inputs only)

Pinned against the reference's own 100 golden files and known-answer ids
(tests/golden/, see tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import gzip
import json
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liborc.so"

_ERRORS = {1: "duplicate pair", 2: "reserved key", 3: "out of memory", 4: "bad argument"}


# ------------------------------------------------------------ byte codec


def byte_symbols() -> list[str]:
    """byte value -> one-character symbol (byte_codec.py:26,37-55)."""
    keep = set(range(0x21, 0x7F)) | set(range(0xA1, 0xAD)) | set(range(0xAE, 0x100))
    out: list[str] = []
    nxt = 256
    for b in range(256):
        if b in keep:
            out.append(chr(b))
        else:
            out.append(chr(nxt))
            nxt += 1
    return out


def _read_text(path) -> str:
    path = Path(path)
    raw = path.read_bytes()
    if path.suffix == ".gz":
        raw = gzip.decompress(raw)
    return raw.decode("utf-8")


@dataclass
class OracleTables:
    symbol_to_id: dict[str, int]
    base_ids: np.ndarray  # uint32[256]
    left: np.ndarray  # uint32[n_rules]
    right: np.ndarray
    rank: np.ndarray
    new: np.ndarray

    @property
    def pair_map(self) -> dict[tuple[int, int], tuple[int, int]]:
        return {
            (int(l), int(r)): (int(k), int(n))
            for l, r, k, n in zip(self.left, self.right, self.rank, self.new)
        }


def load_tables(vocab_path, merges_path) -> OracleTables:
    vocab = json.loads(_read_text(vocab_path))
    lines = _read_text(merges_path).splitlines()
    if lines and lines[0].startswith("#"):
        lines = lines[1:]
    left, right, new = [], [], []
    for line in lines:
        a, b = line.split(" ")
        left.append(vocab[a])
        right.append(vocab[b])
        new.append(vocab[a + b])
    syms = byte_symbols()
    base = np.array([vocab[s] for s in syms], dtype=np.uint32)
    n = len(left)
    return OracleTables(
        vocab,
        base,
        np.array(left, dtype=np.uint32),
        np.array(right, dtype=np.uint32),
        np.arange(n, dtype=np.uint32),
        np.array(new, dtype=np.uint32),
    )


# ------------------------------------------------------------ pure python


def greedy_merge(ids, pair_map) -> list[int]:
    """Naive rescan loop: merge the lowest-rank pair, leftmost on ties."""
    ids = [int(t) for t in ids]
    while len(ids) >= 2:
        best, pos = None, -1
        for i in range(len(ids) - 1):
            hit = pair_map.get((ids[i], ids[i + 1]))
            if hit is not None and (best is None or hit[0] < best):
                best, pos = hit[0], i
        if best is None:
            break
        ids[pos : pos + 2] = [pair_map[(ids[pos], ids[pos + 1])][1]]
    return ids


# ------------------------------------------------------------ C core


def build_lib() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build_lib()
        L = ctypes.CDLL(str(LIB_PATH))
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64 = ctypes.c_uint64
        L.orc_table_build.argtypes = [u32p, u32p, u32p, u32p, u64, ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(u64)]
        L.orc_table_build.restype = ctypes.c_int
        L.orc_table_free.argtypes = [ctypes.c_void_p]
        L.orc_table_lookup.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p]
        L.orc_table_lookup.restype = ctypes.c_int
        L.orc_sequential_bpe.argtypes = [ctypes.c_void_p, u32p, u64, u32p, ctypes.POINTER(u64), u32p]
        L.orc_sequential_bpe.restype = u64
        L.orc_tokenize_batch.argtypes = [ctypes.c_void_p, u32p, ctypes.c_void_p, ctypes.c_void_p,
                                         u64, u64, u64, ctypes.c_int, u32p, ctypes.c_void_p,
                                         ctypes.POINTER(u64)]
        L.orc_tokenize_batch.restype = ctypes.c_int
        _lib = L
    return _lib


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


class OracleEncoder:
    """C restatement of Tokenizer + sequential_bpe + tokenize_batch."""

    def __init__(self, base_ids, left, right, rank, new):
        self.base_ids = np.ascontiguousarray(base_ids, dtype=np.uint32)
        arrs = [np.ascontiguousarray(a, dtype=np.uint32) for a in (left, right, rank, new)]
        self._arrs = arrs
        h = ctypes.c_void_p()
        err = ctypes.c_uint64()
        rc = lib().orc_table_build(*[_u32p(a) for a in arrs], len(arrs[0]), ctypes.byref(h),
                                   ctypes.byref(err))
        if rc:
            raise ValueError(f"oracle table build: {_ERRORS.get(rc, rc)} at rule {err.value}")
        self._h = h

    @classmethod
    def from_tables(cls, t: OracleTables) -> "OracleEncoder":
        return cls(t.base_ids, t.left, t.right, t.rank, t.new)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.orc_table_free(h)
            self._h = None

    def lookup(self, l: int, r: int):
        n, k = ctypes.c_uint32(), ctypes.c_uint32()
        if lib().orc_table_lookup(self._h, l, r, ctypes.byref(n), ctypes.byref(k)):
            return n.value, k.value
        return None

    def base(self, data: bytes) -> np.ndarray:
        return self.base_ids[np.frombuffer(bytes(data), dtype=np.uint8)]

    def sequential_bpe(self, tokens, with_trace: bool = False):
        toks = np.ascontiguousarray(tokens, dtype=np.uint32)
        out = np.empty(max(len(toks), 1), dtype=np.uint32)
        trace = np.empty(max(len(toks), 1), dtype=np.uint32) if with_trace else None
        passes = ctypes.c_uint64(0)
        m = lib().orc_sequential_bpe(self._h, _u32p(toks), len(toks), _u32p(out),
                                     ctypes.byref(passes), _u32p(trace) if with_trace else None)
        if m == 2**64 - 1:
            raise MemoryError("oracle")
        if with_trace:
            return out[:m].copy(), trace[: passes.value].copy()
        return out[:m].copy()

    def encode_packed(self, data: np.ndarray, offs: np.ndarray, max_seq_len: int,
                      chunk_budget: int, threads: int = 1):
        """Packed CSR batch -> (ids uint32[total], offsets int64[n_docs+1], passes)."""
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        n_docs = len(offs) - 1
        total = int(offs[-1]) if n_docs > 0 else 0
        ids = np.empty(max(total, 1), dtype=np.uint32)
        out_offs = np.zeros(n_docs + 1, dtype=np.int64)
        passes = ctypes.c_uint64(0)
        rc = lib().orc_tokenize_batch(
            self._h, _u32p(self.base_ids), data.ctypes.data_as(ctypes.c_void_p),
            offs.ctypes.data_as(ctypes.c_void_p), n_docs, int(max_seq_len), int(chunk_budget),
            int(threads), _u32p(ids), out_offs.ctypes.data_as(ctypes.c_void_p), ctypes.byref(passes))
        if rc:
            raise ValueError(f"oracle batch: {_ERRORS.get(rc, rc)}")
        return ids[: int(out_offs[-1])], out_offs, passes.value

    def encode_docs(self, docs, max_seq_len: int = 8192, chunk_budget: int | None = None,
                    threads: int = 1) -> list[np.ndarray]:
        data, offs = pack_docs(docs)
        ids, out_offs, _ = self.encode_packed(data, offs, max_seq_len,
                                              chunk_budget or max_seq_len, threads)
        return [ids[out_offs[i] : out_offs[i + 1]] for i in range(len(offs) - 1)]


def pack_docs(docs) -> tuple[np.ndarray, np.ndarray]:
    bs = [d.encode("utf-8") if isinstance(d, str) else bytes(d) for d in docs]
    offs = np.zeros(len(bs) + 1, dtype=np.int64)
    if bs:
        offs[1:] = np.cumsum([len(b) for b in bs])
    data = np.frombuffer(b"".join(bs), dtype=np.uint8) if bs else np.empty(0, np.uint8)
    return data, offs


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
