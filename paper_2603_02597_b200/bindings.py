"""Serving handle: the counterpart of the reference's `lanebpe_bindings`.

`TokenizerHandle` keeps the constructor and call signature of
/root/reference/pkg/bindings/src/lanebpe_bindings/__init__.py:20-62: the
engine name is validated before anything is loaded, the tokenizer (and here
its device tables) is built once, and `tokenize_batch(texts)` returns
`(list[list[int]], engine_ms)` with engine_ms measured by CUDA events around
the encode kernels (the paper's kernel_time_ms).  One handle is
safe for concurrent calls: each call holds the device context's lock.
"""

from __future__ import annotations

from .chunker import ENGINE_NAMES, Tokenizer, tokenize_batch
from .engine import BlockConfig

__version__ = "0.1.0"  # mirrors the core package (bindings/__init__.py:15)


class TokenizerHandle:
    """`devices` (extension): an int N or a list of GPU indices to shard every
    batch across (tokenize_batch(..., devices=...)); default the current GPU."""

    __slots__ = ("_tokenizer", "_engine", "_workers", "_devices")

    def __init__(self, vocab_path, merges_path, engine: str = "optimized", *, lane_count: int = 256,
                 max_seq_len: int = 8192, chunk_budget: int | None = None,
                 workers: int | None = None, devices=None):
        if engine not in ENGINE_NAMES:
            raise ValueError(f"unknown engine {engine!r}, expected one of {ENGINE_NAMES}")
        cfg = BlockConfig(lane_count=lane_count, max_seq_len=max_seq_len, chunk_budget=chunk_budget)
        self._tokenizer = Tokenizer.from_files(vocab_path, merges_path, cfg)
        self._engine = engine
        self._workers = workers
        self._devices = devices

    @property
    def tokenizer(self) -> Tokenizer:
        return self._tokenizer

    def tokenize_batch(self, texts) -> tuple[list[list[int]], float]:
        res = tokenize_batch(texts, self._tokenizer, self._engine, workers=self._workers, devices=self._devices)
        return [ids.tolist() for ids in res.token_ids], res.engine_time_ms
