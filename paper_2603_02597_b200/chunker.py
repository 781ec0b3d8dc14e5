"""Tokenizer bundle and the batch API -- the drop-in surface of the encode path.

Mirrors /root/reference/pkg/src/lanebpe/chunker.py:
  * `Tokenizer(vocab, table, config=None, encoder=None)`, `.from_files`,
    `.encode` (bytes -> base ids), `.decode` (:67-101);
  * `tokenize_batch(texts, tokenizer, variant, workers) -> BatchResult`
    (:110-187) with the same output semantics: per input, greedy BPE of each
    fixed-offset chunk (`chunk_budget`, only when len > max_seq_len),
    concatenated; str inputs are UTF-8 encoded; BatchError(i) on a bad input;
    ValueError for an unknown engine name, raised before any work;
  * `chunk_tokens` / `Chunk` (:33-53) as host utilities.
The difference is where the work runs: the whole batch crosses to the GPU in
one packed call (bytes + offsets), chunking and merging happen on the device,
and one device-to-host copy returns the ids.  Every engine name the reference
accepts runs the CUDA engine (their outputs are identical by contract).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .byte_codec import ByteEncoder, Vocab, base_id_table, build_byte_encoder, decode_tokens, symbol_bytes
from .engine import BlockConfig, PassCounters
from .errors import BatchError, DeviceError, InvalidBudget, TokenizerError
from .merge_table import PackedPairTable, build_table, parse_merges, rule_arrays

ENGINE_NAMES = ("sequential", "baseline", "optimized", "cuda")


@dataclass(frozen=True)
class Chunk:
    source_index: int
    chunk_index: int
    tokens: np.ndarray


def chunk_tokens(tokens: np.ndarray, chunk_budget: int, source_index: int = 0) -> list[Chunk]:
    if chunk_budget < 2:
        raise InvalidBudget(f"chunk_budget must be >= 2, got {chunk_budget}")
    starts = range(0, len(tokens), chunk_budget)
    return [Chunk(source_index, k, tokens[s : s + chunk_budget]) for k, s in enumerate(starts)]


@dataclass
class BatchResult:
    token_ids: list[np.ndarray]
    engine_time_ms: float
    encode_ms: float = 0.0
    assemble_ms: float = 0.0
    counters: PassCounters = field(default_factory=PassCounters)
    device_stats: dict = field(default_factory=dict)


class Tokenizer:
    """Vocabulary + merge table + config; device tables are built lazily,
    once per GPU, on first use."""

    def __init__(self, vocab: Vocab, table: PackedPairTable, config: BlockConfig | None = None,
                 encoder: ByteEncoder | None = None):
        self.encoder = encoder if encoder is not None else build_byte_encoder()
        self.vocab = vocab
        self.table = table
        self.config = config if config is not None else BlockConfig()
        self._base_ids = base_id_table(self.encoder, vocab)
        self._devices: dict = {}

    @classmethod
    def from_files(cls, vocab_path, merges_path, config: BlockConfig | None = None) -> "Tokenizer":
        vocab = Vocab.from_file(vocab_path)
        rules = parse_merges(Path(merges_path).read_bytes(), vocab)
        return cls(vocab, build_table(rules), config)

    def encode(self, text: bytes) -> np.ndarray:
        """bytes -> base token ids, one per byte (no merges)."""
        return self._base_ids[np.frombuffer(bytes(text), dtype=np.uint8)]

    def decode(self, tokens) -> bytes:
        """Token ids -> bytes on the device (decode_tokens semantics,
        byte_codec.py:121-146; UnknownTokenId for ids outside the vocab)."""
        return self.device_encoder().decode_host([tokens])[0]

    def decode_batch(self, seqs) -> list[bytes]:
        """Many id sequences -> their byte strings in one device call."""
        return self.device_encoder().decode_host(seqs)

    def _decode_strings(self):
        """(ids, blob, offs) of every id whose symbol maps to bytes."""
        ids, pieces = [], []
        for tid, sym in self.vocab.id_to_symbol.items():
            b = symbol_bytes(sym, self.encoder)
            if b:
                ids.append(tid)
                pieces.append(b)
        offs = np.zeros(len(pieces) + 1, dtype=np.uint64)
        if pieces:
            offs[1:] = np.cumsum([len(p) for p in pieces])
        return np.array(ids, dtype=np.uint32), np.frombuffer(b"".join(pieces), dtype=np.uint8), offs

    def _vocab_strings(self):
        ids, pieces = [], []
        for tid, sym in self.vocab.id_to_symbol.items():
            b = symbol_bytes(sym, self.encoder)
            if b is not None and len(b) >= 2:
                ids.append(tid)
                pieces.append(b)
        offs = np.zeros(len(pieces) + 1, dtype=np.uint64)
        if pieces:
            offs[1:] = np.cumsum([len(p) for p in pieces])
        blob = np.frombuffer(b"".join(pieces), dtype=np.uint8)
        return np.array(ids, dtype=np.uint32), blob, offs

    def device_encoder(self, device: int | None = None, memo: bool = True, strict: bool = False):
        """The DeviceEncoder for `device` (built once, then cached)."""
        from .device import DeviceEncoder, _require_cuda

        if device is None:
            try:
                import torch

                device = torch.cuda.current_device()
            except Exception:  # no CUDA: DeviceError below
                _require_cuda()
                raise
        key = (int(device), memo, strict)
        enc = self._devices.get(key)
        if enc is None:
            _require_cuda()
            dev = int(device)
            left, right, rank, new = rule_arrays(self.table)
            vids, blob, offs = self._vocab_strings() if memo else (None, None, None)
            enc = DeviceEncoder(self._base_ids, left, right, rank, new, vids, blob, offs,
                                device=dev, memo=memo, strict=strict)
            enc.set_vocab(*self._decode_strings())
            self._devices[key] = enc
        return enc


def _as_bytes(text) -> bytes:
    return text.encode("utf-8") if isinstance(text, str) else bytes(text)


def pack_texts(texts) -> tuple[np.ndarray, np.ndarray]:
    """list[str|bytes] -> (uint8 data, int64 offsets); BatchError(i) on a bad item."""
    parts = []
    for i, text in enumerate(texts):
        try:
            parts.append(_as_bytes(text))
        except (TypeError, ValueError, UnicodeError) as exc:
            raise BatchError(i, str(exc)) from exc
    n = len(parts)
    offs = np.zeros(n + 1, dtype=np.int64)
    if n == 1:
        offs[1] = len(parts[0])
        return np.frombuffer(parts[0], dtype=np.uint8), offs
    if n:
        np.cumsum(np.fromiter(map(len, parts), dtype=np.int64, count=n), out=offs[1:])
    data = np.frombuffer(b"".join(parts), dtype=np.uint8)
    return data, offs


def tokenize_batch(texts, tokenizer: Tokenizer, variant: str = "optimized",
                   workers: int | None = None, pretokenize: str | None = None) -> BatchResult:
    """Tokenize a batch of str (UTF-8 encoded) or bytes documents on the GPU.

    `workers` is accepted for signature compatibility; the device engine
    parallelises internally.  pretokenize=None is the reference's semantics
    (no pre-tokenization); pretokenize="gpt2" splits at tiktoken's GPT-2
    regex first (ids equal tiktoken's GPT-2 encode_ordinary for valid UTF-8;
    an optional mode, never the default).
    """
    if variant not in ENGINE_NAMES:
        raise ValueError(f"unknown engine {variant!r}, expected one of {ENGINE_NAMES}")
    if pretokenize not in (None, "gpt2"):
        raise ValueError(f"unknown pretokenize {pretokenize!r}, expected None or 'gpt2'")
    cfg = tokenizer.config
    t0 = time.perf_counter()
    data, offs = pack_texts(texts)
    encode_ms = (time.perf_counter() - t0) * 1000.0
    n_docs = len(offs) - 1
    if n_docs == 0:
        return BatchResult([], 0.0, encode_ms, 0.0, PassCounters())
    try:
        enc = tokenizer.device_encoder()
        from ._native import MODE_DEFAULT, MODE_GPT2_REGEX

        ids, out_offs, st, engine_ms = enc.encode_packed_host(
            data, offs, cfg.max_seq_len, cfg.chunk_budget,
            MODE_GPT2_REGEX if pretokenize == "gpt2" else MODE_DEFAULT)
    except DeviceError:
        raise
    except TokenizerError as exc:  # pragma: no cover - the device reports no per-input errors
        raise BatchError(0, str(exc)) from exc
    t2 = time.perf_counter()
    token_ids = [ids[out_offs[i] : out_offs[i + 1]] for i in range(n_docs)]
    assemble_ms = (time.perf_counter() - t2) * 1000.0
    counters = PassCounters(passes=int(data.size) - int(ids.size))
    return BatchResult(token_ids, engine_ms, encode_ms, assemble_ms, counters, st)
