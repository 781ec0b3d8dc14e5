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

from . import engine as _engine
from .byte_codec import ByteEncoder, Vocab, base_id_table, build_byte_encoder, decode_tokens, symbol_bytes
from .engine import BlockConfig, PassCounters, run_block_engine, sequential_bpe
from .errors import BatchError, DeviceError, InvalidBudget, TokenizerError
from .merge_table import MergeRule, PackedPairTable, build_table, parse_merges, rule_arrays

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

    def __init__(self, vocab: Vocab, table: PackedPairTable | None, config: BlockConfig | None = None,
                 encoder: ByteEncoder | None = None, *, rules=None):
        self.encoder = encoder if encoder is not None else build_byte_encoder()
        self.vocab = vocab
        if table is None and rules is None:
            raise ValueError("a Tokenizer needs a table (or the rule arrays it is built from)")
        self._table = table
        self._rules = rules  # (left, right, rank, new) uint32 in rank order, when parsed on the device
        self.config = config if config is not None else BlockConfig()
        self._base_ids = base_id_table(self.encoder, vocab)
        self._devices: dict = {}

    @property
    def table(self) -> PackedPairTable:
        """The packed pair table (merge_table.build_table, the reference's slot
        layout); built on first use when the merges were parsed on the device."""
        if self._table is None:
            left, right, rank, new = self._rules
            self._table = build_table([MergeRule(int(a), int(b), int(k), int(c))
                                       for a, b, k, c in zip(left.tolist(), right.tolist(), rank.tolist(),
                                                             new.tolist())])
        return self._table

    @table.setter
    def table(self, value: PackedPairTable) -> None:
        self._table = value
        self._rules = None

    def rule_arrays(self):
        """(left, right, rank, new) uint32 arrays in rank order."""
        return self._rules if self._rules is not None else rule_arrays(self.table)

    @classmethod
    def from_files(cls, vocab_path, merges_path, config: BlockConfig | None = None) -> "Tokenizer":
        vocab = Vocab.from_file(vocab_path)
        text = Path(merges_path).read_bytes()
        rules = _device_rules(text, vocab) if _device_parse_enabled() else None
        if rules is None:
            return cls(vocab, build_table(parse_merges(text, vocab)), config)
        return cls(vocab, None, config, rules=rules)

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

    def encode_batch_tensors(self, data, doc_offs):
        """Tensor-native batch encode: a packed batch
        already on the GPU -- data uint8[n], doc_offs int64[n_docs + 1] (cuda
        tensors) -> (ids int32[n_ids], offsets int64[n_docs + 1]) on the same
        device, under this tokenizer's BlockConfig.  One launch, one sync."""
        ids, offs, _ = self.device_encoder(data.device.index).encode_tensors(
            data, doc_offs, self.config.max_seq_len, self.config.chunk_budget)
        return ids, offs

    def _producers(self) -> dict:
        """token -> (left, right) of the lowest-rank rule producing it."""
        cached = getattr(self, "_prod_cache", None)
        if cached is None:
            cached = {}
            for a, b, c in zip(*(x.tolist() for x in (self.rule_arrays()[i] for i in (0, 1, 3)))):
                cached.setdefault(c, (a, b))
            self._prod_cache = cached
        return cached

    def _symbol_bytes(self):
        """(ids uint32[], blob uint8[], offs uint64[]) of every id whose symbol maps
        to a byte string -- empty symbols included, as b"" (decode_tokens,
        byte_codec.py:121-146) -- vectorised: all symbols are translated at
        once through a code point -> byte table."""
        cached = getattr(self, "_sym_cache", None)
        if cached is not None:
            return cached
        items = list(self.vocab.id_to_symbol.items())
        n = len(items)
        ids = np.fromiter((k for k, _ in items), dtype=np.uint32, count=n)
        syms = [v for _, v in items]
        lens = np.fromiter(map(len, syms), dtype=np.int64, count=n)
        cps = np.frombuffer("".join(syms).encode("utf-32-le"), dtype=np.uint32)
        s2b = self.encoder.symbol_to_byte
        top = max(map(ord, s2b)) + 1 if s2b else 1
        lut = np.full(top, -1, dtype=np.int32)
        for ch, byte in s2b.items():
            lut[ord(ch)] = byte
        val = np.where(cps < top, lut[np.minimum(cps, top - 1)], -1)
        seg = np.repeat(np.arange(n), lens)  # symbol index of every character
        bad = np.zeros(n, dtype=bool)
        bad[seg[val < 0]] = True
        keep = ~bad
        blob = val[keep[seg]].astype(np.uint8) if cps.size else np.empty(0, np.uint8)
        offs = np.zeros(int(keep.sum()) + 1, dtype=np.uint64)
        np.cumsum(lens[keep], out=offs[1:])
        self._sym_cache = (ids[keep], blob, offs)
        return self._sym_cache

    def _decode_strings(self):
        """(ids, blob, offs) of every id whose symbol maps to bytes."""
        return self._symbol_bytes()

    def _vocab_strings(self):
        """(ids, blob, offs) of the ids whose byte strings are >= 2 bytes (memo candidates)."""
        ids, blob, offs = self._symbol_bytes()
        lens = np.diff(offs)
        sel = lens >= 2
        if sel.all():
            return ids, blob, offs
        starts = offs[:-1][sel].astype(np.int64)
        ln = lens[sel].astype(np.int64)
        idx = np.repeat(starts - np.r_[0, np.cumsum(ln)[:-1]], ln) + np.arange(int(ln.sum()))
        o2 = np.zeros(int(sel.sum()) + 1, dtype=np.uint64)
        np.cumsum(ln, out=o2[1:].view(np.int64))
        return ids[sel], blob[idx], o2

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
            left, right, rank, new = self.rule_arrays()
            vids, blob, offs = self._vocab_strings() if memo else (None, None, None)
            enc = DeviceEncoder(self._base_ids, left, right, rank, new, vids, blob, offs,
                                device=dev, memo=memo, strict=strict)
            enc.set_vocab(*self._decode_strings())
            self._devices[key] = enc
        return enc


def _device_parse_enabled() -> bool:
    """Merges are parsed on the GPU when one is
    present; GPUBPE_HOST_PARSE=1 forces the host parser."""
    import os

    if os.environ.get("GPUBPE_HOST_PARSE"):
        return False
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover - torch is part of the image
        return False


def _device_rules(text: bytes, vocab: Vocab):
    """Rule arrays from the device parser, or None when the host path must run
    (it then raises the reference's exact error, or handles str.splitlines
    breaks): a duplicated pair or the reserved key go to build_table."""
    from .merge_table import EMPTY_KEY, parse_merges_device

    rules = parse_merges_device(text, vocab)
    if rules is None:
        return None
    left, right = rules[0].astype(np.uint64), rules[1].astype(np.uint64)
    keys = (left << np.uint64(32)) | right
    if (keys == np.uint64(EMPTY_KEY)).any() or np.unique(keys).size != keys.size:
        return None
    return rules


def _as_bytes(text) -> bytes:
    return text.encode("utf-8") if isinstance(text, str) else bytes(text)


def _as_parts(texts) -> list:
    """Every input as bytes (str UTF-8 encoded); BatchError(i) on a bad item."""
    if type(texts) is list and all(type(t) is bytes for t in texts):
        return texts  # already bytes: no per-item conversion
    parts = []
    for i, text in enumerate(texts):
        try:
            parts.append(_as_bytes(text))
        except (TypeError, ValueError, UnicodeError) as exc:
            raise BatchError(i, str(exc)) from exc
    return parts


def pack_texts(texts) -> tuple[np.ndarray, np.ndarray]:
    """list[str|bytes] -> (uint8 data, int64 offsets); BatchError(i) on a bad item."""
    parts = _as_parts(texts)
    n = len(parts)
    offs = np.zeros(n + 1, dtype=np.int64)
    if n == 1:
        offs[1] = len(parts[0])
        return np.frombuffer(parts[0], dtype=np.uint8), offs
    if n:
        np.cumsum(np.fromiter(map(len, parts), dtype=np.int64, count=n), out=offs[1:])
    data = np.frombuffer(b"".join(parts), dtype=np.uint8)
    return data, offs


class _LazyCounters(PassCounters):
    """PassCounters computed on first access (the batch path's counters are
    bookkeeping over the per-chunk id counts; most callers never read them)."""

    _FIELDS = ("passes", "lookups", "compaction_moves", "buffer_allocations")

    def __init__(self, fn):
        object.__setattr__(self, "_fn", fn)

    def __getattribute__(self, name):
        if name in _LazyCounters._FIELDS:
            d = object.__getattribute__(self, "__dict__")
            fn = d.pop("_fn", None)
            if fn is not None:
                d.update(fn())
        return object.__getattribute__(self, name)


def _split_views(ids: np.ndarray, offs: np.ndarray) -> list:
    """[ids[offs[i]:offs[i + 1]] for each document], built in C (csrc/hostlist.c)."""
    from .device import _hostlist

    o = np.ascontiguousarray(offs, dtype=np.int64)
    return _hostlist().split_views(np.ascontiguousarray(ids), o.ctypes.data, max(len(o) - 1, 0))


def _tri(x: np.ndarray) -> np.ndarray:
    return x * (x + 1) // 2


def _batch_counters(variant: str, tokenizer: "Tokenizer", clens: np.ndarray, couts: np.ndarray,
                    chunk_edges=None) -> dict:
    """The reference's PassCounters for a batch (chunker.py:166-172 sums the
    per-chunk engine counters) from each chunk's length n and id count:
    passes = n - out (every engine); lane engines (engines.py:338-403): one
    merge per pass, every evaluation probes cur_len - 1 pairs (a final one
    finds none while >= 2 ids remain), cur_len - 1 compaction moves per merge,
    two pool buffers per run of >= 2 ids; sequential (engines.py:269-335):
    n - 1 initial probes plus one per neighbour of every merge -- merges on
    the first output id's left spine / the last one's right spine lack one
    (walked through the rule producing each id)."""
    n = np.asarray(clens, dtype=np.int64)
    out = np.asarray(couts, dtype=np.int64)
    m = n - out
    run = n >= 2
    res = {"passes": int(m.sum()), "lookups": 0, "compaction_moves": 0, "buffer_allocations": 0}
    if variant == "sequential":
        lk = (n - 1) + 2 * m
        if chunk_edges is not None and m.any():
            prod = tokenizer._producers()
            for k in np.flatnonzero(m > 0).tolist():
                (fi, li), (fo, lo) = chunk_edges(k)
                lk[k] -= _spine(prod, fo, fi, 0) + _spine(prod, lo, li, 1)
        res["lookups"] = int(lk[run].sum())
        return res
    a = np.where(out >= 2, out, out + 1)
    res["lookups"] = int(((_tri(n - 1) - _tri(a - 2)) * run).sum())
    res["compaction_moves"] = int((m * (n - 1) - m * (m - 1) // 2).sum())
    res["buffer_allocations"] = 2 * int(np.count_nonzero(run))
    return res


def _spine(prod: dict, top: int, leaf: int, side: int) -> int:
    k = 0
    while top != leaf and top in prod:
        top = prod[top][side]
        k += 1
    return k


def _chunk_units(lens: np.ndarray, cfg: BlockConfig):
    """Chunks of a batch as tokenize_batch cuts them (chunker.py:139-144: a
    document longer than max_seq_len becomes chunk_budget-sized chunks).
    Returns (doc of each chunk, offset of each chunk in its document, chunk
    lengths, first chunk of each document + total) or None when no document
    is cut."""
    lens = np.asarray(lens, dtype=np.int64)
    long = lens > cfg.max_seq_len
    if not long.any():
        return None
    cb = cfg.chunk_budget
    k = np.where(long, (lens + cb - 1) // cb, 1)
    first = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(k, out=first[1:])
    doc = np.repeat(np.arange(len(lens)), k)
    idx = np.arange(int(first[-1])) - first[doc]
    off = idx * cb
    clen = np.where(long[doc], np.minimum(cb, lens[doc] - off), lens[doc])
    return doc, off, clen, first


def _per_chunk(parts, tokenizer: Tokenizer, variant: str) -> BatchResult:
    """The reference's per-chunk pipeline (chunker.py:139-179) through this
    module's `sequential_bpe` / `run_block_engine` (each a device engine run):
    the plugin seam the reference dispatches on.  tokenize_batch takes it only
    when one of those names was replaced (a caller's own engine, a test
    double) or a compaction fault is armed for the lane engines; otherwise
    the whole batch crosses to the device in one call."""
    cfg = tokenizer.config
    t0 = time.perf_counter()
    chunks = []
    for i, text in enumerate(parts):
        try:
            ids = tokenizer.encode(text)
        except (TokenizerError, TypeError, ValueError) as exc:
            raise BatchError(i, str(exc)) from exc
        chunks.extend(chunk_tokens(ids, cfg.chunk_budget, i) if len(ids) > cfg.max_seq_len else [Chunk(i, 0, ids)])
    encode_ms = (time.perf_counter() - t0) * 1000.0
    engine_s = 0.0
    totals = PassCounters()
    per_input: list[list[np.ndarray]] = [[] for _ in parts]
    for chunk in chunks:
        start = time.perf_counter()
        try:
            if variant == "sequential":
                out, counters = sequential_bpe(chunk.tokens, tokenizer.table)
            else:
                out, counters = run_block_engine(chunk.tokens, tokenizer.table, cfg,
                                                 "optimized" if variant == "cuda" else variant)
        except TokenizerError as exc:
            raise BatchError(chunk.source_index, str(exc)) from exc
        engine_s += time.perf_counter() - start
        totals.merge_from(counters)
        per_input[chunk.source_index].append(out)
    t2 = time.perf_counter()
    token_ids = [np.concatenate(p) if p else np.empty(0, dtype=np.uint32) for p in per_input]
    return BatchResult(token_ids, engine_s * 1000.0, encode_ms, (time.perf_counter() - t2) * 1000.0, totals)


def _device_list(devices) -> list[int] | None:
    if devices is None:
        return None
    if isinstance(devices, int):
        if devices < 1:
            raise ValueError(f"devices must be >= 1, got {devices}")
        return list(range(devices))
    lst = [int(d) for d in devices]
    if not lst:
        raise ValueError("devices must name at least one GPU")
    return lst


def _encode_units(parts, ptrs, lens, tokenizer: "Tokenizer", devs: list[int], mode: int):
    """Encode units (host address, length) -- whole documents or their chunks,
    each an independent BPE sequence -- on one or several GPUs.  Several: one
    host thread per GPU (the native calls release the GIL) over contiguous
    unit ranges balanced by bytes (multigpu.shard_batch); a unit larger than
    a GPU's share is split at exact cuts first (multigpu.split_points).
    Returns (list of (ids, unit offsets) per GPU, unit -> source unit index,
    engine_ms, stats).  No collective: per-GPU D2H of the ids only."""
    import threading

    from . import multigpu

    cfg = tokenizer.config
    g = len(devs)
    src = np.arange(len(lens))
    if g > 1 and len(lens):
        total = int(lens.sum())
        big = np.flatnonzero(lens > max(total // g, 1 << 20))
        if big.size:  # pieces at junction misses (exact cuts)
            jb = tokenizer.device_encoder(devs[0]).junction_bits()
            P, L, S = [], [], []
            bigset = set(big.tolist())
            for u in range(len(lens)):
                if u in bigset:
                    doc = ctypes_string(int(ptrs[u]), int(lens[u]))
                    pts = multigpu.split_points(doc, g, jb, 1 << 62, 1 << 62)
                    for a, b in zip(pts, pts[1:]):
                        if b > a:
                            P.append(int(ptrs[u]) + a), L.append(b - a), S.append(u)
                else:
                    P.append(int(ptrs[u])), L.append(int(lens[u])), S.append(u)
            ptrs, lens, src = np.array(P, np.uint64), np.array(L, np.uint64), np.array(S, np.int64)
        offs = np.zeros(len(lens) + 1, np.int64)
        np.cumsum(lens.astype(np.int64), out=offs[1:])
        ranges = multigpu.shard_batch(offs, g)
    else:
        ranges = [(0, len(lens))]
    encs = [tokenizer.device_encoder(d) for d in devs[: len(ranges)]]
    results: list = [None] * len(ranges)
    errs: list = []

    def run(k):
        try:
            a, b = ranges[k]
            if b > a:
                results[k] = encs[k].encode_ptrs_host(ptrs[a:b], lens[a:b], cfg.max_seq_len, cfg.chunk_budget, mode)
        except BaseException as exc:  # re-raised in the caller
            errs.append(exc)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(1, len(ranges))]
    for t in threads:
        t.start()
    run(0)
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    done = [r for r in results if r is not None]
    if len(ranges) == 1:
        st = done[0][2] if done else {"n_bytes": 0, "allocations": 0}
    else:
        st = {"devices": devs, "per_device": [r[2] if r else None for r in results],
              "n_bytes": sum(int(r[2]["n_bytes"]) for r in done),
              "allocations": sum(int(r[2]["allocations"]) for r in done)}
    engine_ms = max((r[3] for r in done), default=0.0)  # the GPUs run concurrently
    return [(r[0], r[1]) for r in done], src, engine_ms, st


def ctypes_string(ptr: int, n: int) -> bytes:
    import ctypes

    return ctypes.string_at(ptr, n)


def tokenize_batch(texts, tokenizer: Tokenizer, variant: str = "optimized",
                   workers: int | None = None, pretokenize: str | None = None,
                   devices=None) -> BatchResult:
    """Tokenize a batch of str (UTF-8 encoded) or bytes documents on the GPU.

    `workers` is accepted for signature compatibility; the device engine
    parallelises internally.  `devices` (an int N for GPUs 0..N-1, or a list
    of GPU indices; default: the current GPU) shards the batch across GPUs
    from this one process.  pretokenize=None is the reference's semantics
    (no pre-tokenization); pretokenize="gpt2" splits at tiktoken's GPT-2
    regex first (ids equal tiktoken's GPT-2 encode_ordinary for valid UTF-8;
    an optional mode, never the default).

    Documents longer than max_seq_len cross to the device as their chunks
    (the reference encodes chunks independently, chunker.py:139-144), so the
    per-chunk id counts -- and with them the reference's counters -- come
    back with the ids.  device_stats["allocations"] counts device / pinned
    buffers the call allocated (0 in steady state).
    """
    if variant not in ENGINE_NAMES:
        raise ValueError(f"unknown engine {variant!r}, expected one of {ENGINE_NAMES}")
    if pretokenize not in (None, "gpt2"):
        raise ValueError(f"unknown pretokenize {pretokenize!r}, expected None or 'gpt2'")
    devs = _device_list(devices)
    cfg = tokenizer.config
    t0 = time.perf_counter()
    parts = _as_parts(texts)
    encode_ms = (time.perf_counter() - t0) * 1000.0
    n_docs = len(parts)
    if n_docs == 0:
        return BatchResult([], 0.0, encode_ms, 0.0, PassCounters())
    if pretokenize is None and (
            run_block_engine is not _engine.run_block_engine or sequential_bpe is not _engine.sequential_bpe
            or (variant in ("baseline", "optimized") and getattr(_engine._fault_armed, "flag", False))):
        return _per_chunk(parts, tokenizer, variant)
    from ._native import MODE_DEFAULT, MODE_GPT2_REGEX

    mode = MODE_GPT2_REGEX if pretokenize == "gpt2" else MODE_DEFAULT
    if n_docs == 1 and (devs is None or len(devs) == 1):
        # one document (the latency path): one buffer staged piecewise, overlapping
        # its DMA; a document longer than max_seq_len goes as its chunks
        enc = tokenizer.device_encoder(devs[0] if devs else None)
        doc = parts[0]
        n = len(doc)
        if mode == MODE_DEFAULT:  # one C call: chunk offsets, encode, counters
            ids, out_offs, st, engine_ms = enc.encode_bytes_host(doc, cfg.max_seq_len, cfg.chunk_budget)
        else:
            ids, out_offs, st, engine_ms = enc.encode_packed_host(np.frombuffer(doc, dtype=np.uint8),
                                                                  np.array([0, n], np.int64),
                                                                  cfg.max_seq_len, cfg.chunk_budget, mode)
        t1 = time.perf_counter()
        chunked = mode == MODE_DEFAULT and n > cfg.max_seq_len

        def counters1():  # (on first read) the chunk offsets the device encoded, then the counters
            offs = (np.append(np.arange(0, n, cfg.chunk_budget, dtype=np.int64), n) if chunked
                    else np.array([0, n], np.int64))
            base, data = tokenizer._base_ids, np.frombuffer(doc, dtype=np.uint8)

            def edges1(k):
                a, b, c, d = int(offs[k]), int(offs[k + 1]), int(out_offs[k]), int(out_offs[k + 1])
                return (int(base[data[a]]), int(base[data[b - 1]])), (int(ids[c]), int(ids[d - 1]))

            return _batch_counters(variant, tokenizer, np.diff(offs), np.diff(out_offs), edges1)

        counters = _LazyCounters(counters1)
        return BatchResult([ids], engine_ms, encode_ms, (time.perf_counter() - t1) * 1000.0, counters, st)
    from .device import bytes_ptrs_lens

    ptrs, lens = bytes_ptrs_lens(parts)
    cut = _chunk_units(lens, cfg) if mode == MODE_DEFAULT else None
    if cut is not None:  # documents longer than max_seq_len as their chunks
        cdoc, coff, clen, first = cut
        uptrs, ulens = ptrs[cdoc] + coff.astype(np.uint64), clen.astype(np.uint64)
    else:
        uptrs, ulens = ptrs, lens
    pieces, src, engine_ms, st = _encode_units(parts, uptrs, ulens, tokenizer, devs or [None], mode)
    t1 = time.perf_counter()
    # per source unit: id count; per document: its ids (one slice when on one GPU)
    if len(pieces) == 1 and len(src) == len(ulens):
        ids, uo = pieces[0]
        uout = np.diff(uo)
        token_ids = _split_views(ids, uo if cut is None else uo[first])
    else:
        pout = np.concatenate([np.diff(o) for _, o in pieces])
        uout = np.bincount(src, weights=pout, minlength=len(ulens)).astype(np.int64)
        flat = np.concatenate([i for i, _ in pieces]) if pieces else np.empty(0, np.uint32)
        uo = np.zeros(len(ulens) + 1, np.int64)
        np.cumsum(uout, out=uo[1:])
        token_ids = _split_views(flat, uo if cut is None else uo[first])
    cl = ulens.astype(np.int64)
    uo_all = np.zeros(len(cl) + 1, np.int64)
    np.cumsum(uout, out=uo_all[1:])
    all_ids = token_ids  # for the sequential counters' edge ids

    def edges(k):
        d = int(cdoc[k]) if cut is not None else k
        o = int(coff[k]) if cut is not None else 0
        b = parts[d]
        base = tokenizer._base_ids
        ids_d = all_ids[d]
        lo = int(uo_all[k] - (uo_all[first[d]] if cut is not None else uo_all[k]))
        hi = lo + int(uout[k])
        return ((int(base[b[o]]), int(base[b[o + int(cl[k]) - 1]])), (int(ids_d[lo]), int(ids_d[hi - 1])))

    counters = _LazyCounters(lambda: _batch_counters(variant, tokenizer, cl, uout, edges))
    return BatchResult(token_ids, engine_ms, encode_ms, (time.perf_counter() - t1) * 1000.0, counters, st)
