"""Deterministic synthetic English-like text for parity fixtures and the bench.

WikiText-103 is not available offline, so the benchmark text is generated:
Zipf-weighted GPT-2 word tokens (the vocab symbols "Ġ[a-z]+" that are
dictionary words, ranked by id, which tracks merge rank and therefore corpus
frequency),
capitalised sentence starts, commas, numbers, sentence punctuation and
paragraph breaks ("\\n\\n").  Generation is vectorised numpy, deterministic for
a given (seed, numpy version).

`SIZES` pins, for each named workload, the byte length that BPE-encodes to the
named number of output tokens under whole-sequence semantics (P-whole).  The
lengths were calibrated with the CPU oracle (oracle/, pinned to the reference)
by tests/golden/make_golden.py; the bench re-checks the count on the device.
"""

from __future__ import annotations

import gzip
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
GPT2_DIR = REPO / "tests" / "golden" / "gpt2"
VOCAB_GZ = GPT2_DIR / "vocab.json.gz"
MERGES_GZ = GPT2_DIR / "merges.txt.gz"

# name -> (seed, n_bytes, expected P-whole tokens); filled by make_golden.py
SIZES_FILE = REPO / "tests" / "golden" / "synth_sizes.json"


WORDS_GZ = REPO / "tests" / "golden" / "synth_words.txt.gz"


@lru_cache(maxsize=1)
def _word_table():
    """Returns (blob uint8, offs int64, lens int64, probs, n) for the word pool.

    synth_words.txt.gz lists the GPT-2 "Ġ[a-z]+" symbols that are dictionary
    words, in GPT-2 id order (made once by tests/golden/make_golden.py).
    """
    words = gzip.decompress(WORDS_GZ.read_bytes()).decode("ascii").split()
    lower = [(" " + w).encode("ascii") for w in words]
    n = len(lower)
    ranks = np.arange(n, dtype=np.float64)
    probs = 1.0 / np.power(ranks + 2.7, 1.07)
    probs /= probs.sum()
    variants = []  # [lower, capitalised with space, capitalised no space]
    for w in lower:
        variants.append(w)
    for w in lower:
        variants.append(b" " + w[1:2].upper() + w[2:])
    for w in lower:
        variants.append(w[1:2].upper() + w[2:])
    lens = np.array([len(v) for v in variants], dtype=np.int64)
    offs = np.zeros(len(variants) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    blob = np.frombuffer(b"".join(variants), dtype=np.uint8)
    return blob, offs, lens, probs, n


def _numbers(rng: np.random.Generator, k: int) -> list[bytes]:
    out = []
    kinds = rng.integers(0, 4, size=k)
    vals = rng.integers(0, 100000, size=k)
    for kind, v in zip(kinds, vals):
        if kind == 0:
            out.append(b" %d" % (1800 + v % 225))
        elif kind == 1:
            out.append(b" %d" % (v % 100))
        elif kind == 2:
            out.append(b" %d.%d" % (v % 50, v % 10))
        else:
            out.append((" " + format(int(v) * 10, ",")).encode())
    return out


BLOCK_WORDS = 1 << 16


def _block(seed: int, i: int) -> bytes:
    """Block i of the stream for `seed` (~380 KB); blocks are independent."""
    blob, offs, lens, probs, n = _word_table()
    rng = np.random.default_rng([seed, i])
    k = BLOCK_WORDS
    idx = rng.choice(n, size=k, p=probs)
    # sentence structure: 6..20 words, paragraph break after ~1 in 5 sentences
    sent_len = rng.integers(6, 21, size=k // 6 + 2)
    ends = np.cumsum(sent_len)
    ends = ends[ends < k]
    starts = np.concatenate(([0], ends))
    para = rng.random(len(starts)) < 0.2
    variant = np.zeros(k, dtype=np.int64)
    variant[starts] = 1
    variant[starts[para]] = 2
    if i == 0:
        variant[0] = 2
    wid = idx + variant * n
    wl = lens[wid]
    pos = np.repeat(offs[wid] - np.concatenate(([0], np.cumsum(wl)[:-1])), wl)
    text = blob[pos + np.arange(int(wl.sum()))].tobytes()
    # splice punctuation / numbers at word boundaries
    bounds = np.concatenate(([0], np.cumsum(wl)))
    marks: dict[int, bytes] = {}
    punct = rng.random(len(ends))
    for e, p, brk in zip(ends, punct, para[1 : len(ends) + 1]):
        mark = b"." if p < 0.9 else (b"?" if p < 0.95 else b"!")
        marks[int(bounds[e])] = mark + (b"\n\n" if brk else b"")
    for c in np.nonzero(rng.random(k) < 0.06)[0]:
        marks.setdefault(int(bounds[c + 1]), b",")
    nums = np.nonzero(rng.random(k) < 0.02)[0]
    for c, t in zip(nums, _numbers(rng, len(nums))):
        b = int(bounds[c + 1])
        marks[b] = marks.get(b, b"") + t
    pieces = []
    last = 0
    for b in sorted(marks):
        pieces.append(text[last:b])
        pieces.append(marks[b])
        last = b
    pieces.append(text[last:])
    return b"".join(pieces) + b"."


def english_bytes(n_bytes: int, seed: int = 0) -> bytes:
    """The first n_bytes of the synthetic prose stream for `seed`.

    The stream is a concatenation of independently seeded blocks, so a
    shorter request is always a prefix of a longer one.
    """
    parts = []
    total = 0
    i = 0
    while total < n_bytes:
        blk = _block(seed, i)
        parts.append(blk)
        total += len(blk)
        i += 1
    return b"".join(parts)[: max(n_bytes, 0)]


def load_sizes() -> dict:
    if SIZES_FILE.exists():
        return json.loads(SIZES_FILE.read_text())
    return {}


def workload_doc(name: str) -> tuple[bytes, int]:
    """(bytes, expected P-whole token count) for a calibrated named workload."""
    spec = load_sizes()[name]
    return english_bytes(spec["n_bytes"], spec["seed"]), spec["tokens_whole"]


def _corpus_layout(total_bytes: int, seed: int, min_doc: int, max_doc: int, pool_bytes: int):
    """(pool, sizes, starts, offs) of the corpus: document i is
    pool[starts[i] : starts[i] + sizes[i]], packed at offs[i]."""
    rng = np.random.default_rng(seed + 7919)
    pool = np.frombuffer(english_bytes(min(pool_bytes, max(total_bytes, max_doc) + max_doc), seed),
                         dtype=np.uint8)
    # sizes drawn one uniform per document until the total is reached (vectorised:
    # a generous draw to find the count, then exactly that many from a fresh
    # generator, so the stream position of the start draws below is unchanged)
    lo, hi = np.log(min_doc), np.log(max_doc)
    guess = int(total_bytes / np.exp((lo + hi) / 2) * 1.5) + 64
    while True:
        s = np.exp(np.random.default_rng(seed + 7919).uniform(lo, hi, size=guess)).astype(np.int64)
        c = np.cumsum(s)
        k = int(np.searchsorted(c, total_bytes, side="left")) + 1  # documents needed
        if k <= guess or total_bytes <= 0:
            break
        guess *= 2
    if total_bytes <= 0:
        k = 0
    rng.uniform(lo, hi, size=k)  # advance past the size draws
    sizes = s[:k].copy()
    if k:
        sizes[-1] = total_bytes - (int(c[k - 2]) if k > 1 else 0)
    offs = np.zeros(len(sizes) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(sizes)
    starts = rng.integers(0, len(pool) - max_doc, size=len(sizes))
    return pool, sizes, starts, offs


def _fill(pool, sizes, starts, docs) -> tuple[np.ndarray, np.ndarray]:
    """Pack the documents `docs` (indices, in order) -> (uint8 data, int64 offsets)."""
    docs = np.asarray(docs, dtype=np.int64)
    offs = np.zeros(len(docs) + 1, dtype=np.int64)
    if len(docs):
        np.cumsum(sizes[docs], out=offs[1:])
    data = np.empty(int(offs[-1]), dtype=np.uint8)
    for k, i in enumerate(docs.tolist()):
        st = int(starts[i])
        data[offs[k] : offs[k + 1]] = pool[st : st + int(sizes[i])]
    return data, offs


def corpus_docs(total_bytes: int, seed: int = 0, min_doc: int = 1024, max_doc: int = 65536,
                pool_bytes: int = 64 << 20) -> tuple[np.ndarray, np.ndarray]:
    """Packed corpus of documents with log-uniform sizes in [min_doc, max_doc].

    Documents are slices of a pool of generated prose (so 10 GB does not need
    10 GB of generation).  Returns (uint8 data, int64 offsets).
    """
    pool, sizes, starts, offs = _corpus_layout(total_bytes, seed, min_doc, max_doc, pool_bytes)
    return _fill(pool, sizes, starts, np.arange(len(sizes)))


def corpus_layout_offsets(total_bytes: int, seed: int = 0, min_doc: int = 1024, max_doc: int = 65536,
                          pool_bytes: int = 64 << 20) -> np.ndarray:
    """The corpus's document offsets only (no data)."""
    return _corpus_layout(total_bytes, seed, min_doc, max_doc, pool_bytes)[3]


def corpus_range(total_bytes: int, d0: int, d1: int, seed: int = 0, min_doc: int = 1024,
                 max_doc: int = 65536, pool_bytes: int = 64 << 20) -> tuple[np.ndarray, np.ndarray]:
    """Documents [d0, d1) of corpus_docs(total_bytes, seed) -- one rank's shard,
    generated without the rest of the corpus.  Returns (data, offsets from 0)."""
    pool, sizes, starts, _ = _corpus_layout(total_bytes, seed, min_doc, max_doc, pool_bytes)
    return _fill(pool, sizes, starts, np.arange(d0, d1))


def corpus_sample(total_bytes: int, frac: float, sample_seed: int, seed: int = 0, min_doc: int = 1024,
                  max_doc: int = 65536, pool_bytes: int = 64 << 20):
    """A seeded sample of about `frac` of the corpus's documents:
    (document indices, data, offsets) -- the documents are byte-identical to
    those of corpus_docs(total_bytes, seed)."""
    pool, sizes, starts, _ = _corpus_layout(total_bytes, seed, min_doc, max_doc, pool_bytes)
    rng = np.random.default_rng(sample_seed)
    pick = np.flatnonzero(rng.random(len(sizes)) < frac)
    data, offs = _fill(pool, sizes, starts, pick)
    return pick, data, offs


def corpus_shard(total_bytes: int, rank: int, world: int, seed: int = 0):
    """Rank `rank`'s contiguous, byte-balanced document range of
    corpus_docs(total_bytes, seed) (the same split as multigpu.shard_batch),
    generated without the other ranks' documents.  Returns (data, offsets
    from 0, (d0, d1), total documents)."""
    pool, sizes, starts, offs = _corpus_layout(total_bytes, seed, 1024, 65536, 64 << 20)
    n_docs = len(sizes)
    bounds = [0]
    for r in range(1, world):
        d = int(np.searchsorted(offs[:n_docs], int(offs[-1]) * r // world, side="left"))
        bounds.append(max(bounds[-1], min(d, n_docs)))
    bounds.append(n_docs)
    d0, d1 = bounds[rank], bounds[rank + 1]
    data, o = _fill(pool, sizes, starts, np.arange(d0, d1))
    return data, o, (d0, d1), n_docs
