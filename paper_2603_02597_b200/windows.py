"""Benchmark windows: the paper's methodology of
fixed-length windows, in byte space or in token space.

Mirrors /root/reference/pkg/src/lanebpe/bench.py:20-47 (`SweepSpec`) and
:83-126 (`make_windows`): the same `random.Random(seed)` draw order, so the
same windows come out for the same inputs.  Token-space windows are slices of
a golden token stream decoded back to bytes; here all slices of one call are
decoded together by the device decode (`Tokenizer.decode_batch`, decode.cu)
instead of one host `decode_tokens` per window.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .errors import CorpusTooSmall

DEFAULT_LENGTHS = (256, 1024, 4096, 16384, 131072)


@dataclass(frozen=True)
class SweepSpec:
    """Shape of a benchmark sweep (bench.py:23-47): ascending positive lengths,
    samples per length, warm-up and measured runs."""

    lengths: tuple[int, ...] = DEFAULT_LENGTHS
    samples_per_length: int = 3
    warmup_runs: int = 3
    measured_runs: int = 10

    def __post_init__(self):
        if not self.lengths:
            raise ValueError("lengths must be nonempty")
        if any(n < 1 for n in self.lengths):
            raise ValueError(f"lengths must be positive, got {self.lengths}")
        if list(self.lengths) != sorted(self.lengths):
            raise ValueError(f"lengths must be ascending, got {self.lengths}")
        for name in ("samples_per_length", "warmup_runs", "measured_runs"):
            if getattr(self, name) < (0 if name == "warmup_runs" else 1):
                raise ValueError(f"{name} must be positive, got {getattr(self, name)}")


def make_windows(corpus: bytes, golden_tokens, spec: SweepSpec, tokenizer=None,
                 seed: int = 0) -> dict[int, list[bytes]]:
    """Deterministic fixed-length windows per sweep length (bench.py:83-126).

    Without golden_tokens: byte slices of the corpus.  With golden_tokens
    (requires the tokenizer): slices of the token stream decoded back to
    bytes, so window boundaries land on token boundaries.
    """
    if not corpus:
        raise CorpusTooSmall("corpus is empty")
    if golden_tokens is not None and tokenizer is None:
        raise ValueError("token-space windows require a tokenizer for decoding")
    rng = random.Random(seed)
    windows: dict[int, list[bytes]] = {}
    if golden_tokens is not None:
        slices, keys = [], []
        for length in spec.lengths:
            if len(golden_tokens) < length:
                raise CorpusTooSmall(f"golden stream has {len(golden_tokens)} tokens, window needs {length}")
            for _ in range(spec.samples_per_length):
                off = rng.randrange(len(golden_tokens) - length + 1)
                slices.append(golden_tokens[off:off + length])
                keys.append(length)
        decoded = tokenizer.decode_batch(slices)  # one device call for every window
        for length, w in zip(keys, decoded):
            windows.setdefault(length, []).append(w)
        return windows
    for length in spec.lengths:
        if len(corpus) < length:
            raise CorpusTooSmall(f"corpus has {len(corpus)} bytes, window needs {length}")
        windows[length] = [corpus[off:off + length]
                           for off in (rng.randrange(len(corpus) - length + 1)
                                       for _ in range(spec.samples_per_length))]
    return windows
