"""Code point classes for the optional GPT-2 regex pre-tokenization mode
(pretok.cu).

tiktoken's GPT-2 pattern distinguishes \\p{L}, \\p{N}, \\s and everything else;
the device pass needs those four classes for every code point.  They are
taken from the `regex` module (the same Unicode property tables the pattern
uses in Python) once per process: 2 bits per code point, four per byte
(272 KiB for the 1,114,112 code points).
"""

from __future__ import annotations

import functools

import numpy as np

N_CPS = 0x110000
CLS_O, CLS_L, CLS_N, CLS_S = 0, 1, 2, 3


@functools.lru_cache(maxsize=1)
def gpt2_classes() -> np.ndarray:
    """uint8[N_CPS / 4]: packed 2-bit classes (0 other, 1 letter, 2 number, 3 \\s)."""
    try:
        import regex
    except ImportError as exc:  # pragma: no cover - regex is part of the image
        raise RuntimeError("GPT-2 regex mode needs the `regex` module") from exc
    cls = np.zeros(N_CPS, dtype=np.uint8)
    # all code points except surrogates, as one string; runs found with the
    # pattern's own property classes
    cps = np.concatenate([np.arange(0, 0xD800), np.arange(0xE000, N_CPS)])
    text = "".join(map(chr, cps.tolist()))
    idx = np.array(cps, dtype=np.int64)
    for c, pat in ((CLS_L, r"\p{L}+"), (CLS_N, r"\p{N}+"), (CLS_S, r"\s+")):
        for m in regex.finditer(pat, text):
            cls[idx[m.start():m.end()]] = c
    packed = cls.reshape(-1, 4)
    return (packed[:, 0] | (packed[:, 1] << 2) | (packed[:, 2] << 4) | (packed[:, 3] << 6)).astype(np.uint8)
