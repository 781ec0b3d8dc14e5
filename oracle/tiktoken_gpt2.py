"""tiktoken's GPT-2 encoding, built offline -- TEST INFRASTRUCTURE ONLY (the
oracle of the optional GPT-2 regex pre-tokenization mode).

tiktoken 0.12 cannot download its "gpt2" files here, so the Encoding is built
from the same GPT-2 vocab.json the reference loads: mergeable ranks = token
bytes -> id (GPT-2 merged tokens have id 256 + merge rank) and tiktoken's GPT-2
pattern.  Only tests/ import this module.
"""

from __future__ import annotations

import json

GPT2_PAT = r"""'(?:[sdmt]|ll|ve|re)| ?\p{L}+| ?\p{N}+| ?[^\s\p{L}\p{N}]+|\s+(?!\S)|\s+"""


def build(vocab_path):
    import tiktoken

    from .oracle import byte_symbols

    inv = {c: i for i, c in enumerate(byte_symbols())}
    vocab = json.loads(open(vocab_path, encoding="utf-8").read())
    ranks = {}
    for sym, tid in vocab.items():
        try:
            ranks[bytes(inv[c] for c in sym)] = tid
        except KeyError:
            pass  # symbols with non-byte characters (none in GPT-2 besides specials)
    special = {"<|endoftext|>": 50256}
    ranks = {k: v for k, v in ranks.items() if v != 50256}
    return tiktoken.Encoding(name="gpt2_offline", pat_str=GPT2_PAT, mergeable_ranks=ranks,
                             special_tokens=special)
