"""GPT-2 regex pre-tokenization mode on CPU: the code point
class table, and the local token-start rules pretok.cu applies, restated in
Python and checked against the pattern itself (the `regex` module)."""

import random

import numpy as np
import regex

from oracle.tiktoken_gpt2 import GPT2_PAT
from paper_2603_02597_b200 import pretok

O, L, N, S = 0, 1, 2, 3


def _cls_of(cp: int) -> int:
    t = pretok.gpt2_classes()
    return int((t[cp >> 2] >> (2 * (cp & 3))) & 3)


def test_class_table():
    assert pretok.gpt2_classes().shape == (pretok.N_CPS // 4,)
    for c in " \t\n\r  　":
        assert _cls_of(ord(c)) == S, repr(c)
    for c in "aZéßΩж日本ア":
        assert _cls_of(ord(c)) == L, c
    for c in "09²½Ⅻ٣":
        assert _cls_of(ord(c)) == N, c
    for c in "'.,?!_-—😀\x1c":
        assert _cls_of(ord(c)) == O, repr(c)


def starts(text: str) -> list[str]:
    """pretok.cu's rules (module docstring there), on code points."""
    cps = list(text)
    n = len(cps)
    C = [_cls_of(ord(c)) for c in cps]

    def ch(k):
        return cps[k] if 0 <= k < n else ""

    def tstart(j):
        return j == 0 or C[j - 1] in (L, N) or (C[j - 1] == S and cps[j - 1] != " ")

    def clen(j):
        if not (0 <= j < n) or cps[j] != "'" or not tstart(j):
            return 0
        a, b = ch(j + 1), ch(j + 2)
        if a in ("s", "d", "m", "t"):
            return 2
        return 3 if (a, b) in (("l", "l"), ("v", "e"), ("r", "e")) else 0

    out, cur = [], ""
    for k in range(n):
        if k == 0:
            b = True
        elif C[k] == S:
            b = C[k - 1] != S or (k + 1 < n and C[k + 1] != S)
        elif C[k - 1] == S:
            b = cps[k - 1] != " "
        elif clen(k - 1) or clen(k - 2) == 3:
            b = False
        elif clen(k - 2) == 2 or clen(k - 3) == 3:
            b = True
        else:
            b = C[k] != C[k - 1]
        if b and cur:
            out.append(cur)
            cur = ""
        cur += cps[k]
    if cur:
        out.append(cur)
    return out


def test_rules_match_the_pattern():
    cases = ["hello world", "it's", "it'sa", "IT'S", "x'll y've z're 'd 'm 't", "  x", "\n\nhello", "x  ",
             " 's", "\n's", "?'s", "''s", "a1b2", "hello   world  \n\n  x", "don't stop'n'roll", "½ ², ³x",
             "日本語 テキスト", "x\t\ty", " ' ", "'", "e.g. U.S.A.", "3.14159", "\r\n\r\nfoo", "x \n y"]
    for t in cases:
        assert starts(t) == regex.findall(GPT2_PAT, t), repr(t)
    rng = random.Random(7)
    alphabet = list("ab's dmtlvre'  \n\t1.?!,") + ["é", " ", "　", "½", "日", "😀"]
    for _ in range(5000):
        t = "".join(rng.choice(alphabet) for _ in range(rng.randint(1, 14)))
        assert starts(t) == regex.findall(GPT2_PAT, t), repr(t)
