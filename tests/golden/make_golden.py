#!/usr/bin/env python3
"""Generate the committed parity fixtures by running the REFERENCE itself.

Runs only in the build container, where the reference is mounted read-only at
/root/reference (pure Python package `lanebpe`).  Nothing at test/bench time
reads /root/reference; everything needed is written next to this script:

  gpt2/vocab.json.gz, gpt2/merges.txt.gz   the GPT-2 tables the reference loads
                                           (pkg/tests/data/gpt2, md5 checked)
  prose_corpus.txt.gz + golden_prose.npz   the reference's 100 prose samples and
                                           its 100 golden id files
                                           (pkg/tests/data/{prose_corpus.txt,golden/})
  batch_fixture.txt.gz + batch_fixture_ids.npz
                                           the bindings' 50-doc fixture and the ids
                                           lanebpe.tokenize_batch returns for it
  mixed_cases.npz                          mixed_blob inputs (pkg/tests/reference.py
                                           kinds 0-3), regression strings and
                                           adversarial runs, each with the
                                           reference's ids under several BlockConfigs
  known_answers.json                       small hand-checkable ids
  synth_sizes.json                         calibrated synthetic workload lengths and
                                           the reference's sha256 of the ids

Usage:  python tests/golden/make_golden.py [--skip-large]
"""

from __future__ import annotations

import argparse
import gzip
import hashlib
import json
import random
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tools"))

import lanebpe  # noqa: E402  (the reference)
from reference import mixed_blob  # noqa: E402  (reference test helper)

VOCAB = REF / "tests/data/gpt2/vocab.json"
MERGES = REF / "tests/data/gpt2/merges.txt"
MD5 = {"vocab.json": "dffec25a898b1f5e569bec4dffd7e5c0", "merges.txt": "75a37753dd7a28a2c5df80c28bf06e4e"}

# BlockConfigs the fixtures are produced under: (name, max_seq_len, chunk_budget)
CONFIGS = [
    ("default", 8192, 8192),
    ("s64_b32", 64, 32),
    ("s256_b256", 256, 256),
    ("s512_b100", 512, 100),
    ("whole", 1 << 40, 1 << 40),
]


def gz_write(path: Path, data: bytes) -> None:
    path.write_bytes(gzip.compress(data, 9, mtime=0))


def sha_ids(ids) -> str:
    return hashlib.sha256(np.asarray(ids, dtype="<u4").tobytes()).hexdigest()


def ref_tok(max_seq_len: int, chunk_budget: int):
    if max_seq_len >= 1 << 40:
        return None
    cfg = lanebpe.BlockConfig(max_seq_len=max_seq_len, chunk_budget=chunk_budget)
    return lanebpe.Tokenizer.from_files(VOCAB, MERGES, cfg)


def ref_encode(docs, max_seq_len, chunk_budget, base_tok):
    if max_seq_len >= 1 << 40:  # P-whole: the engine on the whole sequence
        return [lanebpe.sequential_bpe(base_tok.encode(d), base_tok.table)[0] for d in docs]
    tok = ref_tok(max_seq_len, chunk_budget)
    return lanebpe.tokenize_batch(docs, tok, "sequential", workers=1).token_ids


def pack(arrs):
    offs = np.zeros(len(arrs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(a) for a in arrs]) if arrs else []
    flat = np.concatenate([np.asarray(a, dtype=np.uint32) for a in arrs]) if arrs else np.empty(0, np.uint32)
    return flat.astype(np.uint32), offs


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-large", action="store_true")
    args = ap.parse_args()

    (HERE / "gpt2").mkdir(exist_ok=True)
    for src in (VOCAB, MERGES):
        raw = src.read_bytes()
        assert hashlib.md5(raw).hexdigest() == MD5[src.name], src
        gz_write(HERE / "gpt2" / (src.name + ".gz"), raw)

    tok = lanebpe.Tokenizer.from_files(VOCAB, MERGES)

    # 1. reference prose corpus + its golden files
    corpus = (REF / "tests/data/prose_corpus.txt").read_bytes()
    gz_write(HERE / "prose_corpus.txt.gz", corpus)
    samples = corpus.rstrip(b"\n").split(b"\n")
    golds = [lanebpe.load_golden_file(REF / f"tests/data/golden/sample_{i:03d}.tokens")
             for i in range(len(samples))]
    ids, offs = pack(golds)
    np.savez_compressed(HERE / "golden_prose.npz", ids=ids, offs=offs)
    print(f"golden prose: {len(samples)} samples, {len(ids)} ids")

    # 2. bindings fixture (50 docs) under the handle's defaults
    fixture = (REF / "bindings/tests/data/batch_fixture.txt").read_bytes()
    gz_write(HERE / "batch_fixture.txt.gz", fixture)
    docs = fixture.rstrip(b"\n").split(b"\n")
    out = lanebpe.tokenize_batch(docs, tok, "sequential", workers=1).token_ids
    ids, offs = pack(out)
    np.savez_compressed(HERE / "batch_fixture_ids.npz", ids=ids, offs=offs)

    # 3. known answers
    ka = {
        "hello world": [int(x) for x in tok.encode(b"hello world")],
    }
    known = {}
    for text in [b"hello world", b" between", b"\n\nhello", b"x\n\n\n\ny", b"the", b"", b"a",
                 b"<|endoftext|>", b"\xff\xfe broken \x80 bytes", "héllo".encode()]:
        known[text.hex()] = [int(x) for x in ref_encode([text], 8192, 8192, tok)[0]]
    ka = {"cases": known, "base_the": [int(x) for x in tok.encode(b"the")]}
    (HERE / "known_answers.json").write_text(json.dumps(ka, indent=1) + "\n")

    # 4. mixed cases: mixed_blob kinds 0-3, regressions, adversarial
    rng = random.Random(20261017)
    inputs: list[bytes] = []
    for i in range(240):
        kind = i % 4
        length = rng.choice([0, 1, 2, 3, 7, 31, 64, 65, 100, 257, 600, 1500, rng.randrange(0, 2500)])
        inputs.append(mixed_blob(rng, kind, length, corpus))
    inputs += [b" between", b"\n\nhello", b"x\n\n\n\ny", b"", b"a", b"ab" * 50]
    inputs += [b"0123456789" * 300, b"\n" * 9000, b"a" * 5000, b" " * 4097,
               bytes(rng.choice(b"abcdefghijklmnopqrstuvwxyz") for _ in range(6000)),
               bytes(rng.choice(b"0123456789") for _ in range(7000)),
               bytes(rng.choice(b"0123456789abcdef") for _ in range(3000)),
               bytes(rng.choice(b"\n \t") for _ in range(2000)),
               bytes(rng.randrange(256) for _ in range(20000))]
    data_flat = np.frombuffer(b"".join(inputs), dtype=np.uint8)
    in_offs = np.zeros(len(inputs) + 1, dtype=np.int64)
    in_offs[1:] = np.cumsum([len(x) for x in inputs])
    save = {"data": data_flat, "offs": in_offs}
    for name, msl, cb in CONFIGS:
        t0 = time.time()
        outs = ref_encode(inputs, msl, cb, tok)
        ids, offs = pack(outs)
        save[f"ids_{name}"] = ids
        save[f"offs_{name}"] = offs
        save[f"cfg_{name}"] = np.array([min(msl, 2**62), min(cb, 2**62)], dtype=np.int64)
        print(f"mixed[{name}]: {len(inputs)} docs, {len(ids)} ids, {time.time() - t0:.1f}s")
    np.savez_compressed(HERE / "mixed_cases.npz", **save)

    # 5. calibrated synthetic workloads (P-whole exact token counts)
    import synth_corpus  # noqa: E402
    from oracle.oracle import OracleEncoder, load_tables  # noqa: E402

    orc = OracleEncoder.from_tables(load_tables(VOCAB, MERGES))

    def count(b: bytes) -> int:
        return len(orc.sequential_bpe(orc.base(b)))

    targets = [("c0_1k", 1024, 0), ("c1_8k", 8192, 1), ("c1_32k", 32768, 2),
               ("c1_131k", 131072, 3), ("c3_1m", 1 << 20, 4)]
    sizes = {}
    for name, ntok, seed in targets:
        big = synth_corpus.english_bytes(int(ntok * 6.5) + 4096, seed)
        lo, hi = 1, len(big)
        while lo < hi:  # smallest prefix with >= ntok tokens
            mid = (lo + hi) // 2
            if count(big[:mid]) >= ntok:
                hi = mid
            else:
                lo = mid + 1
        nb = lo
        while count(big[:nb]) != ntok:
            nb += 1
        doc = big[:nb]
        assert synth_corpus.english_bytes(nb, seed) == doc
        entry = {"seed": seed, "n_bytes": nb, "tokens_whole": ntok}
        if not (args.skip_large and ntok > 200000):
            t0 = time.time()
            whole = lanebpe.sequential_bpe(tok.encode(doc), tok.table)[0]
            t_whole = time.time() - t0
            assert len(whole) == ntok, (name, len(whole))
            t0 = time.time()
            dflt = lanebpe.tokenize_batch([doc], tok, "sequential", workers=1).token_ids[0]
            t_dflt = time.time() - t0
            entry.update(sha_whole=sha_ids(whole), sha_default=sha_ids(dflt),
                         tokens_default=int(len(dflt)), ref_seconds_whole=round(t_whole, 3),
                         ref_seconds_default=round(t_dflt, 3))
        sizes[name] = entry
        print(name, entry)
    (HERE / "synth_sizes.json").write_text(json.dumps(sizes, indent=1) + "\n")


if __name__ == "__main__":
    main()
