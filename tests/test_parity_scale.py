"""Parity at scale: every BASELINE config that
had only an id count checked, and the exactness fuzz of the multi-merge rule
on random merge tables at >= 10,000 cases per level.

* C2: 4,096 prompts x ~2.3 KB (P-default), every document against the oracle;
* corpus_256m: the whole 256 MiB corpus (17,195 documents, P-default);
* C4: a seeded 1% document sample of the 10 GiB corpus, byte-identical to
  the documents the bench encodes, plus an id-array checksum;
* token level: 2 x 400 random tables (well-formed: exact multi-merge passes;
  shuffled ranks: strict passes) x 25 sequences = 20,000 cases, through
  gpubpe_merge_tokens with many sequences per launch (the tables live side
  by side in one context on disjoint id ranges, so no sequence can see
  another table's rules);
* byte level: 2 x 100 random byte-level tables x 60 documents = 12,000 cases (k_encode: the
  junction cuts, the verified memo, warp / CTA / grid engines; runs up to
  20 KB so giants > 4 KiB occur under tables that are not well-formed).
The oracle is oracle/ (the C restatement pinned to the reference's goldens).
"""

from __future__ import annotations

import hashlib
import os
import random

import numpy as np
import pytest

import paper_2603_02597_b200 as bpe
from oracle.oracle import OracleEncoder, default_threads, greedy_merge

pytestmark = pytest.mark.gpu


def _csr(ids, offs):
    o = np.asarray(offs).tolist()
    return [ids[a:b] for a, b in zip(o, o[1:])]


def _first_diff(got, want):
    for i, (g, w) in enumerate(zip(got, want)):
        if not np.array_equal(g, w):
            return i
    return None


def test_c2_4096_prompts_match_oracle(tokenizer, oracle):
    import synth_corpus

    n_docs, doc_bytes = 4096, 2300  # tools/perf.py c2_4096x512 (~512 tokens each)
    pool = np.frombuffer(synth_corpus.english_bytes(n_docs * doc_bytes + (1 << 20), 5), np.uint8)
    data = pool[: n_docs * doc_bytes].copy()
    offs = np.arange(n_docs + 1, dtype=np.int64) * doc_bytes
    docs = [data[offs[i]:offs[i + 1]].tobytes() for i in range(n_docs)]
    got = bpe.tokenize_batch(docs, tokenizer).token_ids
    w_ids, w_offs, _ = oracle.encode_packed(data, offs, 8192, 8192, default_threads())
    want = _csr(w_ids, w_offs)
    assert _first_diff(got, want) is None
    assert sum(len(g) for g in got) == len(w_ids) > 4096 * 400


def test_corpus_256m_every_document_matches_oracle(tokenizer, oracle):
    import synth_corpus

    data, offs = synth_corpus.corpus_docs(256 << 20, seed=0)
    enc = tokenizer.device_encoder()
    ids, oo, st, _ = enc.encode_packed_host(data, offs, 8192, 8192)
    w_ids, w_offs, w_passes = oracle.encode_packed(data, offs, 8192, 8192, default_threads())
    assert np.array_equal(oo, w_offs)
    assert np.array_equal(ids, w_ids)
    assert st["passes"] == w_passes == len(data) - len(w_ids)


def test_c4_one_percent_sample_matches_oracle(tokenizer, oracle):
    import synth_corpus

    pick, data, offs = synth_corpus.corpus_sample(10240 << 20, 0.01, sample_seed=2024)
    assert len(pick) > 6000  # ~1% of 692,805 documents
    enc = tokenizer.device_encoder()
    ids, oo, _, _ = enc.encode_packed_host(data, offs, 8192, 8192)
    w_ids, w_offs, _ = oracle.encode_packed(data, offs, 8192, 8192, default_threads())
    assert np.array_equal(oo, w_offs) and np.array_equal(ids, w_ids)
    digest = hashlib.sha256(ids.astype("<u4").tobytes()).hexdigest()
    assert digest == hashlib.sha256(w_ids.astype("<u4").tobytes()).hexdigest()


def _random_rules(rng, well_formed, base, rank_base, n_alpha):
    alpha = [base + k for k in range(n_alpha)]
    toks = list(alpha)
    rules, seen = [], set()
    for _ in range(rng.randrange(5, 48)):
        a, b = rng.choice(toks), rng.choice(toks)
        if (a, b) in seen:
            continue
        seen.add((a, b))
        rules.append([a, b, len(rules), base + 64 + len(rules)])
        toks.append(rules[-1][3])
    if not well_formed:
        ranks = list(range(len(rules)))
        rng.shuffle(ranks)
        for r, k in zip(rules, ranks):
            r[2] = k
    for r in rules:
        r[2] += rank_base
    return rules, alpha


@pytest.mark.parametrize("well_formed", [True, False])
def test_token_level_fuzz_20k(well_formed):
    """400 random tables x 25 sequences of <= 60 ids per mode (SURVEY A.3's
    fuzz), one device launch per mode; every sequence against the C oracle,
    every 10th against the naive greedy too."""
    import torch

    from paper_2603_02597_b200 import _native
    from paper_2603_02597_b200.device import DeviceEncoder

    rng = random.Random(1000 + well_formed)
    n_tables, per_table = 400, 25
    all_rules, seqs, owner = [], [], []
    tables = []
    for t in range(n_tables):
        rules, alpha = _random_rules(rng, well_formed, base=t * 128, rank_base=t * 64, n_alpha=rng.randrange(2, 7))
        all_rules += rules
        tables.append(rules)
        for _ in range(per_table):
            seqs.append([rng.choice(alpha) for _ in range(rng.randrange(0, 61))])
            owner.append(t)
    R = np.array(sorted(all_rules, key=lambda r: r[2]), dtype=np.uint32)
    L, Rt, K, N = R[:, 0].copy(), R[:, 1].copy(), R[:, 2].copy(), R[:, 3].copy()
    enc = DeviceEncoder(np.zeros(256, np.uint32), L, Rt, K, N, memo=False)
    assert bool(enc.query()["well_formed"]) == well_formed
    orc = OracleEncoder(np.zeros(256, np.uint32), L, Rt, K, N)
    offs = np.zeros(len(seqs) + 1, np.uint64)
    np.cumsum([len(s) for s in seqs], out=offs[1:].view(np.int64))
    flat = np.array([x for s in seqs for x in s], np.uint32)
    d_in = torch.from_numpy(flat.view(np.int32)).cuda()
    d_out = torch.empty_like(d_in)
    counts = np.zeros(len(seqs), np.uint64)
    rc = enc._lib.gpubpe_merge_tokens(enc._h, d_in.data_ptr(), offs.ctypes.data, len(seqs), d_out.data_ptr(),
                                      counts.ctypes.data, torch.cuda.current_stream().cuda_stream)
    _native.check(rc, enc._h, "gpubpe_merge_tokens")
    out = d_out.cpu().numpy().view(np.uint32)
    bad = []
    for i, s in enumerate(seqs):
        got = out[int(offs[i]): int(offs[i]) + int(counts[i])]
        want = orc.sequential_bpe(np.array(s, np.uint32))
        if not np.array_equal(got, want):
            bad.append(i)
        elif i % 10 == 0:
            pm = {(a, b): (k, n) for a, b, k, n in tables[owner[i]]}
            assert want.tolist() == greedy_merge(s, pm)
    assert not bad, f"{len(bad)} of {len(seqs)} sequences differ, first {bad[:5]}"
    assert len(seqs) == 10_000


@pytest.mark.parametrize("well_formed", [True, False])
def test_byte_level_fuzz(well_formed):
    """100 random byte-level tables x 60 documents per mode through
    tokenize_batch (k_encode), P-whole, including 4-20 KB runs (deferred
    and giant segments)."""
    # GPUBPE_FUZZ_TABLES / GPUBPE_FUZZ_SEED widen the run by hand (longer GPU soaks)
    n_tables = int(os.environ.get("GPUBPE_FUZZ_TABLES", "100"))
    rng = random.Random(2000 + well_formed + 7919 * int(os.environ.get("GPUBPE_FUZZ_SEED", "0")))
    enc = bpe.build_byte_encoder()
    b2s = {b: s for s, b in enc.symbol_to_byte.items()}
    total, giants = 0, 0
    for t in range(n_tables):
        symbols = {b2s[b]: b for b in range(256)}
        sym_of = {b: b2s[b] for b in range(256)}
        alphabet = bytes(rng.sample(range(256), rng.randrange(2, 7)))
        ids = list(alphabet)
        rules = []
        for _ in range(rng.randrange(10, 120)):
            a, b = rng.choice(ids), rng.choice(ids)
            s = sym_of[a] + sym_of[b]
            if s in symbols or len(s) > 48:
                continue
            symbols[s] = 256 + len(rules)
            sym_of[256 + len(rules)] = s
            rules.append(bpe.MergeRule(a, b, len(rules), 256 + len(rules)))
            ids.append(256 + len(rules) - 1)
        if not well_formed:
            ranks = list(range(len(rules)))
            rng.shuffle(ranks)
            rules = sorted((bpe.MergeRule(r.left, r.right, ranks[i], r.new_token) for i, r in enumerate(rules)),
                           key=lambda r: r.rank)
        tok = bpe.Tokenizer(bpe.Vocab(symbols), bpe.build_table(rules),
                            bpe.BlockConfig(max_seq_len=1 << 40, chunk_budget=1 << 40))
        left, right, rank, new = tok.rule_arrays()
        orc = OracleEncoder(tok._base_ids, left, right, rank, new)
        docs = []
        for _ in range(60):
            n = int(np.exp(rng.uniform(0, np.log(20000))))
            docs.append(bytes(rng.choice(alphabet) for _ in range(n)) if n < 2000 else
                        bytes(rng.choices(alphabet[:2], k=n)))
        giants += sum(len(d) > 4096 for d in docs)
        got = bpe.tokenize_batch(docs, tok).token_ids
        want = orc.encode_docs(docs, 1 << 40, 1 << 40)
        i = _first_diff(got, want)
        assert i is None, f"table {t}: doc {i} (len {len(docs[i])}) differs"
        total += len(docs)
        for d in tok._devices.values():
            d.close()
    assert total == 60 * n_tables and giants > n_tables
