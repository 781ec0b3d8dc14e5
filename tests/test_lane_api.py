"""The reference's lane-engine surface on the device (engines.py:68-266,
merge_table.py:119-243): eval_pairs, compact_scan / compact_double_buffer,
ProbeScratch + lookup_keys_into, traces for tables that are not well-formed,
inject_compaction_fault, and the per-chunk engine seam of tokenize_batch.
Oracles: the naive greedy loop, plain slicing, the scalar host probe, the C
oracle's sequential_bpe trace (oracle/, pinned to the reference)."""

from __future__ import annotations

import random

import numpy as np
import pytest

import paper_2603_02597_b200 as bpe
from paper_2603_02597_b200 import chunker, errors

pytestmark = pytest.mark.gpu


def _tiny():
    symbols = {"a": 5, "b": 9, "c": 13, "d": 21, "e": 34, "f": 55,
               "ab": 100, "abc": 101, "cd": 103, "ef": 105, "bc": 107}
    rules = bpe.parse_merges("a b\nab c\nc d\ne f\nb c\n", bpe.Vocab(symbols))
    return symbols, rules, bpe.build_table(rules)


def _naive_eval(ids, pair_map):
    best = None
    for i in range(len(ids) - 1):
        hit = pair_map.get((int(ids[i]), int(ids[i + 1])))
        if hit is not None and (best is None or hit[0] < best[1]):
            best = (i, hit[0], hit[1])
    return best


def _random_table(rng, well_formed: bool, base: int = 0, n_alpha: int = 6, max_rules: int = 40, id_step: int = 1):
    """Random merge rules over a small alphabet (new ids usable by later rules);
    shuffled ranks when not well-formed.  Returns (rules, alphabet ids)."""
    alpha = [base + id_step * k for k in range(n_alpha)]
    toks = list(alpha)
    rules, seen = [], set()
    for _ in range(rng.randrange(5, max_rules)):
        a, b = rng.choice(toks), rng.choice(toks)
        if (a, b) in seen:
            continue
        seen.add((a, b))
        new = base + id_step * (1000 + len(rules))
        rules.append(bpe.MergeRule(a, b, len(rules), new))
        toks.append(new)
    if not well_formed:
        ranks = list(range(len(rules)))
        rng.shuffle(ranks)
        rules = sorted((bpe.MergeRule(r.left, r.right, ranks[i], r.new_token) for i, r in enumerate(rules)),
                       key=lambda r: r.rank)
    return rules, alpha


def test_eval_pairs_matches_naive(tokenizer):
    symbols, rules, table = _tiny()
    pm = {(r.left, r.right): (r.rank, r.new_token) for r in rules}
    rng = random.Random(3)
    for _ in range(60):
        ids = np.array([symbols[c] for c in "".join(rng.choice("abcdef") for _ in range(rng.randrange(0, 50)))],
                       np.uint32)
        cand = bpe.eval_pairs(ids, table)
        want = _naive_eval(ids, pm)
        assert (None if cand is None else (cand.pos, cand.rank, cand.new_token)) == want
    # ids the table never mentions (above and between its ids) are inert
    ids = np.array([5, 9, 7, 5, 9, 2**32 - 1, 13, 21], np.uint32)
    cand = bpe.eval_pairs(ids, table)
    assert (cand.pos, cand.rank, cand.new_token) == (0, 0, 100)
    c = bpe.PassCounters()
    bpe.eval_pairs(np.array([5, 9, 13], np.uint32), table, counters=c)
    assert c.lookups == 2
    gp = {(int(a), int(b)): (int(k), int(n)) for a, b, k, n in zip(*tokenizer.rule_arrays())}
    for doc in (b"the quick brown fox", b" between", b"\xff\x00 x"):
        ids = tokenizer.encode(doc)
        cand = bpe.eval_pairs(ids, tokenizer.table)
        assert (cand.pos, cand.rank, cand.new_token) == _naive_eval(ids, gp)


def test_compactions_match_slicing():
    rng = np.random.default_rng(4)
    for n in [2, 3, 5, 31, 32, 33, 1023, 1024, 1025, 5000]:
        for _ in range(3):
            toks = rng.integers(0, 2**32, size=n, dtype=np.uint32)
            pos = int(rng.integers(0, n - 1))
            new = int(rng.integers(0, 2**32))
            want = toks.tolist()
            want[pos:pos + 2] = [new]
            for fn in (bpe.compact_scan, bpe.compact_double_buffer):
                assert fn(toks, pos, new).tolist() == want
                out = np.zeros(n + 3, np.uint32)
                res = fn(toks, pos, new, out=out)
                assert res.tolist() == want and out[: n - 1].tolist() == want
    for fn in (bpe.compact_scan, bpe.compact_double_buffer):
        for pos in (-1, 2, 3):
            with pytest.raises(errors.OutOfRange):
                fn(np.array([1, 2, 3], np.uint32), pos, 9)


def test_lookup_keys_into_matches_scalar_probe(tokenizer):
    table = tokenizer.table
    left, right, rank, new = tokenizer.rule_arrays()
    rng = np.random.default_rng(5)
    absent_l = rng.integers(0, 60000, 20000).astype(np.uint64)
    absent_r = rng.integers(0, 60000, 20000).astype(np.uint64)
    keys = np.concatenate([(left.astype(np.uint64) << np.uint64(32)) | right.astype(np.uint64),
                           (absent_l << np.uint64(32)) | absent_r,
                           np.array([2**64 - 1, 0, (2**32 - 1) << 32], np.uint64)])
    scratch = bpe.ProbeScratch(len(keys) + 10)
    hit, vals = table.lookup_keys_into(keys, scratch)
    assert hit.base is scratch.hit or hit is scratch.hit[: len(keys)] or np.shares_memory(hit, scratch.hit)
    for i in range(0, len(keys), 7):
        k = int(keys[i])
        want = table.lookup(k >> 32, k & 0xFFFFFFFF) if k != 2**64 - 1 else None
        assert bool(hit[i]) == (want is not None)
        if want is not None:
            assert bpe.unpack_value(int(vals[i])) == want
    assert hit[: len(left)].all()
    assert np.array_equal(vals[: len(left)] & np.uint64(0xFFFFFFFF), rank.astype(np.uint64))
    assert not hit[-3]
    found, nw, rk = table.lookup_pairs(left[:500], right[:500])
    assert found.all() and np.array_equal(rk, rank[:500]) and np.array_equal(nw, new[:500])


def test_wide_id_tables():
    """Ids anywhere in [0, 2^32) (the reference accepts any 32-bit id):
    densely renumbered for the device context and mapped back."""
    rng = random.Random(6)
    for trial in range(20):
        rules, alpha = _random_table(rng, trial % 2 == 0, base=2**31 + 17, id_step=65537)
        table = bpe.build_table(rules)
        pm = {(r.left, r.right): (r.rank, r.new_token) for r in rules}
        from oracle.oracle import greedy_merge

        for _ in range(20):
            ids = [rng.choice(alpha + [3, 2**32 - 2]) for _ in range(rng.randrange(0, 40))]
            out, c = bpe.sequential_bpe(ids, table)
            assert out.tolist() == greedy_merge(ids, pm)
            cand = bpe.eval_pairs(np.array(ids, np.uint32), table)
            assert (None if cand is None else (cand.pos, cand.rank, cand.new_token)) == _naive_eval(ids, pm)
        r0 = rules[0]
        hit, vals = table.lookup_keys_into(np.array([bpe.pack_key(r0.left, r0.right), 5], np.uint64),
                                           bpe.ProbeScratch(2))
        assert hit.tolist() == [True, False] and bpe.unpack_value(int(vals[0])) == (r0.new_token, r0.rank)


@pytest.mark.parametrize("well_formed", [True, False])
def test_traces_and_lookups_match_the_oracle(well_formed):
    """Merge-rank traces on any table (the device records them; strict passes
    when not well-formed) against the C oracle's sequential_bpe trace, and the
    lookup counter against the reference's formula through the oracle trace."""
    from oracle.oracle import OracleEncoder, greedy_merge

    rng = random.Random(40 + well_formed)
    for trial in range(12):
        rules, alpha = _random_table(rng, well_formed)
        table = bpe.build_table(rules)
        left, right, rank, new = bpe.rule_arrays(table)
        orc = OracleEncoder(np.zeros(256, np.uint32), left, right, rank, new)
        pm = {(r.left, r.right): (r.rank, r.new_token) for r in rules}
        for _ in range(25):
            ids = [rng.choice(alpha) for _ in range(rng.randrange(0, 60))]
            tr = []
            out, c = bpe.sequential_bpe(ids, table, trace=tr)
            w_out, w_tr = orc.sequential_bpe(np.array(ids, np.uint32), with_trace=True)
            assert out.tolist() == w_out.tolist() == greedy_merge(ids, pm)
            assert tr == w_tr.tolist(), (trial, ids)
            tr2 = []
            out2, c2 = bpe.run_block_engine(ids, table, trace=tr2)
            assert out2.tolist() == w_out.tolist() and tr2 == w_tr.tolist()


def test_sequential_lookup_counter_matches_reference_formula():
    """lookups = (n - 1) + one per neighbour of every merge (engines.py:296-330)."""
    symbols, rules, table = _tiny()
    pm = {(r.left, r.right): (r.rank, r.new_token) for r in rules}
    rng = random.Random(8)
    for _ in range(100):
        ids = [symbols[c] for c in "".join(rng.choice("abcdef") for _ in range(rng.randrange(0, 30)))]
        # naive count: simulate the reference's heap loop's probes
        cur, probes = list(ids), max(len(ids) - 1, 0)
        while len(cur) >= 2:
            best = _naive_eval(cur, pm)
            if best is None:
                break
            p = best[0]
            cur[p:p + 2] = [best[2]]
            probes += (p > 0) + (p + 1 < len(cur))
        out, c = bpe.sequential_bpe(ids, table)
        assert out.tolist() == cur and c.lookups == probes


def test_compaction_fault_is_caught_by_the_parity_harness(tokenizer, oracle):
    """inject_compaction_fault corrupts one pass inside the device engine; the
    oracle comparison the parity tests use must catch it, and the flag is
    one-shot (engines.py:252-266, test_engines.py:318-326)."""
    ids = tokenizer.encode(b"the quick brown fox jumps over the lazy dog")
    want = oracle.sequential_bpe(ids)
    clean, _ = bpe.run_block_engine(ids, tokenizer.table, tokenizer.config)
    assert np.array_equal(clean, want)
    with bpe.inject_compaction_fault():
        faulty, _ = bpe.run_block_engine(ids, tokenizer.table, tokenizer.config)
    assert not np.array_equal(faulty, want)
    again, _ = bpe.run_block_engine(ids, tokenizer.table, tokenizer.config)
    assert np.array_equal(again, want)
    # through the batch API: a lane engine takes the armed fault (per-chunk seam)
    docs = [b"hello world", b"the quick brown fox jumps over the lazy dog"]
    with bpe.inject_compaction_fault():
        res = bpe.tokenize_batch(docs, tokenizer, "optimized", workers=1)
    assert [t.tolist() for t in res.token_ids] != [x.tolist() for x in oracle.encode_docs(docs)]
    res = bpe.tokenize_batch(docs, tokenizer, "optimized", workers=1)
    assert [t.tolist() for t in res.token_ids] == [x.tolist() for x in oracle.encode_docs(docs)]
    # many sequences: exactly one of them diverges
    rng = random.Random(9)
    prose = b" ".join(__import__("fixtures").prose_samples()[:5])
    bad = 0
    for k in range(30):
        at = rng.randrange(0, len(prose) - 300)
        ids = tokenizer.encode(prose[at:at + rng.randrange(20, 300)])
        with bpe.inject_compaction_fault():
            got, _ = bpe.run_block_engine(ids, tokenizer.table, tokenizer.config)
        bad += not np.array_equal(got, oracle.sequential_bpe(ids))
    assert bad >= 25, bad  # a shifted merge almost always changes the ids


def test_per_chunk_engine_seam(tokenizer, monkeypatch):
    """Replacing chunker.run_block_engine (the reference's dispatch point,
    chunker.py:146-155) routes tokenize_batch through it per chunk, with
    BatchError carrying the input index."""
    def boom(tokens, table, config=None, variant="optimized", trace=None):
        raise errors.SequenceTooLong("forced failure")

    monkeypatch.setattr(chunker, "run_block_engine", boom)
    with pytest.raises(errors.BatchError) as err:
        bpe.tokenize_batch([b"ok", b"bad"], tokenizer, workers=1)
    assert err.value.input_index == 0
    monkeypatch.undo()
    calls = []
    real = chunker.run_block_engine

    def spy(tokens, table, config=None, variant="optimized", trace=None):
        calls.append(len(tokens))
        return real(tokens, table, config, variant, trace)

    monkeypatch.setattr(chunker, "run_block_engine", spy)
    cfg = bpe.BlockConfig(max_seq_len=64, chunk_budget=16)
    tok = bpe.Tokenizer(tokenizer.vocab, tokenizer.table, cfg)
    res = bpe.tokenize_batch([b"x" * 65, b"hello"], tok, workers=1)
    assert calls == [16, 16, 16, 16, 1, 5]
    monkeypatch.undo()
    assert [t.tolist() for t in bpe.tokenize_batch([b"x" * 65, b"hello"], tok).token_ids] == \
        [t.tolist() for t in res.token_ids]
    assert res.counters.buffer_allocations == 2 * 5  # the 1-id chunk takes no buffers


def test_batch_counters_follow_the_lane_model(tokenizer, prose_samples):
    docs = prose_samples[:3] + [b"", b"x"]
    res = bpe.tokenize_batch(docs, tokenizer, workers=1)
    assert sum(len(d) for d in docs) - res.counters.passes == sum(len(t) for t in res.token_ids)
    assert res.counters.buffer_allocations == 2 * 3
    assert bpe.tokenize_batch(docs, tokenizer, "sequential").counters.buffer_allocations == 0


def test_batch_counters_equal_per_chunk_engine_runs(tokenizer, prose_samples):
    """tokenize_batch's counters (all engine names) equal the sum of the
    token-level engines' counters over the reference's chunks
    (chunker.py:166-172), with documents longer than max_seq_len."""
    cfg = bpe.BlockConfig(max_seq_len=700, chunk_budget=300)
    tok = bpe.Tokenizer(tokenizer.vocab, tokenizer.table, cfg)
    tok._devices = tokenizer._devices
    docs = prose_samples[:6] + [b"", b"x", b"ab", prose_samples[7][:700], prose_samples[8][:701]]
    for variant in ("sequential", "baseline", "optimized"):
        want = bpe.PassCounters()
        for d in docs:
            ids = tok.encode(d)
            chunks = bpe.chunk_tokens(ids, 300) if len(ids) > 700 else [bpe.Chunk(0, 0, ids)]
            for c in chunks:
                fn = bpe.sequential_bpe if variant == "sequential" else bpe.run_block_engine
                _, cc = fn(c.tokens, tok.table) if variant == "sequential" else fn(c.tokens, tok.table, cfg, variant)
                want.merge_from(cc)
        got = bpe.tokenize_batch(docs, tok, variant).counters
        assert (got.passes, got.lookups, got.compaction_moves, got.buffer_allocations) == \
            (want.passes, want.lookups, want.compaction_moves, want.buffer_allocations), variant
        one = bpe.tokenize_batch([docs[0]], tok, variant).counters  # the one-document path
        assert one.passes > 0 and one.lookups > 0


def test_multi_device_batches_match_single_device(tokenizer, oracle, prose_samples):
    """tokenize_batch(devices=...) shards units across GPUs from one process:
    documents (P-default chunks included) by bytes, a lone huge document at
    exact junction cuts.  On a one-GPU box, devices=[0, 0] runs the same
    sharding, threads and reassembly against one context."""
    import synth_corpus

    docs = prose_samples[:40] + [b"", b"x" * 9000, synth_corpus.english_bytes(3 << 20, 4)]
    want = oracle.encode_docs(docs, 8192, 8192, 8)
    for devs in ([0, 0], [0, 0, 0]):
        res = bpe.tokenize_batch(docs, tokenizer, devices=devs)
        assert [t.tolist() for t in res.token_ids] == [w.tolist() for w in want]
        assert res.counters.passes == sum(map(len, docs)) - sum(map(len, want))
    whole = bpe.Tokenizer(tokenizer.vocab, tokenizer.table, bpe.BlockConfig(max_seq_len=1 << 40, chunk_budget=1 << 40))
    whole._devices = tokenizer._devices
    big = synth_corpus.english_bytes(5 << 20, 9)
    w = oracle.encode_docs([big], 1 << 40, 1 << 40, 1)[0]
    for devs in ([0, 0], 4):
        got = bpe.tokenize_batch([big], whole, devices=[0] * devs if isinstance(devs, int) else devs).token_ids[0]
        assert np.array_equal(got, w)
    h = bpe.TokenizerHandle.__new__(bpe.TokenizerHandle)
    h._tokenizer, h._engine, h._workers, h._devices = tokenizer, "optimized", None, [0, 0]
    assert h.tokenize_batch(["hello world", b""])[0] == [[31373, 995], []]
