"""Host-side mirror of the reference API (construction, validation, errors).

Modelled on the reference's own unit tests (pkg/tests/test_byte_codec.py,
test_merge_table.py, test_chunker.py); expected values are the reference's.
"""

import numpy as np
import pytest

import paper_2603_02597_b200 as bpe
from paper_2603_02597_b200 import errors


def test_byte_encoder_is_a_bijection_with_reference_anchors():
    enc = bpe.build_byte_encoder()
    assert len(set(enc.byte_to_symbol)) == 256
    assert enc.byte_to_symbol[0x20] == "Ġ"
    assert enc.byte_to_symbol[0x7F] == "ġ"
    assert enc.byte_to_symbol[0xAD] == "Ń"
    assert enc.byte_to_symbol[0x00] == "Ā"
    assert all(enc.symbol_to_byte[s] == b for b, s in enumerate(enc.byte_to_symbol))


def test_vocab_validation():
    with pytest.raises(errors.MalformedVocab):
        bpe.Vocab({"a": -1})
    with pytest.raises(errors.MalformedVocab):
        bpe.Vocab({"a": 1, "b": 1})
    with pytest.raises(errors.MalformedVocab):
        bpe.Vocab({"a": True})
    with pytest.raises(errors.MalformedVocab):
        bpe.Vocab({"a": 2**32})


def test_gpt2_tables(tokenizer):
    assert len(tokenizer.vocab) == 50257
    assert tokenizer.table.count == 50000
    assert tokenizer.table.capacity == 131072
    assert tokenizer.encode(b"the").tolist() == [83, 71, 68]
    assert tokenizer.vocab.id_to_symbol[1169] == "the"
    assert bpe.decode_tokens([31373, 995], tokenizer.encoder, tokenizer.vocab) == b"hello world"


def test_table_lookups_and_rule_recovery(tokenizer, oracle_tables):
    t = tokenizer.table
    for i in range(0, 50000, 997):
        l, r = int(oracle_tables.left[i]), int(oracle_tables.right[i])
        assert t.lookup(l, r) == (int(oracle_tables.new[i]), i)
    assert t.lookup(50256, 50256) is None
    left, right, rank, new = bpe.rule_arrays(t)
    assert np.array_equal(left, oracle_tables.left) and np.array_equal(right, oracle_tables.right)
    assert np.array_equal(rank, oracle_tables.rank) and np.array_equal(new, oracle_tables.new)
    hits = [t.lookup(int(a), int(b)) for a, b in zip(left[:1000].tolist(), right[:1000].tolist())]
    assert [h[1] for h in hits] == rank[:1000].tolist() and [h[0] for h in hits] == new[:1000].tolist()


def test_parse_merges_errors():
    v = bpe.Vocab({"a": 0, "b": 1, "ab": 2})
    assert bpe.parse_merges("#version\na b\n", v) == [bpe.MergeRule(0, 1, 0, 2)]
    with pytest.raises(errors.MalformedLine):
        bpe.parse_merges("a b c\n", v)
    with pytest.raises(errors.UnknownSymbol):
        bpe.parse_merges("a c\n", v)


def test_build_table_errors():
    with pytest.raises(errors.DuplicatePair):
        bpe.build_table([bpe.MergeRule(1, 2, 0, 3), bpe.MergeRule(1, 2, 1, 4)])
    with pytest.raises(errors.ReservedKey):
        bpe.build_table([bpe.MergeRule(2**32 - 1, 2**32 - 1, 0, 3)])
    empty = bpe.build_table([])
    assert empty.capacity == 1 and empty.lookup(1, 2) is None


def test_missing_byte_symbol():
    with pytest.raises(errors.MissingSymbol):
        bpe.Tokenizer(bpe.Vocab({"a": 1}), bpe.build_table([]))


def test_block_config_validation():
    assert bpe.BlockConfig().chunk_budget == 8192
    for kw in ({"lane_count": 0}, {"max_seq_len": 1}, {"max_seq_len": 64, "chunk_budget": 65},
               {"chunk_budget": 1}):
        with pytest.raises(ValueError):
            bpe.BlockConfig(**kw)


def test_chunk_tokens():
    toks = np.arange(10, dtype=np.uint32)
    assert [len(c.tokens) for c in bpe.chunk_tokens(toks, 4)] == [4, 4, 2]
    assert bpe.chunk_tokens(np.empty(0, np.uint32), 4) == []
    with pytest.raises(errors.InvalidBudget):
        bpe.chunk_tokens(toks, 1)


def test_unknown_engine_rejected_before_work(tokenizer):
    with pytest.raises(ValueError):
        bpe.tokenize_batch([b"x"], tokenizer, "warp")
    with pytest.raises(ValueError):
        bpe.TokenizerHandle("missing.json", "missing.txt", engine="warp")


def test_bad_input_raises_batch_error_with_index(tokenizer):
    with pytest.raises(errors.BatchError) as exc:
        bpe.tokenize_batch([b"ok", 12.5], tokenizer)
    assert exc.value.input_index == 1


def test_pack_texts():
    data, offs = bpe.pack_texts(["héllo", b"", b"ab"])
    assert data.tobytes() == "héllo".encode() + b"ab"
    assert offs.tolist() == [0, 6, 6, 8]


def test_empty_batch_needs_no_device(tokenizer):
    res = bpe.tokenize_batch([], tokenizer)
    assert res.token_ids == [] and res.counters.passes == 0


# ------------------------------------------------------------- make_windows


def _windows_fixture():
    import gzip
    import json
    from pathlib import Path

    here = Path(__file__).resolve().parent / "golden"
    fx = json.loads((here / "windows.json").read_text())
    lines = gzip.decompress((here / "prose_corpus.txt.gz").read_bytes()).split(b"\n")
    return fx, b"\n".join(lines[: fx["corpus_lines"]])


def test_sweep_spec_validation():
    with pytest.raises(ValueError):
        bpe.SweepSpec(lengths=())
    with pytest.raises(ValueError):
        bpe.SweepSpec(lengths=(64, 16))
    with pytest.raises(ValueError):
        bpe.SweepSpec(measured_runs=0)
    bpe.SweepSpec(warmup_runs=0)


def test_make_windows_byte_mode_matches_reference():
    fx, corpus = _windows_fixture()
    for case in fx["cases"]:
        if case["mode"] != "byte":
            continue
        spec = bpe.SweepSpec(lengths=tuple(case["lengths"]), samples_per_length=case["samples"])
        got = bpe.make_windows(corpus, None, spec, seed=case["seed"])
        assert {str(k): [w.hex() for w in v] for k, v in got.items()} == case["windows"]
    with pytest.raises(errors.CorpusTooSmall):
        bpe.make_windows(b"short", None, bpe.SweepSpec(lengths=(256,)))
    with pytest.raises(errors.CorpusTooSmall):
        bpe.make_windows(b"", None, bpe.SweepSpec(lengths=(256,)))
    with pytest.raises(ValueError):
        bpe.make_windows(corpus, [1, 2, 3], bpe.SweepSpec(lengths=(1,)))


class _HostDecoder:
    """Stands in for the device decode on CPU (the reference's own algorithm)."""

    def __init__(self, tok):
        self.tok = tok

    def decode_batch(self, seqs):
        return [bpe.decode_tokens(s, self.tok.encoder, self.tok.vocab) for s in seqs]


def test_make_windows_token_mode_matches_reference_cpu(tokenizer):
    fx, corpus = _windows_fixture()
    for case in fx["cases"]:
        if case["mode"] != "token":
            continue
        spec = bpe.SweepSpec(lengths=tuple(case["lengths"]), samples_per_length=case["samples"])
        got = bpe.make_windows(corpus, fx["stream"], spec, tokenizer=_HostDecoder(tokenizer), seed=case["seed"])
        assert {str(k): [w.hex() for w in v] for k, v in got.items()} == case["windows"]


def _symbol_bytes_loop(tok, minlen):
    from paper_2603_02597_b200.byte_codec import symbol_bytes

    ids, pieces = [], []
    for tid, sym in tok.vocab.id_to_symbol.items():
        b = symbol_bytes(sym, tok.encoder)
        if b is not None and len(b) >= minlen:
            ids.append(tid)
            pieces.append(b)
    offs = np.zeros(len(pieces) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(p) for p in pieces])
    return np.array(ids, np.uint32), np.frombuffer(b"".join(pieces), np.uint8), offs


def test_vectorised_symbol_bytes_match_symbol_bytes(tokenizer):
    """The device tables' vocab strings (memo candidates, decode LUT) equal
    symbol_bytes applied symbol by symbol -- on GPT-2 and on a vocab with
    empty symbols, non-byte characters and astral code points."""
    enc = bpe.build_byte_encoder()
    b2s = {b: s for s, b in enc.symbol_to_byte.items()}
    base = {b2s[b]: b for b in range(256)}
    odd = dict(base)
    odd.update({"": 300, "a b": 301, b2s[104] + b2s[105]: 302, "\U0001F600": 303,
                b2s[0] + "一": 304, b2s[255] * 5: 305, "x": 306 if "x" not in base else 307})
    small = bpe.Tokenizer(bpe.Vocab(odd), bpe.build_table([]))
    for tok in (tokenizer, small):
        for got, minlen in ((tok._decode_strings(), 0), (tok._vocab_strings(), 2)):
            want = _symbol_bytes_loop(tok, minlen)
            assert all(np.array_equal(g, w) for g, w in zip(got, want))


def test_report_schema_matches_reference(tmp_path):
    """emit_report / compare_golden / load_golden_file reproduce the reference's
    output byte for byte (tests/golden/report.json, made by the reference itself:
    tests/golden/make_report_golden.py)."""
    import json
    from pathlib import Path

    from paper_2603_02597_b200 import report

    fx = json.loads((Path(__file__).parent / "golden" / "report.json").read_text())
    for case in fx["reports"]:
        recs = [report.BenchRecord(*r) for r in fx["records"][case["set"]]]
        assert report.emit_report(recs, case["fmt"], case["baseline"]) == case["text"], case
    for i, g in enumerate(fx["golden_files"]):
        p = tmp_path / f"g{i}.tokens"
        p.write_text(g["body"])
        assert report.load_golden_file(p) == g["loaded"]
        r = report.compare_golden(g["tokens"], p)
        assert (r.match, r.first_divergence, r.divergences) == (g["match"], g["first"], g["divergences"]), g
    with pytest.raises(errors.EmptyRecords):
        report.emit_report([], "csv")
    with pytest.raises(ValueError):
        report.emit_report([report.BenchRecord("a", 1, 1.0, 0.0, 1.0)], "xml")


def test_golden_file_errors(tmp_path):
    from paper_2603_02597_b200 import report

    for body in ("[1, 2, true]", "[1, 2", "1\nx\n", '{"a": 1}'):
        p = tmp_path / "g.tokens"
        p.write_text(body)
        with pytest.raises(errors.MalformedGoldenFile):
            report.load_golden_file(p)


def test_batch_counters_match_the_lane_engine_formulas():
    """_batch_counters (chunk lengths + id counts -> the reference's summed
    PassCounters) against run_block_engine's per-chunk formulas
    (engines.py:338-403, test_engines.py:266-289) and the tiny known answer."""
    from paper_2603_02597_b200.chunker import _batch_counters

    rng = np.random.default_rng(3)
    n = rng.integers(0, 300, 200)
    out = np.array([int(rng.integers(min(k, 1), k + 1)) if k else 0 for k in n])
    got = _batch_counters("optimized", None, n, out)
    lk = mv = al = 0
    for a, o in zip(n.tolist(), out.tolist()):
        if a < 2:
            continue
        last = o
        lk += sum(L - 1 for L in range(last if last >= 2 else last + 1, a + 1))
        mv += sum(a - k - 1 for k in range(a - o))
        al += 2
    assert got == {"passes": int((n - out).sum()), "lookups": lk, "compaction_moves": mv, "buffer_allocations": al}
    assert _batch_counters("baseline", None, np.array([4]), np.array([2])) == \
        {"passes": 2, "lookups": 6, "compaction_moves": 5, "buffer_allocations": 2}


def test_chunk_units_match_chunk_tokens():
    from paper_2603_02597_b200.chunker import _chunk_units

    cfg = bpe.BlockConfig(max_seq_len=64, chunk_budget=16)
    lens = np.array([0, 1, 64, 65, 200, 3])
    doc, off, clen, first = _chunk_units(lens, cfg)
    want = []
    for d, L in enumerate(lens.tolist()):
        if L > 64:
            want += [(d, c.chunk_index * 16, len(c.tokens)) for c in bpe.chunk_tokens(np.zeros(L, np.uint32), 16, d)]
        else:
            want.append((d, 0, L))
    assert list(zip(doc.tolist(), off.tolist(), clen.tolist())) == want
    assert first.tolist() == [0, 1, 2, 3, 8, 21, 22]
    assert _chunk_units(np.array([5, 64]), cfg) is None


def test_lazy_counters_compute_once_on_first_read():
    from paper_2603_02597_b200.chunker import _LazyCounters

    calls = []

    def fn():
        calls.append(1)
        return {"passes": 3, "lookups": 4, "compaction_moves": 5, "buffer_allocations": 6}

    c = _LazyCounters(fn)
    assert not calls
    assert (c.passes, c.lookups, c.compaction_moves, c.buffer_allocations) == (3, 4, 5, 6)
    total = bpe.PassCounters()
    total.merge_from(c)
    assert total == bpe.PassCounters(3, 4, 5, 6) and len(calls) == 1
