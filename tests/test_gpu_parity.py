"""Parity of the CUDA path (through the C ABI) with the reference / oracle.

Every expected value is either the reference's own output (committed goldens
made by tests/golden/make_golden.py) or the C oracle pinned to it
(tests/test_oracle.py).  Bit-exact comparison throughout (integer ids).
"""

import hashlib
import random
import threading

import numpy as np
import pytest

import fixtures
import paper_2603_02597_b200 as bpe

pytestmark = pytest.mark.gpu


def sha(ids) -> str:
    return hashlib.sha256(np.asarray(ids, dtype="<u4").tobytes()).hexdigest()


def with_config(tokenizer, msl, cb):
    tok = bpe.Tokenizer(tokenizer.vocab, tokenizer.table, bpe.BlockConfig(max_seq_len=msl, chunk_budget=cb))
    tok._devices = tokenizer._devices  # share the device tables (config is per call)
    return tok


def assert_same(got, want, label=""):
    assert len(got) == len(want), label
    bad = [i for i, (g, w) in enumerate(zip(got, want)) if not np.array_equal(g, w)]
    assert not bad, f"{label}: {len(bad)} docs differ, first {bad[:8]}"


def test_native_library_is_the_engine(tokenizer):
    res = bpe.tokenize_batch([b"hello world"], tokenizer, "cuda")
    assert res.token_ids[0].tolist() == [31373, 995]
    from paper_2603_02597_b200 import _native

    assert _native._lib is not None


def test_golden_prose_100(tokenizer, prose_samples):
    res = bpe.tokenize_batch(prose_samples, tokenizer)
    assert_same(res.token_ids, fixtures.golden_prose(), "golden")
    assert res.counters.passes == sum(map(len, prose_samples)) - sum(map(len, res.token_ids))
    assert res.device_stats["memo_hits"] > 0


def test_golden_prose_one_by_one(tokenizer, prose_samples):
    gold = fixtures.golden_prose()
    for doc, want in list(zip(prose_samples, gold))[:10]:
        assert np.array_equal(bpe.tokenize_batch([doc], tokenizer).token_ids[0], want)


def test_handle_on_bindings_fixture(gpt2_paths):
    h = bpe.TokenizerHandle(*gpt2_paths)
    ids, ms = h.tokenize_batch(fixtures.batch_fixture())
    want = fixtures.batch_fixture_ids()
    assert ids == [w.tolist() for w in want] and ms >= 0.0


@pytest.mark.parametrize("cfg", ["default", "s64_b32", "s256_b256", "s512_b100", "whole"])
def test_mixed_cases(tokenizer, cfg):
    docs, cfgs = fixtures.mixed_cases()
    msl, cb, want = cfgs[cfg]
    res = bpe.tokenize_batch(docs, with_config(tokenizer, msl, cb))
    assert_same(res.token_ids, want, cfg)


@pytest.mark.parametrize("cfg", ["default", "s64_b32", "whole"])
def test_mixed_cases_one_doc_per_call(tokenizer, cfg):
    docs, cfgs = fixtures.mixed_cases()
    msl, cb, want = cfgs[cfg]
    tok = with_config(tokenizer, msl, cb)
    for i in range(0, len(docs), 7):
        got = bpe.tokenize_batch([docs[i]], tok).token_ids[0]
        assert np.array_equal(got, want[i]), (cfg, i)


def test_known_answers(tokenizer):
    ka = fixtures.known_answers()
    docs = [bytes.fromhex(h) for h in ka["cases"]]
    res = bpe.tokenize_batch(docs, tokenizer)
    for g, w in zip(res.token_ids, ka["cases"].values()):
        assert g.tolist() == w


@pytest.mark.parametrize("name", ["c0_1k", "c1_8k", "c1_32k", "c1_131k", "c3_1m"])
def test_synthetic_workloads_against_reference_digests(tokenizer, name):
    import synth_corpus

    spec = fixtures.synth_sizes()[name]
    doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
    whole = bpe.tokenize_batch([doc], with_config(tokenizer, 1 << 40, 1 << 40)).token_ids[0]
    assert len(whole) == spec["tokens_whole"] and sha(whole) == spec["sha_whole"]
    dflt = bpe.tokenize_batch([doc], tokenizer).token_ids[0]
    assert len(dflt) == spec["tokens_default"] and sha(dflt) == spec["sha_default"]


ADVERSARIAL = {
    "digits": lambda n, r: bytes(r.choice(b"0123456789") for _ in range(n)),
    "newlines": lambda n, r: b"\n" * n,
    "aaaa": lambda n, r: b"a" * n,
    "letters": lambda n, r: bytes(r.choice(b"abcdefghijklmnopqrstuvwxyz") for _ in range(n)),
    "spaces": lambda n, r: b" " * n,
    "hex": lambda n, r: bytes(r.choice(b"0123456789abcdef") for _ in range(n)),
}


@pytest.mark.parametrize("kind", sorted(ADVERSARIAL))
@pytest.mark.parametrize("n", [1000, 2047, 2048, 3000, 40000, 300000])
def test_adversarial_long_segments(tokenizer, oracle, kind, n):
    doc = ADVERSARIAL[kind](n, random.Random(n))
    for msl, cb in ((1 << 40, 1 << 40), (8192, 8192), (5000, 3000)):
        got = bpe.tokenize_batch([doc, b"x" + doc], with_config(tokenizer, msl, cb)).token_ids
        want = oracle.encode_docs([doc, b"x" + doc], msl, cb)
        assert_same(got, want, f"{kind}/{n}/{msl}")


def test_million_byte_adversarial(tokenizer, oracle):
    r = random.Random(11)
    docs = [bytes(r.choice(b"0123456789") for _ in range(1 << 20)), b"a" * (1 << 20),
            b"\n" * (1 << 20)]
    got = bpe.tokenize_batch(docs, with_config(tokenizer, 1 << 40, 1 << 40))
    assert_same(got.token_ids, oracle.encode_docs(docs, 1 << 40, 1 << 40), "1M adversarial")
    assert got.device_stats["giant_segments"] >= 3


def test_many_giant_documents(tokenizer, oracle):
    """Many giant segments (> 4 KiB without a junction cut) in one call: up to
    64 KiB each is encoded by one CTA, concurrently (kernels.cu cta_giants);
    longer ones by the whole grid.  Digits, hex, letters and newline runs of
    4-90 KB, with prose between some, under both chunking configs."""
    r = random.Random(17)
    kinds = ["digits", "hex", "letters", "newlines", "aaaa"]
    docs = []
    for i in range(160):
        n = r.choice([4100, 5000, 9000, 17000, 33000, 65536, 70000, 90000]) if i % 7 else r.randint(4097, 12000)
        body = ADVERSARIAL[kinds[i % len(kinds)]](n, r)
        docs.append(body if i % 3 else b"The table " + body + b" ends here.")
    for msl, cb in ((1 << 40, 1 << 40), (8192, 8192)):
        got = bpe.tokenize_batch(docs, with_config(tokenizer, msl, cb))
        assert_same(got.token_ids, oracle.encode_docs(docs, msl, cb), f"giant docs {msl}")
        assert got.device_stats["giant_segments"] >= 20


def test_deferred_segment_routes(tokenizer, oracle):
    """Deferred segments of every route (kernels.cu encode_deferred / cta_giants):
    <= 221 B on a warp in its shared tile staging, 222-1024 B on a warp in the
    arena (129 B and up on one CTA when a call has few records), 1025 B - 7 KB
    on one CTA in shared memory, longer on one CTA in the arena, and a lone
    routed segment on one CTA (<= 4 KiB) or the whole grid.  Many per call and
    one per call, under both chunking configs."""
    r = random.Random(23)
    kinds = ["digits", "hex", "letters", "newlines", "aaaa", "spaces"]
    sizes = [33, 100, 128, 129, 221, 222, 223, 400, 512, 513, 900, 1024, 1025, 1026, 2000, 4096, 4097, 7100,
             7185, 7186, 7300, 8192]
    docs = []
    for i in range(300):
        n = sizes[i % len(sizes)] if i < 2 * len(sizes) else r.randint(33, 9000)
        body = ADVERSARIAL[kinds[i % len(kinds)]](n, r)
        docs.append(body if i % 4 else b"Value: " + body + b".")
    for msl, cb in ((1 << 40, 1 << 40), (8192, 8192), (3000, 3000)):
        got = bpe.tokenize_batch(docs, with_config(tokenizer, msl, cb))
        assert_same(got.token_ids, oracle.encode_docs(docs, msl, cb), f"routes {msl}")
    for n in (130, 600, 4096, 4097, 5000):  # one routed segment alone: one CTA up to 4 KiB, else the grid
        doc = ADVERSARIAL["digits"](n, r)
        got = bpe.tokenize_batch([doc], with_config(tokenizer, 1 << 40, 1 << 40)).token_ids
        assert_same(got, oracle.encode_docs([doc], 1 << 40, 1 << 40), f"lone {n}")


def test_many_small_and_empty_docs(tokenizer, oracle):
    r = random.Random(5)
    docs = []
    for i in range(5000):
        k = r.choice([0, 0, 1, 2, 3, 5, 8, 13, 40, 300])
        docs.append(bytes(r.choice(b"ab \ncde.,0") for _ in range(k)))
    docs += [b""] * 100
    for msl, cb in ((8192, 8192), (4, 2), (16, 5)):
        got = bpe.tokenize_batch(docs, with_config(tokenizer, msl, cb)).token_ids
        assert_same(got, oracle.encode_docs(docs, msl, cb, threads=8), f"small/{msl}")


def test_only_empty_docs(tokenizer):
    res = bpe.tokenize_batch([b"", b"", ""], tokenizer)
    assert [x.tolist() for x in res.token_ids] == [[], [], []]


def test_random_bytes_large_batch(tokenizer, oracle):
    rng = np.random.default_rng(9)
    docs = [rng.integers(0, 256, size=int(rng.integers(0, 20000)), dtype=np.uint8).tobytes()
            for _ in range(64)]
    got = bpe.tokenize_batch(docs, tokenizer).token_ids
    assert_same(got, oracle.encode_docs(docs, 8192, 8192, threads=8), "random bytes")


def test_memo_off_and_strict_engines_agree(tokenizer, oracle, prose_samples):
    docs, cfgs = fixtures.mixed_cases()
    msl, cb, want = cfgs["default"]
    for memo, strict in ((False, False), (True, True)):
        enc = tokenizer.device_encoder(memo=memo, strict=strict)
        data, offs = bpe.pack_texts(docs)
        ids, out_offs, st, _ = enc.encode_packed_host(data, offs, msl, cb)
        got = [ids[out_offs[i]:out_offs[i + 1]] for i in range(len(docs))]
        assert_same(got, want, f"memo={memo} strict={strict}")
        if not memo:
            assert st["memo_hits"] == 0


def test_device_pair_table_matches_rules(tokenizer, oracle_tables):
    enc = tokenizer.device_encoder()
    nw, rk = enc.lookup_pairs(oracle_tables.left, oracle_tables.right)
    assert np.array_equal(nw, oracle_tables.new) and np.array_equal(rk, oracle_tables.rank)
    rng = np.random.default_rng(1)
    l = rng.integers(0, 50257, 10000).astype(np.uint32)
    r = rng.integers(0, 50257, 10000).astype(np.uint32)
    pm = oracle_tables.pair_map
    nw, rk = enc.lookup_pairs(l, r)
    for a, b, n, k in zip(l, r, nw, rk):
        hit = pm.get((int(a), int(b)))
        assert (k == 0xFFFFFFFF) if hit is None else (int(k), int(n)) == hit


def test_concurrent_handle_calls(gpt2_paths):
    h = bpe.TokenizerHandle(*gpt2_paths)
    docs = fixtures.batch_fixture()[:8]
    first, _ = h.tokenize_batch(docs)
    out = [None] * 4

    def work(k):
        out[k] = h.tokenize_batch(docs)[0]

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(o == first for o in out)


def test_device_csr_api(tokenizer, prose_samples):
    import torch

    enc = tokenizer.device_encoder()
    data, offs = bpe.pack_texts(prose_samples[:10])
    d = torch.from_numpy(data.copy()).cuda()
    o = torch.from_numpy(offs).cuda()
    ids, out_offs, st = enc.encode_tensors(d, o, 8192, 8192)
    gold = fixtures.golden_prose()[:10]
    oo = out_offs.cpu().numpy()
    h = ids.cpu().numpy().view(np.uint32)
    for i in range(10):
        assert np.array_equal(h[oo[i]:oo[i + 1]], gold[i])
    assert st["n_bytes"] == len(data) and st["n_ids"] == len(h)
    assert st["passes"] == st["n_bytes"] - st["n_ids"] == sum(len(d) for d in prose_samples[:10]) - len(h)


def test_device_junction_bits_match_rules_and_split_exactly(tokenizer, oracle, oracle_tables):
    from paper_2603_02597_b200 import multigpu
    from test_multigpu import junction_bits

    jb = tokenizer.device_encoder().junction_bits()
    assert np.array_equal(jb, junction_bits(oracle_tables))
    doc = b"".join(fixtures.prose_samples()[:20])
    for msl, cb in ((1 << 40, 1 << 40), (8192, 8192), (5000, 3000)):
        tok = with_config(tokenizer, msl, cb)
        want = oracle.encode_docs([doc], msl, cb)[0]
        for world in (2, 4, 8):
            shards = multigpu.split_document(doc, world, jb, msl, cb)
            got = [bpe.tokenize_batch(s, tok).token_ids for s in shards if s]
            got = np.concatenate([i for g in got for i in g])
            assert np.array_equal(got, want), (msl, world)


# ---------------------------------------------------------------- decode


def test_decode_known_answers(tokenizer):
    assert tokenizer.decode([31373, 995]) == b"hello world"
    assert tokenizer.decode([1169]) == b"the"  # test_byte_codec.py:78-81
    assert tokenizer.decode([]) == b""  # test_byte_codec.py:74-75
    assert tokenizer.decode([50256]) == b"<|endoftext|>"
    with pytest.raises(bpe.errors.UnknownTokenId):
        tokenizer.decode([2**32 - 1])  # test_byte_codec.py:84-86
    with pytest.raises(bpe.errors.UnknownTokenId):
        tokenizer.decode([31373, 50257, 995])


def test_decode_roundtrips_and_matches_host_helper(tokenizer):
    docs, cfgs = fixtures.mixed_cases()
    msl, cb, want = cfgs["default"]
    got = tokenizer.decode_batch(want)
    assert got == [bytes(d) if isinstance(d, (bytes, bytearray)) else d.encode() for d in docs]
    rng = np.random.default_rng(4)
    seqs = [rng.integers(0, 50257, int(rng.integers(0, 3000))) for _ in range(40)]
    host = [bpe.decode_tokens(s, tokenizer.encoder, tokenizer.vocab) for s in seqs]
    assert tokenizer.decode_batch(seqs) == host


def test_decode_large_and_adversarial(tokenizer, oracle):
    import synth_corpus

    spec = fixtures.synth_sizes()["c3_1m"]
    doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
    ids = bpe.tokenize_batch([doc], with_config(tokenizer, 1 << 40, 1 << 40)).token_ids[0]
    assert tokenizer.decode(ids) == doc
    longest = max(tokenizer.vocab.id_to_symbol, key=lambda i: len(tokenizer.vocab.id_to_symbol[i]))
    big = [longest] * 20000  # ~2.5 MB of output from 80 KB of ids: unstaged tiles
    assert tokenizer.decode(big) == bpe.decode_tokens([longest], tokenizer.encoder, tokenizer.vocab) * 20000


def test_make_windows_token_mode_device_decode_matches_reference(tokenizer):
    from test_api import _windows_fixture

    fx, corpus = _windows_fixture()
    for case in fx["cases"]:
        if case["mode"] != "token":
            continue
        spec = bpe.SweepSpec(lengths=tuple(case["lengths"]), samples_per_length=case["samples"])
        got = bpe.make_windows(corpus, fx["stream"], spec, tokenizer=tokenizer, seed=case["seed"])
        assert {str(k): [w.hex() for w in v] for k, v in got.items()} == case["windows"]


# ---------------------------------------------------------------- GPT-2 regex mode


@pytest.fixture(scope="module")
def tiktoken_gpt2(gpt2_paths):
    from oracle.tiktoken_gpt2 import build

    return build(gpt2_paths[0])


def test_regex_mode_matches_tiktoken(tokenizer, tiktoken_gpt2):
    import random as _r

    docs = [d for d in fixtures.prose_samples()]
    docs += [s.encode() for s in ["hello world", "it's", "IT'S don't we'll you've they're I'd I'm",
                                  "\n\nhello", "  x  ", "x \n y", "日本語のテキスト、です。", "naïve café ½ ²",
                                  "e.g. U.S.A. 3.14159 $1,000,000!!!", "\t\ttabs\tand nbsp　x", "",
                                  "a" * 3000, "1234567890" * 50, "\n" * 100 + "x"]]
    rng = _r.Random(3)
    alphabet = "ab's dmtlvre'  \n\t1.?!,é日😀"
    docs += ["".join(rng.choice(alphabet) for _ in range(rng.randint(0, 200))).encode() for _ in range(300)]
    # long ASCII documents: the bit-parallel paths of k_pretok (with and without apostrophes,
    # every ASCII whitespace, controls and the class edges @ [ ` { / : 0x1c-0x1f 0x7f)
    ascii_alpha = ["abZ zy  \n\t\r\x0b\x0c1909.?!,_@[`{/:\x1c\x1f\x7f", "ab's dmtlvre'  \n1."]
    for k in range(120):
        a = ascii_alpha[k % 2]
        docs.append("".join(rng.choice(a) for _ in range(rng.randint(0, 3000))).encode())
    for k in range(400):  # short ASCII documents: several per 32-byte word
        a = ascii_alpha[k % 2]
        docs.append("".join(rng.choice(a) for _ in range(rng.randint(0, 40))).encode())
    tok = with_config(tokenizer, 1 << 40, 1 << 40)
    got = bpe.tokenize_batch(docs, tok, pretokenize="gpt2").token_ids
    for i, (d, g) in enumerate(zip(docs, got)):
        assert g.tolist() == tiktoken_gpt2.encode_ordinary(d.decode("utf-8")), i
    # the default mode is untouched afterwards
    assert bpe.tokenize_batch([b"\n\nhello"], tokenizer).token_ids[0].tolist() == [628, 31373]


def test_regex_mode_large_document(tokenizer, tiktoken_gpt2):
    import synth_corpus

    spec = fixtures.synth_sizes()["c3_1m"]
    doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
    got = bpe.tokenize_batch([doc], with_config(tokenizer, 1 << 40, 1 << 40), pretokenize="gpt2").token_ids[0]
    assert got.tolist() == tiktoken_gpt2.encode_ordinary(doc.decode("utf-8"))
    with pytest.raises(ValueError):
        bpe.tokenize_batch([doc], tokenizer, pretokenize="o200k")


@pytest.mark.parametrize("regex,pinned_in,pinned_out", [(False, False, True), (True, False, True),
                                                         (False, True, True), (False, True, False),
                                                         (False, False, False)])
def test_streamed_host_encode_matches_device_encode(tokenizer, oracle, monkeypatch, regex, pinned_in,
                                                    pinned_out):
    """gpubpe_encode_host on a batch larger than two parts runs the two-slot
    pipeline (parts of GPUBPE_STREAM_MB MiB, here 1): its ids, offsets and
    counters equal one device-resident encode of the whole batch; docs of every
    size, empty ones and a document larger than a part included."""
    import torch
    import synth_corpus

    rng = np.random.default_rng(11)
    pool = synth_corpus.english_bytes(3 << 20, 4)
    docs, at = [], 0
    for k in range(700):
        n = int(rng.choice([0, 1, 17, 300, 5000, 20000])) if k != 350 else (2 << 20) + 12345
        docs.append(pool[at % (1 << 20): at % (1 << 20) + n] if k != 350 else pool[:n])
        at += 7919
    data, offs = bpe.pack_texts(docs)
    assert data.size > (2 << 20)
    enc = tokenizer.device_encoder()
    mode = 1 if regex else 0
    monkeypatch.setenv("GPUBPE_STREAM_MB", "0")
    d = torch.from_numpy(data.copy()).cuda()
    o = torch.from_numpy(offs).cuda()
    enc.set_mode(mode)
    try:
        ids_d, offs_d, st_d = enc.encode_tensors(d, o, 8192, 8192)
    finally:
        enc.set_mode(0)
    want_ids, want_offs = ids_d.cpu().numpy().view(np.uint32), offs_d.cpu().numpy()
    monkeypatch.setenv("GPUBPE_STREAM_MB", "1")
    if pinned_in:  # the DMA reads the caller's bytes directly
        pd = bpe.pinned_empty(data.size)
        pd[:] = data
        data = pd
    if not pinned_out:  # result buffer in pageable memory: ids staged through the slots
        from paper_2603_02597_b200 import device

        monkeypatch.setattr(device, "_POOLED_MAX", 0)
    ids, oo, st, _ = enc.encode_packed_host(data, offs, 8192, 8192, mode=mode)
    assert np.array_equal(oo, want_offs)
    assert np.array_equal(ids, want_ids)
    for k in ("n_ids", "passes"):  # (segment/pass counters depend on the tiling)
        assert st[k] == st_d[k], k
    if not regex:  # and against the oracle on a sample of documents
        sample = list(range(0, 700, 37)) + [350]
        want = oracle.encode_docs([docs[i] for i in sample], 8192, 8192)
        for i, w in zip(sample, want):
            assert np.array_equal(ids[oo[i]:oo[i + 1]], w), i


def _parse_errors(fn, text, vocab):
    try:
        fn(text, vocab)
    except Exception as exc:  # noqa: BLE001 - the exact type and message are compared
        return type(exc), str(exc)
    return None


def test_device_merges_parse_matches_host(gpt2_paths):
    """merges.txt parsed on the device gives the reference's rules,
    and Tokenizer.from_files built from them has the reference's packed table."""
    from pathlib import Path

    from paper_2603_02597_b200.merge_table import parse_merges_device

    vocab = bpe.Vocab.from_file(gpt2_paths[0])
    text = Path(gpt2_paths[1]).read_bytes()
    left, right, rank, new = parse_merges_device(text, vocab)
    rules = bpe.parse_merges(text, vocab)
    assert len(left) == len(rules) == 50000
    assert left.tolist() == [r.left for r in rules] and right.tolist() == [r.right for r in rules]
    assert new.tolist() == [r.new_token for r in rules] and rank.tolist() == [r.rank for r in rules]
    tok = bpe.Tokenizer.from_files(*gpt2_paths)
    assert tok._rules is not None  # took the device parser
    ref = bpe.build_table(rules)
    assert np.array_equal(tok.table.keys, ref.keys) and np.array_equal(tok.table.values, ref.values)


def test_device_merges_parse_errors_match_host(gpt2_paths):
    from paper_2603_02597_b200.merge_table import parse_merges_device

    vocab = bpe.Vocab.from_file(gpt2_paths[0])
    good = "#version: 0.2\nĠ t\nĠ a\nh e\n"
    cases = [good, good.rstrip("\n"), "Ġ t\n", "Ġ t\n\nh e\n", "Ġ t x\n", "Ġt\n", " t\n", "Ġ \n",
             "Ġ t\nzzz§ q\n", "Ġ t\nh e\n# comment later\n", "#only header\n", "", "\n", "Ġ t\r\nh e\r\n",
             "Ġ t\x0bh e\n", "Ġ t\n" * 3]
    for c in cases:
        raw = c.encode("utf-8")
        want = _parse_errors(bpe.parse_merges, raw, vocab)
        got = _parse_errors(parse_merges_device, raw, vocab)
        if want is not None:
            assert got == want, (c, got, want)
        else:
            assert got is None, (c, got)
            res = parse_merges_device(raw, vocab)
            if res is not None:  # (None: line breaks only the host parser handles)
                rules = bpe.parse_merges(raw, vocab)
                assert res[0].tolist() == [r.left for r in rules], c
                assert res[3].tolist() == [r.new_token for r in rules], c
    bad_utf8 = b"\xff\xfe t\n"
    assert _parse_errors(parse_merges_device, bad_utf8, vocab) == _parse_errors(bpe.parse_merges, bad_utf8, vocab)


def test_device_junction_build_matches_host_loops(tokenizer, prose_samples):
    from paper_2603_02597_b200.device import DeviceEncoder

    left, right, rank, new = tokenizer.rule_arrays()
    vids, blob, offs = tokenizer._vocab_strings()
    dev = DeviceEncoder(tokenizer._base_ids, left, right, rank, new, vids, blob, offs, device=0)
    host = DeviceEncoder(tokenizer._base_ids, left, right, rank, new, vids, blob, offs, device=0,
                         host_tables=True)
    assert np.array_equal(dev.junction_bits(), host.junction_bits())
    data, doffs = bpe.pack_texts(prose_samples[:20])
    a = dev.encode_packed_host(data, doffs, 8192, 8192)
    b = host.encode_packed_host(data, doffs, 8192, 8192)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_steady_state_needs_no_allocations(tokenizer, prose_samples):
    """Workspaces are grow-only: repeating a call allocates nothing on the
    device (device_stats["allocations"])."""
    docs = prose_samples[:50]
    bpe.tokenize_batch(docs, tokenizer)
    again = bpe.tokenize_batch(docs, tokenizer)
    assert again.device_stats["allocations"] == 0
    bpe.tokenize_batch(docs * 40, tokenizer)  # may grow the workspace once
    assert bpe.tokenize_batch(docs * 40, tokenizer).device_stats["allocations"] == 0


def test_batch_beyond_4_gib_offsets(tokenizer, oracle):
    """A 4.3 GiB batch: byte and id offsets past 2**32 (64-bit positions end to
    end); documents around the 2**32 boundary and a random sample equal the
    oracle, and the CSR is consistent."""
    import torch
    import synth_corpus

    total = (1 << 32) + (300 << 20)
    data, offs = synth_corpus.corpus_docs(total, seed=3)
    d = torch.from_numpy(data).cuda()
    o = torch.from_numpy(offs).cuda()
    del data
    enc = tokenizer.device_encoder()
    out_ids = torch.empty(d.numel(), dtype=torch.int32, device="cuda")
    out_offs = torch.empty(o.numel(), dtype=torch.int64, device="cuda")
    enc.encode_into(d, o, out_ids, out_offs, 8192, 8192)
    st = enc.query()
    oo = out_offs.cpu().numpy()
    assert oo[0] == 0 and np.all(np.diff(oo) >= 0) and oo[-1] == st["n_ids"]
    assert st["passes"] == total - st["n_ids"]
    b = int(np.searchsorted(offs, 1 << 32, side="right")) - 1  # the document holding byte 2**32
    rng = np.random.default_rng(7)
    sample = sorted(set(range(max(0, b - 3), min(len(offs) - 1, b + 4))) |
                    set(rng.integers(0, len(offs) - 1, 12).tolist()) | {len(offs) - 2})
    docs = [bytes(d[int(offs[i]):int(offs[i + 1])].cpu().numpy()) for i in sample]
    want = oracle.encode_docs(docs, 8192, 8192)
    for i, w in zip(sample, want):
        got = out_ids[int(oo[i]):int(oo[i + 1])].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, w), i
    del d, out_ids
    torch.cuda.empty_cache()


def test_run_sweep_and_profile_run_on_the_device(tokenizer, oracle, prose_samples, tmp_path):
    """The reference's sweep methodology on the device engine:
    windows cut by make_windows, goldens written from the oracle, every window
    matches; the report renders; profile_run's splits and counters hold."""
    corpus = b"\n".join(prose_samples[:30])
    spec = bpe.SweepSpec(lengths=(64, 512, 2048), samples_per_length=3, warmup_runs=1, measured_runs=3)
    windows = bpe.make_windows(corpus, None, spec, seed=5)
    for length, cell in windows.items():
        for k, ids in enumerate(oracle.encode_docs(cell, 8192, 8192)):
            (tmp_path / f"len{length}_s{k:03d}.tokens").write_text("\n".join(map(str, ids.tolist())) + "\n")
    recs = bpe.run_sweep(windows, ["cuda", "optimized"], spec, tokenizer, golden_dir=tmp_path)
    assert len(recs) == 6
    assert all(r.golden_matches == 3 and r.golden_divergences == 0 for r in recs)
    assert all(r.mean_latency_ms > 0 and r.throughput_tokens_per_s > 0 for r in recs)
    table = bpe.emit_report(recs, "table", baseline_engine="cuda")
    assert "optimized speedup_vs_cuda" in table and len(table.splitlines()) == 2 + 3
    prof = bpe.profile_run(prose_samples[:10], tokenizer)
    assert prof.counters.passes == sum(map(len, prose_samples[:10])) - sum(
        len(x) for x in bpe.tokenize_batch(prose_samples[:10], tokenizer).token_ids)
    assert prof.end_to_end_ms >= prof.engine_ms >= 0 and abs(sum(prof.event_shares.values()) - 1.0) < 1e-9


def _tiny():
    from types import SimpleNamespace

    symbols = {"a": 5, "b": 9, "c": 13, "d": 21, "e": 34, "f": 55,
               "ab": 100, "abc": 101, "cd": 103, "ef": 105, "bc": 107}
    rules = bpe.parse_merges("a b\nab c\nc d\ne f\nb c\n", bpe.Vocab(symbols))
    return SimpleNamespace(symbols=symbols, table=bpe.build_table(rules),
                           encode=lambda text: [symbols[ch] for ch in text],
                           pair_map={(r.left, r.right): (r.rank, r.new_token) for r in rules})


def test_token_level_engines_known_answers():
    """sequential_bpe / run_block_engine on token ids (engines.py:269-403) on the
    device: the reference's known answers, traces and counters."""
    tiny = _tiny()
    assert bpe.sequential_bpe([], tiny.table)[0].tolist() == []
    trace = []
    out, c = bpe.sequential_bpe(tiny.encode("abcd"), tiny.table, trace=trace)
    assert out.tolist() == [101, 21] and c.passes == 2 and trace == [0, 1]
    assert (c.lookups, c.compaction_moves, c.buffer_allocations) == (3 + 1 + 1, 0, 0)
    trace = []
    out, _ = bpe.sequential_bpe(tiny.encode("abab"), tiny.table, trace=trace)
    assert out.tolist() == [100, 100] and trace == [0, 0]
    out, c = bpe.run_block_engine(tiny.encode("abcd"), tiny.table)
    assert out.tolist() == [101, 21]
    assert (c.passes, c.buffer_allocations, c.lookups, c.compaction_moves) == (2, 2, 6, 5)
    with pytest.raises(bpe.errors.SequenceTooLong):
        bpe.run_block_engine(list(range(10)), tiny.table, bpe.BlockConfig(max_seq_len=8))
    with pytest.raises(ValueError):
        bpe.run_block_engine([5, 9], tiny.table, variant="fast")


def test_token_level_engines_match_greedy(tokenizer, oracle, oracle_tables):
    """Random tiny texts against the naive greedy (trace and lookups included),
    and GPT-2 prose / random bytes against the C oracle's sequential_bpe."""
    import random as _r

    from oracle.oracle import greedy_merge

    tiny = _tiny()
    rng = _r.Random(5)
    for _ in range(200):
        ids = tiny.encode("".join(rng.choice("abcdef") for _ in range(rng.randrange(0, 40))))
        trace = []
        out, c = bpe.sequential_bpe(ids, tiny.table, trace=trace)
        assert out.tolist() == greedy_merge(ids, tiny.pair_map), ids
        assert c.passes == len(ids) - len(out) and len(trace) == c.passes
        assert trace == sorted(trace)
    for doc in fixtures.prose_samples()[:5] + [bytes(rng.randrange(256) for _ in range(3000))]:
        ids = tokenizer.encode(doc)
        want, want_trace = oracle.sequential_bpe(ids, with_trace=True)
        trace = []
        out, c = bpe.sequential_bpe(ids, tokenizer.table, trace=trace)
        assert np.array_equal(out, want)
        assert trace == want_trace.tolist()
        out2, c2 = bpe.run_block_engine(ids[:8192], tokenizer.table, tokenizer.config)
        assert np.array_equal(out2, oracle.sequential_bpe(ids[:8192]))
    # ids outside the table never merge and stay in place
    out, _ = bpe.sequential_bpe([5, 9, 999999, 5, 9, 13], tiny.table)
    assert out.tolist() == [100, 999999, 101]


def test_decode_two_pass_large_batch(tokenizer):
    """A batch of ~7.5 M ids decodes through the two-pass path (tile totals +
    scan, no look-back): byte-exact round trip and offsets."""
    import torch
    import synth_corpus

    data, offs = synth_corpus.corpus_docs(32 << 20, seed=1)
    enc = tokenizer.device_encoder()
    d = torch.from_numpy(data).cuda()
    o = torch.from_numpy(offs).cuda()
    ids, ioffs, _ = enc.encode_tensors(d, o, 8192, 8192)
    assert ids.numel() > 4 * 148 * 8192
    out = torch.empty(data.size + 64, dtype=torch.uint8, device="cuda")
    oo = torch.empty_like(ioffs)
    n = enc.decode_into(ids, ioffs, out, oo)
    assert n == data.size
    assert torch.equal(out[:data.size], d)
    assert torch.equal(oo, o)


def _host_decode(tokenizer, ids, offs):
    """numpy restatement of decode_tokens over a CSR batch (bytes, byte offsets)."""
    sid, blob, soff = tokenizer._symbol_bytes()
    n = int(max(sid.max(), ids.max())) + 1
    lens = np.zeros(n, np.int64)
    start = np.zeros(n, np.int64)
    lens[sid] = np.diff(soff.astype(np.int64))
    start[sid] = soff[:-1].astype(np.int64)
    L = lens[ids]
    ends = np.cumsum(L)
    total = int(ends[-1]) if L.size else 0
    gather = np.repeat(start[ids] - (ends - L), L) + np.arange(total)
    cum = np.concatenate([[0], ends])
    return blob[gather], cum[offs]


def test_decode_rows_edge_cases(tokenizer):
    """The two-pass decode (first pass: tile and 256-id row totals; second: one
    warp per row range) on ~6 M ids: empty and one-id sequences, sequences that
    start exactly at row boundaries, more than 32 sequences starting in one row,
    rows of long tokens that exceed the warp's stage, an unaligned id pointer, a
    batch length that is not a multiple of 256; same bytes and offsets as the
    host restatement and as the CTA-tile kernel (GPUBPE_DEC_TILES) and the one-pass
    look-back kernel (GPUBPE_DEC_LOOKBACK)."""
    import os

    import torch

    sid, _, soff = tokenizer._symbol_bytes()
    rng = np.random.default_rng(11)
    n = 6_000_003
    ids = sid[rng.integers(0, sid.size, n + 1)].astype(np.uint32)
    lens = np.diff(soff.astype(np.int64))
    longest = sid[np.argsort(lens)[-64:]]
    ids[1_000_000:1_004_096] = longest[rng.integers(0, 64, 4096)]  # rows > 2 KiB of output
    cuts = [0]
    i = 0
    while i < n:
        k = int(rng.choice([0, 0, 1, 2, 3, 7, 256, 300, 5000]))
        if rng.random() < 0.02:
            k = 256 - (i % 256)  # next sequence starts on a row boundary
        i = min(n, i + k)
        cuts.append(i)
    cuts += [n, n]  # trailing empty sequences
    cuts += list(range(2_000_000, 2_004_000, 2)) + [2_000_512] * 40  # dense starts, empty runs
    offs = np.sort(np.asarray(cuts, np.int64))
    assert np.any(np.diff(np.searchsorted(offs, np.arange(0, n, 256))) > 40)  # >32 starts in a row
    enc = tokenizer.device_encoder()
    full = torch.from_numpy(ids.view(np.int32)).cuda()
    d_ids = full[1:]  # 4-byte offset: unaligned id loads
    want_bytes, want_offs = _host_decode(tokenizer, ids[1:], offs)
    o = torch.from_numpy(offs).cuda()
    results = []
    for knob in (None, "GPUBPE_DEC_TILES", "GPUBPE_DEC_LOOKBACK"):  # rows / CTA tiles / one pass
        if knob:
            os.environ[knob] = "1"
        try:
            out = torch.empty(want_bytes.size + 64, dtype=torch.uint8, device="cuda")
            oo = torch.empty_like(o)
            nb = enc.decode_into(d_ids, o, out, oo)
        finally:
            if knob:
                os.environ.pop(knob)
        assert nb == want_bytes.size
        assert np.array_equal(out[:nb].cpu().numpy(), want_bytes)
        assert np.array_equal(oo.cpu().numpy(), want_offs)
        results.append(out[:nb])
    assert torch.equal(results[0], results[1]) and torch.equal(results[0], results[2])
    # an unknown id deep inside the batch is reported by its index
    bad = full.clone()
    bad[3_333_334] = 60000
    with pytest.raises(bpe.errors.UnknownTokenId):
        enc.decode_into(bad[1:], o, torch.empty(want_bytes.size + 64, dtype=torch.uint8, device="cuda"),
                        torch.empty_like(o))
    # too small an output buffer: ValueError, nothing written past it
    with pytest.raises(ValueError):
        enc.decode_into(d_ids, o, torch.empty(want_bytes.size // 2, dtype=torch.uint8, device="cuda"),
                        torch.empty_like(o))


def test_decode_empty_and_long_symbols():
    """decode_tokens semantics (byte_codec.py:121-146) for symbols the GPT-2
    vocabulary does not have: an empty symbol decodes to no bytes, symbols of
    254, 255, 300 and 5000 bytes decode in full, a non-byte symbol is unknown --
    in the single-pass, CTA-tile and two-pass row kernels."""
    import os

    import torch

    from paper_2603_02597_b200.byte_codec import decode_tokens

    enc = bpe.build_byte_encoder()
    b2s = {b: s for s, b in enc.symbol_to_byte.items()}
    vocab = {b2s[b]: b for b in range(256)}
    rng = np.random.default_rng(5)
    long_ids = {}
    for k, n in enumerate((254, 255, 256, 300, 5000)):
        sym = "".join(b2s[int(b)] for b in rng.integers(0, 256, n))
        vocab[sym] = 300 + k
        long_ids[300 + k] = n
    vocab[""] = 400
    vocab["\u2603"] = 401  # not a byte character: unknown
    tok = bpe.Tokenizer(bpe.Vocab(vocab), bpe.build_table([]))
    pool = np.array(list(range(256)) + list(long_ids) + [400] * 20, np.uint32)
    seqs = [pool[rng.integers(0, pool.size, int(rng.integers(0, 40)))] for _ in range(300)]
    seqs += [np.array([400, 400], np.uint32), np.array([], np.uint32), np.array([304] * 3, np.uint32)]
    want = [decode_tokens(s.tolist(), tok.encoder, tok.vocab) for s in seqs]
    assert tok.decode_batch(seqs) == want
    # every kernel on one large batch (the row kernel is the default above ~1.5 M ids)
    big = pool[rng.integers(0, pool.size, 2_000_000)]
    offs = np.concatenate([[0], np.sort(rng.integers(0, big.size, 999)), [big.size]]).astype(np.int64)
    want_bytes = b"".join(decode_tokens(big[offs[i]:offs[i + 1]].tolist(), tok.encoder, tok.vocab)
                          for i in range(offs.size - 1))
    d = tok.device_encoder()
    d_ids = torch.from_numpy(big.view(np.int32)).cuda()
    o = torch.from_numpy(offs).cuda()
    for knob in (None, "GPUBPE_DEC_TILES", "GPUBPE_DEC_LOOKBACK"):
        if knob:
            os.environ[knob] = "1"
        try:
            out = torch.empty(len(want_bytes) + 64, dtype=torch.uint8, device="cuda")
            oo = torch.empty_like(o)
            nb = d.decode_into(d_ids, o, out, oo)
        finally:
            if knob:
                os.environ.pop(knob)
        assert nb == len(want_bytes), knob
        assert out[:nb].cpu().numpy().tobytes() == want_bytes, knob
    with pytest.raises(bpe.errors.UnknownTokenId):
        tok.decode_batch([np.array([1, 401], np.uint32)])


def test_integration_stub_binding(tokenizer, prose_samples):
    """The ctypes binding INTEGRATION.md shows a lanebpe maintainer (host buffers,
    no torch, no memo strings) gives the same ids as tokenize_batch."""
    import ctypes

    from paper_2603_02597_b200 import _native

    lib = ctypes.CDLL(str(_native.LIB_PATH))
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    lib.gpubpe_ctx_create.argtypes = [ctypes.c_int, vp, vp, vp, vp, vp, u64, vp, vp, vp, u64,
                                      ctypes.c_uint32, ctypes.POINTER(vp)]
    lib.gpubpe_encode_host.argtypes = [vp, vp, u64, vp, u64, u64, u64, vp, vp,
                                       ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_float), vp]
    lib.gpubpe_last_error.restype = ctypes.c_char_p
    lib.gpubpe_ctx_destroy.argtypes = [vp]
    keys, vals = tokenizer.table.keys, tokenizer.table.values
    live = keys != np.uint64(2**64 - 1)
    left = (keys[live] >> np.uint64(32)).astype(np.uint32)
    right = (keys[live] & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    new = (vals[live] >> np.uint64(32)).astype(np.uint32)
    rank = (vals[live] & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    base = np.ascontiguousarray(tokenizer._base_ids, np.uint32)
    h = vp()
    p = lambda a: a.ctypes.data  # noqa: E731
    rc = lib.gpubpe_ctx_create(0, p(base), p(left), p(right), p(rank), p(new), len(left), None, None, None, 0, 0,
                               ctypes.byref(h))
    assert rc == 0, lib.gpubpe_last_error(h)
    try:
        texts = prose_samples[:20] + [b"", b"hello world"]
        data = np.frombuffer(b"".join(texts), np.uint8)
        offs = np.zeros(len(texts) + 1, np.int64)
        offs[1:] = np.cumsum([len(x) for x in texts])
        ids = np.empty(max(len(data), 1), np.uint32)
        oo = np.empty(len(texts) + 1, np.int64)
        n, ms = u64(), ctypes.c_float()
        rc = lib.gpubpe_encode_host(h, p(data), len(data), p(offs), len(texts), 8192, 8192, p(ids), p(oo),
                                    ctypes.byref(n), ctypes.byref(ms), None)
        assert rc == 0, lib.gpubpe_last_error(h)
        got = [ids[oo[i]:oo[i + 1]] for i in range(len(texts))]
        assert_same(got, bpe.tokenize_batch(texts, tokenizer).token_ids, "stub")
    finally:
        lib.gpubpe_ctx_destroy(h)


def test_random_batches_random_configs_match_oracle(tokenizer, oracle):
    """Fuzz: random batches (prose, random bytes, runs, empty documents) under
    random chunking configs (tiny chunk budgets included) equal the oracle."""
    import synth_corpus

    rng = np.random.default_rng(2024)
    prose = synth_corpus.english_bytes(1 << 20, 9)
    for trial in range(25):
        docs = []
        for _ in range(int(rng.integers(1, 40))):
            n = int(np.exp(rng.uniform(0, np.log(60000)))) if rng.random() > 0.1 else 0
            kind = rng.integers(0, 4)
            if kind == 0:
                at = int(rng.integers(0, len(prose) - n - 1)) if n < len(prose) - 1 else 0
                docs.append(prose[at:at + n])
            elif kind == 1:
                docs.append(rng.integers(0, 256, n, dtype=np.uint8).tobytes())
            elif kind == 2:
                docs.append(bytes([int(rng.choice(list(b"a1 \n.\x00")))]) * n)
            else:
                docs.append(bytes(rng.choice(list(b"ab cd\n12"), n).tolist()))
        msl = int(rng.choice([2, 3, 17, 100, 1000, 8192, 1 << 40]))
        cb = msl if msl >= 1 << 40 or rng.random() < 0.3 else int(rng.integers(2, msl + 1))
        tok = with_config(tokenizer, msl, cb)
        got = bpe.tokenize_batch(docs, tok).token_ids
        want = oracle.encode_docs(docs, msl, cb)
        assert_same(got, want, f"trial {trial} msl {msl} cb {cb}")


@pytest.mark.parametrize("well_formed", [True, False])
def test_token_engine_random_tables_match_greedy(well_formed):
    """The device engines on random merge tables (well-formed: multi-merge passes;
    not: strict one-merge passes) equal the naive greedy on random sequences."""
    import random as _r

    from oracle.oracle import greedy_merge

    rng = _r.Random(7 if well_formed else 8)
    for trial in range(6):
        k = rng.randrange(3, 8)
        tokens = list(range(k))
        rules, seen = [], set()
        pending = []
        for rank in range(rng.randrange(10, 60)):
            a, b = rng.choice(tokens), rng.choice(tokens)
            if (a, b) in seen:
                continue
            seen.add((a, b))
            new = 100 + len(rules)
            rules.append(bpe.MergeRule(a, b, len(rules), new))
            tokens.append(new)
        if not well_formed:  # ranks shuffled: rules may use tokens produced at higher ranks
            ranks = list(range(len(rules)))
            rng.shuffle(ranks)
            rules = [bpe.MergeRule(r.left, r.right, ranks[i], r.new_token) for i, r in enumerate(rules)]
        table = bpe.build_table(sorted(rules, key=lambda r: r.rank))
        pair_map = {(r.left, r.right): (r.rank, r.new_token) for r in rules}
        for _ in range(40):
            ids = [rng.randrange(k) for _ in range(rng.randrange(0, 60))]
            out, c = bpe.sequential_bpe(ids, table)
            assert out.tolist() == greedy_merge(ids, pair_map), (trial, ids)
            assert c.passes == len(ids) - len(out)


def test_strict_pass_stops_at_first_violation():
    """Strict passes (tables that are not well-formed) merge the minimum-rank
    candidates only up to the first one whose merge creates a pair of rank <=
    the minimum; a candidate's left neighbour is the previous candidate's new
    token when they are adjacent, even across runs.  (a,b)->c r5, (c,c)->d r1,
    (d,a)->e r2 on "ababab": the reference merges @0, @1, then (c,c), then
    (d,a): [e, b]; merging all three (a,b) pairs in one pass would give [d, c]."""
    from oracle.oracle import greedy_merge

    a, b, c, d, e = 10, 11, 20, 21, 22
    rules = [bpe.MergeRule(c, c, 1, d), bpe.MergeRule(d, a, 2, e), bpe.MergeRule(a, b, 5, c)]
    table = bpe.build_table(rules)
    pair_map = {(r.left, r.right): (r.rank, r.new_token) for r in rules}
    for ids in ([a, b, a, b, a, b], [a, b, a, b, a, b, a, b], [b, a, b, a, b, a, b], [a, b] * 20):
        out, _ = bpe.sequential_bpe(ids, table)
        assert out.tolist() == greedy_merge(ids, pair_map), ids
    assert bpe.sequential_bpe([a, b, a, b, a, b], table)[0].tolist() == [e, b]


@pytest.mark.parametrize("well_formed", [True, False])
def test_byte_level_random_tables_match_oracle(well_formed):
    """k_encode (junction cuts, memo verification, warp / CTA / grid engines) with
    random byte-level merge tables, well-formed or not, against the C oracle on
    texts with long runs (deferred and giant segments)."""
    import random as _r

    from oracle.oracle import OracleEncoder

    rng = _r.Random(21 if well_formed else 22)
    enc = bpe.build_byte_encoder()
    b2s = {b: s for s, b in enc.symbol_to_byte.items()}
    symbols = {b2s[b]: b for b in range(256)}
    alphabet = b"abc d\n1"
    sym_of = {b: b2s[b] for b in range(256)}
    ids = [b for b in alphabet]
    rules, next_id = [], 256
    for _ in range(120):
        a, b = rng.choice(ids), rng.choice(ids)
        s = sym_of[a] + sym_of[b]
        if s in symbols or len(s) > 40:
            continue
        symbols[s] = next_id
        sym_of[next_id] = s
        rules.append(bpe.MergeRule(a, b, len(rules), next_id))
        ids.append(next_id)
        next_id += 1
    if not well_formed:
        ranks = list(range(len(rules)))
        rng.shuffle(ranks)
        rules = [bpe.MergeRule(r.left, r.right, ranks[i], r.new_token) for i, r in enumerate(rules)]
        rules.sort(key=lambda r: r.rank)
    tok = bpe.Tokenizer(bpe.Vocab(symbols), bpe.build_table(rules),
                        bpe.BlockConfig(max_seq_len=1 << 40, chunk_budget=1 << 40))
    left, right, rank, new = tok.rule_arrays()
    orc = OracleEncoder(tok._base_ids, left, right, rank, new)
    docs = []
    for _ in range(60):
        n = rng.choice([0, 1, 5, 50, 500, 5000, 20000])
        docs.append(bytes(rng.choice(alphabet) for _ in range(n)))
    docs += [b"a" * 30000, b"ab" * 9000, b"1" * 70000, b"abc d" * 3000]
    got = bpe.tokenize_batch(docs, tok).token_ids
    want = orc.encode_docs(docs, 1 << 40, 1 << 40)
    assert_same(got, want, f"well_formed={well_formed}")


def test_tokenize_batch_gather_paths(tokenizer, monkeypatch):
    """Multi-document batches go through gpubpe_encode_host_gather: piecewise
    staging straight from the documents (small batches) and the contiguous
    copy into the streamed pipeline (large ones, here above 2 x 1 MiB)."""
    import synth_corpus

    rng = np.random.default_rng(5)
    pool = synth_corpus.english_bytes(4 << 20, 6)
    docs = []
    for k in range(300):
        n = int(rng.choice([0, 3, 700, 9000, 40000]))
        at = int(rng.integers(0, len(pool) - n - 1))
        docs.append(pool[at:at + n])
    docs.append(pool[: 2 << 20])  # one document larger than a streamed part
    data, offs = bpe.pack_texts(docs)
    enc = tokenizer.device_encoder()
    ref_ids, ref_offs, _, _ = enc.encode_packed_host(data, offs, 8192, 8192)
    want = [ref_ids[ref_offs[i]:ref_offs[i + 1]].copy() for i in range(len(docs))]
    for stream_mb in ("0", "1"):
        monkeypatch.setenv("GPUBPE_STREAM_MB", stream_mb)
        res = bpe.tokenize_batch(docs, tokenizer)
        assert_same(res.token_ids, want, f"stream {stream_mb}")
        assert res.counters.passes == len(data) - sum(len(x) for x in want)


def test_regex_mode_fast_paths_equal_scalar_path(tokenizer, monkeypatch):
    """k_pretok's bit-parallel paths (SWAR, ASCII masks, Unicode masks) mark
    exactly the scalar code point path's pre-token starts, on valid and invalid
    UTF-8, runs of continuation bytes and documents starting mid-window."""
    import random as _r

    rng = _r.Random(31)
    pieces = ["漢字", "テキスト", "мир ", "café", "😀", " \u3000", "\u00a0x", "'s", "'ll", " 1234", "a", " ",
              "\n", "ß", "\t", "Ü", "\u2028", " \u3000\u3000 "]
    docs = []
    for k in range(400):
        n = rng.choice([0, 1, 3, 9, 33, 70, 200, 900])
        txt = "".join(rng.choice(pieces) for _ in range(n)).encode()
        if k % 5 == 0 and txt:  # invalid UTF-8: cut sequences, stray continuation runs, bad leads
            b = bytearray(txt)
            for _ in range(rng.randrange(1, 4)):
                b.insert(rng.randrange(len(b) + 1), rng.choice([0x80, 0xBF, 0xC3, 0xE6, 0xF0, 0xF8, 0xFF]))
            if rng.random() < 0.3:
                b[rng.randrange(len(b) + 1):0] = bytes([0x80] * rng.randrange(1, 8))
            txt = bytes(b)
        docs.append(txt)
    tok = with_config(tokenizer, 1 << 40, 1 << 40)
    monkeypatch.setenv("GPUBPE_PRETOK_PATHS", "0")
    want = bpe.tokenize_batch(docs, tok, pretokenize="gpt2").token_ids
    for paths in ("7", "6", "4", "2"):
        monkeypatch.setenv("GPUBPE_PRETOK_PATHS", paths)
        got = bpe.tokenize_batch(docs, tok, pretokenize="gpt2").token_ids
        assert_same(got, want, f"paths {paths}")


def test_encode_batch_tensors(tokenizer, prose_samples):
    import torch

    data, offs = bpe.pack_texts(prose_samples[:12])
    ids, oo = tokenizer.encode_batch_tensors(torch.from_numpy(data.copy()).cuda(), torch.from_numpy(offs).cuda())
    assert ids.is_cuda and ids.dtype == torch.int32 and oo.dtype == torch.int64
    h, ho = ids.cpu().numpy().view(np.uint32), oo.cpu().numpy()
    gold = fixtures.golden_prose()[:12]
    assert [h[ho[i]:ho[i + 1]].tolist() for i in range(12)] == [g.tolist() for g in gold]


@pytest.mark.gpu
@pytest.mark.parametrize("overlap", [True, False])
def test_single_document_host_paths(tokenizer, oracle, monkeypatch, overlap):
    """The single-document latency path (hostlist.c encode_one ->
    gpubpe_encode_host): below, at and above the overlapped-launch window
    (128 KiB .. 16 MiB: the kernel is launched while its input is in flight
    and its tiles wait for the arrival word), with chunking on and off, and
    the counters read from the kernel's mapped mirror (no state copy)."""
    import synth_corpus

    if not overlap:
        monkeypatch.setenv("GPUBPE_NO_OVERLAP", "1")
    for n in (100_000, 131_071, 131_072, 600_000, 3_000_000):
        doc = synth_corpus.english_bytes(n, n)
        for msl, cb in ((1 << 40, 1 << 40), (8192, 8192), (100_000, 65_536)):
            res = bpe.tokenize_batch([doc], with_config(tokenizer, msl, cb))
            want = oracle.encode_docs([doc], msl, cb)
            assert_same(res.token_ids, want, f"{n}/{msl}")
            st = res.device_stats
            assert st["n_ids"] == len(want[0]) and st["n_bytes"] == n and st["overflow"] == 0
            assert st["memo_hits"] > 0 and st["n_segments"] >= st["memo_hits"]
    # repeated calls of one size: no allocation
    doc = synth_corpus.english_bytes(600_000, 3)
    bpe.tokenize_batch([doc], with_config(tokenizer, 1 << 40, 1 << 40))
    assert bpe.tokenize_batch([doc], with_config(tokenizer, 1 << 40, 1 << 40)).device_stats["allocations"] == 0
