"""Pin the CPU oracle (oracle/) to the reference's own outputs.

Everything compared here was produced by the reference itself
(tests/golden/make_golden.py): its 100 golden files, the ids it returns for
the bindings fixture, mixed_blob inputs under five BlockConfigs, known-answer
strings, and sha256 digests of the calibrated synthetic workloads.  Only once
these pass is the oracle trusted as the checker of the CUDA path.
"""

import hashlib
import random

import numpy as np
import pytest

import fixtures
from oracle.oracle import OracleEncoder, byte_symbols, greedy_merge


def sha(ids) -> str:
    return hashlib.sha256(np.asarray(ids, dtype="<u4").tobytes()).hexdigest()


def test_byte_symbols_anchor_points():
    syms = byte_symbols()
    assert syms[0x20] == "Ġ" and syms[0x7F] == "ġ" and syms[0xAD] == "Ń"
    assert syms[0x41] == "A" and syms[0x00] == "Ā"
    assert len(set(syms)) == 256


def test_tables_shape(oracle_tables):
    assert len(oracle_tables.left) == 50000
    assert len(oracle_tables.symbol_to_id) == 50257
    assert oracle_tables.base_ids[ord("t")] == 83
    first = (oracle_tables.left[0], oracle_tables.right[0], oracle_tables.new[0])
    assert first == (oracle_tables.symbol_to_id["Ġ"], oracle_tables.symbol_to_id["t"], 256)


def test_golden_prose_100(oracle, prose_samples):
    gold = fixtures.golden_prose()
    assert len(gold) == len(prose_samples) == 100
    got = oracle.encode_docs(prose_samples)
    bad = [i for i, (g, w) in enumerate(zip(got, gold)) if not np.array_equal(g, w)]
    assert not bad


def test_sequential_engine_matches_golden(oracle, prose_samples):
    gold = fixtures.golden_prose()
    for doc, want in list(zip(prose_samples, gold))[:10]:
        assert np.array_equal(oracle.sequential_bpe(oracle.base(doc)), want)


def test_batch_fixture(oracle):
    docs = fixtures.batch_fixture()
    want = fixtures.batch_fixture_ids()
    got = oracle.encode_docs(docs, 8192, 8192, threads=4)
    assert all(np.array_equal(g, w) for g, w in zip(got, want))


@pytest.mark.parametrize("cfg", ["default", "s64_b32", "s256_b256", "s512_b100", "whole"])
def test_mixed_cases(oracle, cfg):
    docs, cfgs = fixtures.mixed_cases()
    msl, cb, want = cfgs[cfg]
    got = oracle.encode_docs(docs, msl, cb, threads=4)
    bad = [i for i, (g, w) in enumerate(zip(got, want)) if not np.array_equal(g, w)]
    assert not bad, f"{cfg}: docs {bad[:10]} differ"


def test_known_answers(oracle):
    ka = fixtures.known_answers()
    for hexs, want in ka["cases"].items():
        assert oracle.encode_docs([bytes.fromhex(hexs)])[0].tolist() == want, hexs
    assert oracle.base(b"the").tolist() == ka["base_the"] == [83, 71, 68]


@pytest.mark.parametrize("name", ["c0_1k", "c1_8k", "c1_32k", "c1_131k", "c3_1m"])
def test_synthetic_workloads(oracle, name):
    import synth_corpus

    spec = fixtures.synth_sizes()[name]
    doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
    whole = oracle.sequential_bpe(oracle.base(doc))
    assert len(whole) == spec["tokens_whole"]
    assert sha(whole) == spec["sha_whole"]
    dflt = oracle.encode_docs([doc], 8192, 8192)[0]
    assert len(dflt) == spec["tokens_default"] and sha(dflt) == spec["sha_default"]


def test_naive_greedy_agrees_small(oracle, oracle_tables):
    pm = oracle_tables.pair_map
    rng = random.Random(3)
    for _ in range(40):
        data = bytes(rng.choice(b"abcdefg th\n0123") for _ in range(rng.randrange(0, 60)))
        assert oracle.encode_docs([data], 1 << 40, 1 << 40)[0].tolist() == greedy_merge(
            oracle.base(data), pm)


def test_trace_is_nondecreasing_for_gpt2(oracle, prose_samples):
    # GPT-2's table is well-formed: merge ranks come out in non-decreasing order.
    _, trace = oracle.sequential_bpe(oracle.base(prose_samples[0]), with_trace=True)
    assert np.all(np.diff(trace.astype(np.int64)) >= 0)
