import os, sys, time, statistics
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np, torch
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
spec = fixtures.synth_sizes()["c3_1m"]
doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
W = 1 << 40
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=W, chunk_budget=W))
def t(fn, k=50):
    for _ in range(5): fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); r = fn(); ts.append(time.perf_counter() - t0); del r
    return 1e6 * statistics.median(ts)
n = len(bpe.tokenize_batch([doc], tok).token_ids[0])
us = t(lambda: bpe.tokenize_batch([doc], tok))
print("c3_1m tokenize_batch %.1f us  (%d ids, %.2f Gtok/s)" % (us, n, n / us / 1e3))
