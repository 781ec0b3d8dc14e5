"""Host-side Python overheads around one tokenize_batch call (131k sequence)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
from paper_2603_02597_b200 import device as dv
spec = fixtures.synth_sizes()["c1_131k"]
doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
W = 1 << 40
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=W, chunk_budget=W))
enc = tok.device_encoder(0)
data, offs = bpe.pack_texts([doc])
def t(fn, k=300):
    for _ in range(10): fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(ts)
s = torch.cuda.current_stream(0)
print("device_encoder()       %6.2f us" % t(lambda: tok.device_encoder()))
print("torch.cuda.device ctx  %6.2f us" % t(lambda: torch.cuda.device(0).__enter__()))
print("current_stream         %6.2f us" % t(lambda: torch.cuda.current_stream(0)))
print("query                  %6.2f us" % t(lambda: enc.query(s)))
def takeput():
    b = dv._RESULTS.take(4 * data.size, enc._lib, 0); a = dv._RESULTS.array(b, np.uint32, 1000); del a
print("pool take+array        %6.2f us" % t(takeput))
print("encode_packed_host     %6.2f us" % t(lambda: enc.encode_packed_host(data, offs, W, W)))
print("tokenize_batch         %6.2f us" % t(lambda: bpe.tokenize_batch([doc], tok)))
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    bpe.tokenize_batch([doc], tok)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
