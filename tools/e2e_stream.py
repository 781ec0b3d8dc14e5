"""Streamed gpubpe_encode_host on a synthetic corpus, per-phase host timing (GPUBPE_HOSTTIME=1)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GPUBPE_HOSTTIME", "1")
import torch  # noqa
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
data, offs = synth_corpus.corpus_docs(mb << 20, seed=0)
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
if os.environ.get("PINNED_INPUT"):
    pd = bpe.pinned_empty(data.size)
    pd[:] = data
    data = pd
for i in range(4):
    t0 = time.perf_counter()
    ids, oo, st, ms = enc.encode_packed_host(data, offs, tok.config.max_seq_len, tok.config.chunk_budget)
    t = time.perf_counter() - t0
    print("python encode_packed_host %.1f ms, %d ids, %.2f Gtok/s" % (t * 1e3, len(ids), len(ids) / t / 1e9), file=sys.stderr)
    del ids
