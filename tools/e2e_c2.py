"""End-to-end tokenize_batch on C2 (4096 prompts of ~2.3 KB): host lists in, per-document id arrays out."""
import os, sys, time, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch  # noqa
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
from paper_2603_02597_b200.chunker import pack_texts
pool = synth_corpus.english_bytes(4096 * 2300 + (1 << 20), 5)
docs = [pool[i * 2300:(i + 1) * 2300] for i in range(4096)]
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
def t(fn, k=30):
    for _ in range(3): fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); r = fn(); ts.append(time.perf_counter() - t0); del r
    return 1e3 * statistics.median(ts)
data, offs = pack_texts(docs)
print("pack_texts          %7.3f ms" % t(lambda: pack_texts(docs)))
print("encode_packed_host  %7.3f ms" % t(lambda: enc.encode_packed_host(data, offs, 8192, 8192)))
ms = t(lambda: bpe.tokenize_batch(docs, tok))
n = sum(len(x) for x in bpe.tokenize_batch(docs, tok).token_ids)
print("tokenize_batch      %7.3f ms  (%d ids, %.2f Gtok/s e2e)" % (ms, n, n / ms / 1e6))
ids, oo, st, _ = enc.encode_packed_host(data, offs, 8192, 8192)
print("split (numpy idx)   %7.3f ms" % t(lambda: [ids[oo[i]:oo[i + 1]] for i in range(len(docs))]))
def split2():
    o = oo.tolist()
    return [ids[a:b] for a, b in zip(o, o[1:])]
print("split (tolist)      %7.3f ms" % t(split2))
print("join                %7.3f ms" % t(lambda: b"".join(docs)))
print("encode_list_host    %7.3f ms" % t(lambda: enc.encode_list_host(docs, 8192, 8192)))
import os
os.environ["GPUBPE_HOSTTIME"] = "1"
enc.encode_list_host(docs, 8192, 8192)
