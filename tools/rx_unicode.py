"""GPT-2 regex mode on non-ASCII text: time k_pretok + k_encode vs the default mode (16 MiB of mixed
CJK / Cyrillic / accented Latin / emoji prose-like text)."""
import os, sys, time, random
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
import fixtures
import paper_2603_02597_b200 as bpe

rng = random.Random(3)
words = ["漢字", "日本語", "テキスト", "мир", "привет", "café", "naïve", "😀", "über", "中文", "word", "the",
         "data", "1234", "ä", "ß", "東京", "北京", "статья", "résumé"]
parts = []
size = 0
while size < (16 << 20):
    w = rng.choice(words) + rng.choice([" ", " ", ", ", ". ", "\n", "'s "])
    parts.append(w)
    size += len(w.encode())
text = "".join(parts).encode()
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=1 << 40, chunk_budget=1 << 40))
enc = tok.device_encoder(0)
docs = [text[i:i + 8192] for i in range(0, len(text), 8192)]
data, offs = bpe.pack_texts(docs)
d = torch.from_numpy(data.copy()).cuda(); o = torch.from_numpy(offs).cuda()
out = torch.empty(d.numel(), dtype=torch.int32, device="cuda"); oo = torch.empty_like(o)
for mode in (0, 1):
    enc.set_mode(mode)
    for _ in range(3):
        enc.encode_into(d, o, out, oo, 1 << 40, 1 << 40)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        enc.encode_into(d, o, out, oo, 1 << 40, 1 << 40)
    e1.record(); e1.synchronize()
    print("mode %d: %.1f us per 16 MiB batch" % (mode, e0.elapsed_time(e1) * 100))
enc.set_mode(0)
enc.encode_into(d, o, out, oo, 1 << 40, 1 << 40)
st = enc.query()
print("stats:", {k: st[k] for k in ("n_bytes", "n_ids", "n_segments", "memo_hits", "medium_segments", "giant_segments", "engine_passes", "tiles")})
