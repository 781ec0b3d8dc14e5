"""Debug: decode round trips in sequence (small workload, then the corpus), checking encode and decode separately."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import fixtures, perf
import paper_2603_02597_b200 as bpe
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
ref = bpe.Tokenizer.from_files(*fixtures.gpt2_paths()).device_encoder(0, memo=True, strict=True)
wl = perf.workloads()
for name in sys.argv[1:] or ["c1_131k", "corpus_256m"]:
    data, offs, _ = wl[name]()
    d = torch.from_numpy(data.copy()).cuda(); o = torch.from_numpy(offs).cuda()
    ids = torch.empty(data.size, dtype=torch.int32, device="cuda"); io = torch.empty_like(o)
    enc.encode_into(d, o, ids, io, 8192, 8192)
    n = int(io[-1].item())
    ids2 = torch.empty(data.size, dtype=torch.int32, device="cuda"); io2 = torch.empty_like(o)
    ref.encode_into(d, o, ids2, io2, 8192, 8192)
    n2 = int(io2[-1].item())
    enc_ok = n == n2 and torch.equal(ids[:n], ids2[:n2]) and torch.equal(io, io2)
    ids = ids[:n]
    out = torch.empty(data.size + 64, dtype=torch.uint8, device="cuda"); oo = torch.empty_like(io)
    enc.decode_into(ids, io, out, oo)
    h = out[:data.size].cpu().numpy()
    bad = np.flatnonzero(h != data)
    print(name, "encode equal to strict ctx:", enc_ok, n, n2, "| decode mismatches", bad.size, bad[:3], flush=True)
    if bad.size:
        b = int(bad[0]); print("got ", bytes(h[b-8:b+24])); print("want", bytes(data[b-8:b+24]))
