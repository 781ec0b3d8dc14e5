"""Cold-start breakdown: parse vocab/merges, build the host tables, create the device context."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
t0 = time.perf_counter()
import torch  # noqa
torch.cuda.init(); torch.empty(1, device="cuda")
t1 = time.perf_counter()
import fixtures
import paper_2603_02597_b200 as bpe
t2 = time.perf_counter()
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
t3 = time.perf_counter()
enc = tok.device_encoder(0)
torch.cuda.synchronize()
t4 = time.perf_counter()
ids = bpe.tokenize_batch([b"hello world"], tok).token_ids[0]
t5 = time.perf_counter()
print("torch+cuda init %.0f ms | import %.0f ms | Tokenizer.from_files %.0f ms | device context %.0f ms | first call %.1f ms"
      % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t5 - t4) * 1e3))
