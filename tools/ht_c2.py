"""Host timeline (GPUBPE_HOSTTIME=1) of gpubpe_encode_host_gather on C2 (4,096 x 2.3 KB)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ["GPUBPE_HOSTTIME"] = "1"  # (read once, at the first host call)
import torch  # noqa: F401
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
pool = synth_corpus.english_bytes(4096 * 2300 + (1 << 20), 5)
docs = [pool[i * 2300:(i + 1) * 2300] for i in range(4096)]
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
for _ in range(8):
    enc.encode_list_host(docs, 8192, 8192)
