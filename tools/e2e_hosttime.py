"""Per-phase host timing of gpubpe_encode_host (GPUBPE_HOSTTIME=1) on the 131k sequence."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GPUBPE_HOSTTIME", "1")
import torch
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
from paper_2603_02597_b200.chunker import pack_texts

spec = fixtures.synth_sizes()["c1_131k"]
doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
W = 1 << 40
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=W, chunk_budget=W))
enc = tok.device_encoder(0)
data, offs = pack_texts([doc])
n = data.size
ids = np.empty(n, np.uint32); oo = np.zeros(2, np.int64)
nid = ctypes.c_uint64(); ms = ctypes.c_float()
s = torch.cuda.current_stream()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    enc._lib.gpubpe_encode_host(enc._h, data.ctypes.data, n, offs.ctypes.data, 1, W, W, ids.ctypes.data,
                                oo.ctypes.data, ctypes.byref(nid), ctypes.byref(ms), s.cuda_stream)
    print("kernel-event span %.1f us" % (ms.value * 1000), file=sys.stderr)
