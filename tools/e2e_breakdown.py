"""Where the end-to-end time of one tokenize_batch([131k-token doc]) goes."""
import ctypes, os, statistics, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.dirname(__file__))
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

def t(fn, k=200):
    for _ in range(5): fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(ts)

def craw():
    enc._lib.gpubpe_encode_host(enc._h, data.ctypes.data, n, offs.ctypes.data, 1, W, W, ids.ctypes.data,
                                oo.ctypes.data, ctypes.byref(nid), ctypes.byref(ms), s.cuda_stream)
print("pack_texts          %8.1f us" % t(lambda: pack_texts([doc])))
ids_pin = bpe.pinned_empty(4 * n).view(np.uint32)
def craw_pinned():
    enc._lib.gpubpe_encode_host(enc._h, data.ctypes.data, n, offs.ctypes.data, 1, W, W, ids_pin.ctypes.data,
                                oo.ctypes.data, ctypes.byref(nid), ctypes.byref(ms), s.cuda_stream)
print("C encode_host, pinned ids %6.1f us" % t(craw_pinned))
print("C encode_host       %8.1f us  (kernel %.1f us)" % (t(craw), ms.value * 1000))
print("encode_packed_host  %8.1f us" % t(lambda: enc.encode_packed_host(data, offs, W, W)))
print("tokenize_batch      %8.1f us" % t(lambda: bpe.tokenize_batch([doc], tok)))
d = torch.from_numpy(data.copy()).cuda(); o = torch.from_numpy(offs).cuda()
out = torch.empty(n, dtype=torch.int32, device="cuda"); oo2 = torch.empty(2, dtype=torch.int64, device="cuda")
def dev(): enc.encode_into(d, o, out, oo2, W, W); torch.cuda.synchronize()
print("device encode+sync  %8.1f us" % t(dev))
hp = torch.empty(n, dtype=torch.uint8, pin_memory=True)
def h2d(): d.copy_(hp, non_blocking=True); torch.cuda.synchronize()
print("H2D 588KB pinned    %8.1f us" % t(h2d))
hq = torch.empty(4 * 131072, dtype=torch.uint8, pin_memory=True); dq = torch.empty(4 * 131072, dtype=torch.uint8, device="cuda")
def d2h(): hq.copy_(dq, non_blocking=True); torch.cuda.synchronize()
print("D2H 512KB pinned    %8.1f us" % t(d2h))
buf = np.empty(n, np.uint8)
print("memcpy 588KB        %8.1f us" % t(lambda: np.copyto(buf, data)))
def sync(): torch.cuda.synchronize()
print("empty sync          %8.1f us" % t(sync))
def enq(): enc.encode_into(d, o, out, oo2, W, W)
for _ in range(5): enq()
torch.cuda.synchronize()
ts = []
for _ in range(100):
    t0 = time.perf_counter(); enq(); ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("enqueue encode_into %8.1f us (host time per call, no sync)" % (1e6 * statistics.median(ts)))
raw_enq = []
for _ in range(100):
    t0 = time.perf_counter()
    enc._lib.gpubpe_encode(enc._h, d.data_ptr(), n, o.data_ptr(), 1, W, W, out.data_ptr(), oo2.data_ptr(), s.cuda_stream)
    raw_enq.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("enqueue C gpubpe_encode %6.1f us" % (1e6 * statistics.median(raw_enq)))
pin = bpe.pinned_empty(n)
pin[:] = data
print("encode_packed_host (pinned input) %8.1f us" % t(lambda: enc.encode_packed_host(pin, offs, W, W)))
