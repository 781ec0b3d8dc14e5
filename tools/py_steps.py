"""Per-step host time of the single-document path (tokenize_batch -> encode_packed_host)."""
import ctypes, os, sys, time, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
from paper_2603_02597_b200 import device as dv, _native
spec = fixtures.synth_sizes()["c1_131k"]
doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
W = 1 << 40
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=W, chunk_budget=W))
enc = tok.device_encoder(0)
acc = {}
def lap(name, t):
    now = time.perf_counter_ns()
    acc.setdefault(name, []).append(now - t)
    return now
for it in range(300):
    t = time.perf_counter_ns()
    data = np.frombuffer(doc, dtype=np.uint8); n = data.size
    offs = np.array([0, n], np.int64)
    t = lap("frombuffer+offs", t)
    data2 = np.ascontiguousarray(data, dtype=np.uint8); offs2 = np.ascontiguousarray(offs, dtype=np.int64)
    t = lap("ascontiguousarray x2", t)
    buf = dv._RESULTS.take(4 * max(n, 1), enc._lib, enc.device)
    ids = buf.view(np.uint32)
    out_offs = np.zeros(2, dtype=np.int64)
    n_ids = ctypes.c_uint64(0); ms = ctypes.c_float(0.0)
    t = lap("take+view+zeros+ctypes objs", t)
    with enc._lock, torch.cuda.device(enc.device):
        t = lap("lock+device ctx enter", t)
        s = torch.cuda.current_stream(enc.device)
        t = lap("current_stream", t)
        a = (enc._h, dv._ptr(data2), n, dv._ptr(offs2), 1, W, W, dv._ptr(ids), dv._ptr(out_offs),
             ctypes.byref(n_ids), ctypes.byref(ms), s.cuda_stream)
        t = lap("args", t)
        rc = enc._lib.gpubpe_encode_host(*a)
        t = lap("native call", t)
        st = enc.query(s)
        t = lap("query", t)
    t = lap("ctx exit", t)
    r = dv._RESULTS.array(buf, np.uint32, n_ids.value)
    t = lap("result array", t)
    del r
for k, v in acc.items():
    print("%-30s %7.2f us" % (k, statistics.median(v[20:]) / 1e3))
