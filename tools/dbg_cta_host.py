"""Debug: CTA timeline of one gpubpe_encode_host call (input arriving while the kernel runs)."""
import os, sys, ctypes
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ["GPUBPE_DEBUG"] = "8"
import torch  # noqa
import perf, fixtures
import paper_2603_02597_b200 as bpe
name = sys.argv[1] if len(sys.argv) > 1 else "c1_131k"
data, offs, _ = perf.workloads()[name]()
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
W = 1 << 40
for i in range(4):
    os.environ["GPUBPE_DEBUG_OUT"] = "/tmp/dbg.bin" if i == 3 else ""
    enc.encode_packed_host(data, offs, W, W)
h = np.fromfile("/tmp/dbg.bin", dtype=np.uint64).astype(np.int64)
cta = h[:1024].reshape(256, 4)[:148]
t0 = cta[:, 0].min()
for k, n in enumerate(["prologue done", "phase A done (warp 0)", "barrier exit", "kernel end"]):
    v = (cta[:, k] - t0) / 1e3
    print("%-24s min %6.1f p50 %6.1f max %6.1f us" % (n, v.min(), np.median(v), v.max()))
tiles = h[1024:1024 + 2 * 4096].reshape(4096, 2)
tiles = tiles[tiles[:, 0] > 0]
st = (tiles[:, 0] - t0) / 1e3
en = (tiles[:, 1] - t0) / 1e3
print("tile start  p10 %6.1f p50 %6.1f p90 %6.1f max %6.1f us" % tuple(np.percentile(st, [10, 50, 90, 100])))
print("tile end    p10 %6.1f p50 %6.1f p90 %6.1f max %6.1f us" % tuple(np.percentile(en, [10, 50, 90, 100])))
print("tile dur    p10 %6.1f p50 %6.1f p90 %6.1f max %6.1f us" % tuple(np.percentile(en - st, [10, 50, 90, 100])))
