"""Debug: one encode with globaltimer stamps (GPUBPE_DEBUG=8), summary of CTA/tile timings."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.dirname(__file__))
import torch
import perf
name = sys.argv[1] if len(sys.argv) > 1 else "c1_8k"
os.environ["GPUBPE_DEBUG"] = os.environ.get("DBG", "8")
data, offs, _ = perf.workloads()[name]()
import fixtures, paper_2603_02597_b200 as bpe
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
d = torch.from_numpy(data.copy()).cuda(); o = torch.from_numpy(offs).cuda()
out = torch.empty(len(data), dtype=torch.int32, device="cuda"); oo = torch.empty(len(offs), dtype=torch.int64, device="cuda")
for i in range(3):
    os.environ["GPUBPE_DEBUG_OUT"] = "/tmp/dbg.bin" if i == 2 else ""
    enc.encode_into(d, o, out, oo, 1 << 40, 1 << 40)
    torch.cuda.synchronize()
h = np.fromfile("/tmp/dbg.bin", dtype=np.uint64).astype(np.int64)
cta = h[:1024].reshape(256, 4)[:148]
t0 = cta[:, 0].min()
print("CTA start spread us", (cta[:, 0].max() - t0) / 1e3)
print("phase A end (us after first start): min %.1f med %.1f max %.1f" % tuple(np.percentile((cta[:, 1] - t0) / 1e3, [0, 50, 100])))
print("barrier exit: min %.1f max %.1f" % ((cta[:, 2].min() - t0) / 1e3, (cta[:, 2].max() - t0) / 1e3))
print("kernel end: max %.1f" % ((cta[:, 3].max() - t0) / 1e3))
tl = h[1024:].reshape(-1, 2)
tl = tl[tl[:, 0] > 0]
dur = (tl[:, 1] - tl[:, 0]) / 1e3
st = (tl[:, 0] - t0) / 1e3
print("tiles", len(tl), "dur us: p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(dur, [50, 90, 100])))
print("tile start us: min %.1f p50 %.1f max %.1f" % tuple(np.percentile(st, [0, 50, 100])))
i = np.argmax(dur); print("slowest tile", i, "start", st[i], "dur", dur[i])
st = h[10240:10240 + 4096].reshape(512, 8)
st = st[st[:, 0] > 0]
pts = [(0, 1, "stage"), (1, 2, "cuts"), (2, 3, "docs"), (3, 5, "segments"), (5, 6, "scan+scatter")]
for i, j, n in pts:
    d = (st[:, j] - st[:, i]) / 1e3
    print("%-14s p50 %.2f p90 %.2f max %.2f us" % (n, *np.percentile(d, [50, 90, 100])))
mhz = st[:, 7] / ((st[:, 6] - st[:, 0]) / 1e3)
print("SM clock during tiles (MHz): p10 %.0f p50 %.0f p90 %.0f" % tuple(np.percentile(mhz, [10, 50, 90])))
