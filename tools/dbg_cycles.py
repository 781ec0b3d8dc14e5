"""Debug: per-step cycle counts inside tiles (GPUBPE_DEBUG=8), for one encode of a workload."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.dirname(__file__))
os.environ["GPUBPE_DEBUG"] = "8"
os.environ.setdefault("GPUBPE_LIB", "libgpubpe_stamps.so")
import torch  # noqa
import perf
name = sys.argv[1] if len(sys.argv) > 1 else "c1_131k"
data, offs, _ = perf.workloads()[name]()
import fixtures, paper_2603_02597_b200 as bpe
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
d = torch.from_numpy(data.copy()).cuda(); o = torch.from_numpy(offs).cuda()
out = torch.empty(len(data), dtype=torch.int32, device="cuda"); oo = torch.empty(len(offs), dtype=torch.int64, device="cuda")
for i in range(3):
    os.environ["GPUBPE_DEBUG_OUT"] = "/tmp/dbg.bin" if i == 2 else ""
    if os.environ.get("FLUSH") and i == 2:
        torch.empty(256 << 20, dtype=torch.uint8, device="cuda").fill_(1)
        torch.cuda.synchronize()
    enc.encode_into(d, o, out, oo, 1 << 40, 1 << 40)
    torch.cuda.synchronize()
h = np.fromfile("/tmp/dbg.bin", dtype=np.uint64).astype(np.int64)
st = h[16384:16384 + 8 * 2048].reshape(2048, 8)
nt = int((st[:, 5] > 0).sum())
st = st[st[:, 5] > 0]
names = ["stage", "cuts", "segments", "packs", "scan+scatter", "docs/end"]
prev = np.zeros(nt)
for k, n in enumerate(names):
    d_ = st[:, k] - prev
    prev = st[:, k]
    print("%-13s cycles p50 %7.0f p90 %7.0f max %7.0f" % (n, *np.percentile(d_, [50, 90, 100])))
tot = st[:, 5]
print("tile total    cycles p50 %7.0f p90 %7.0f max %7.0f" % tuple(np.percentile(tot, [50, 90, 100])))
nm = st[:, 6]
for lo, hi in ((0, 0), (1, 2), (3, 4), (5, 99)):
    m = (nm >= lo) & (nm <= hi)
    if m.any():
        print("misses %d-%d: %4d tiles, total p50 %7.0f max %7.0f, packs p50 %7.0f" % (lo, hi, m.sum(), np.median(tot[m]), tot[m].max(), np.median((st[:, 3] - st[:, 2])[m])))
i = int(np.argmax(tot)); print("slowest tile", i, "misses", nm[i], "steps", np.diff(np.r_[0, st[i, :6]]))
p1 = st[:, 7] - st[:, 1]; p2 = st[:, 2] - st[:, 7]
print("segments pass1 p50 %7.0f p90 %7.0f | pass2 p50 %7.0f p90 %7.0f" % (*np.percentile(p1, [50, 90]), *np.percentile(p2, [50, 90])))
eng = h[32768:32776]
if eng[7]:
    names = (["setup+probe0", "segmented min", "winners+deaths", "neighbour shfl", "probes", "-"]
             if os.environ.get("SEQ", "1") == "1" else
             ["setup+probe0", "seg scan", "segmin+runs", "walks", "compaction", "re-probe"])
    print("warp engine: %d packs, %d passes (%.1f per pack)" % (eng[7], eng[6], eng[6] / eng[7]))
    for q, n in enumerate(names):
        print("  %-14s %8.0f cycles per pack  %6.0f per pass" % (n, eng[q] / eng[7], eng[q] / max(eng[6], 1)))
