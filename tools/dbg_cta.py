"""Debug: CTA-level timeline of one encode (globaltimer stamps, GPUBPE_DEBUG=8)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.dirname(__file__))
os.environ["GPUBPE_DEBUG"] = "8"
import torch  # noqa
import perf
name = sys.argv[1] if len(sys.argv) > 1 else "c1_8k"
data, offs, _ = perf.workloads()[name]()
import fixtures, paper_2603_02597_b200 as bpe
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
enc = tok.device_encoder(0)
d = torch.from_numpy(data.copy()).cuda(); o = torch.from_numpy(offs).cuda()
out = torch.empty(len(data), dtype=torch.int32, device="cuda"); oo = torch.empty(len(offs), dtype=torch.int64, device="cuda")
enc.set_profiling(True)
for i in range(4):
    os.environ["GPUBPE_DEBUG_OUT"] = "/tmp/dbg.bin" if i == 3 else ""
    if os.environ.get("FLUSH") and i == 3:
        torch.empty(256 << 20, dtype=torch.uint8, device="cuda").fill_(1)
        torch.cuda.synchronize()
    enc.encode_into(d, o, out, oo, 1 << 40, 1 << 40)
    torch.cuda.synchronize()
print("kernel (events) %.1f us" % (1000 * enc.kernel_ms()))
h = np.fromfile("/tmp/dbg.bin", dtype=np.uint64).astype(np.int64)
cta = h[:1024].reshape(256, 4)[:148]
t0 = cta[:, 0].min()
for k, n in enumerate(["prologue done", "phase A done (warp 0)", "barrier exit", "kernel end"]):
    v = (cta[:, k] - t0) / 1e3
    print("%-24s min %6.1f p50 %6.1f max %6.1f us" % (n, v.min(), np.median(v), v.max()))
pl = h[36864:36864 + 4 * 148].reshape(148, 4)
for k, n in enumerate(["ids stored (last warp)", "placement base known", "slots discarded (last)"]):
    v = (pl[:, k] - t0) / 1e3
    print("%-24s min %6.1f p50 %6.1f max %6.1f us" % (n, v.min(), np.median(v), v.max()))
te = h[1024:1024 + 2 * 4096].reshape(4096, 2)
te = te[te[:, 1] > 0]
if len(te):
    v = (te[:, 1] - t0) / 1e3
    print("%-24s min %6.1f p50 %6.1f max %6.1f us (%d tiles)" % ("tile end", v.min(), np.median(v), v.max(), len(te)))
    v = (te[:, 0] - t0) / 1e3
    print("%-24s min %6.1f p50 %6.1f max %6.1f us" % ("tile start", v.min(), np.median(v), v.max()))
pp = h[38000:38000 + 4 * 148].reshape(148, 4)
for k, n in enumerate(["place_range_one entry", "tile words loaded (last warp)"]):
    v = pp[:, k]
    v = v[v > 0]
    if len(v):
        v = (v - t0) / 1e3
        print("%-24s min %6.1f p50 %6.1f max %6.1f us" % (n, v.min(), np.median(v), v.max()))
