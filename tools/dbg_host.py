"""Debug: CTA timeline of one host-path tokenize_batch (GPUBPE_DEBUG=8), e.g. the
overlapped launch whose tiles wait for their input pieces."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.dirname(__file__))
os.environ["GPUBPE_DEBUG"] = "8"
import fixtures, synth_corpus
import paper_2603_02597_b200 as bpe
name = sys.argv[1] if len(sys.argv) > 1 else "c1_131k"
spec = fixtures.synth_sizes()[name]
doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
W = 1 << 40
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=W, chunk_budget=W))
for i in range(6):
    os.environ["GPUBPE_DEBUG_OUT"] = "/tmp/dbg_host.bin" if i == 5 else ""
    r = bpe.tokenize_batch([doc], tok)
print("engine_time_ms %.1f us" % (1000 * r.engine_time_ms))
h = np.fromfile("/tmp/dbg_host.bin", dtype=np.uint64).astype(np.int64)
cta = h[:1024].reshape(256, 4)[:148]
t0 = cta[:, 0].min()
def show(n, v):
    v = v[v > 0]
    if len(v):
        v = (v - t0) / 1e3
        print("%-26s min %6.1f p50 %6.1f max %6.1f us" % (n, v.min(), np.median(v), v.max()))
show("prologue done", cta[:, 0])
pl = h[36864:36864 + 4 * 148].reshape(148, 4)
show("data ready (last warp)", pl[:, 3])
te = h[1024:1024 + 2 * 4096].reshape(4096, 2)
show("tile start", te[:, 0])
show("tile end", te[:, 1])
show("completion seen", cta[:, 2])
show("placement base known", pl[:, 1])
show("ids stored (last warp)", pl[:, 0])
show("kernel end", cta[:, 3])
