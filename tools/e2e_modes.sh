#!/bin/bash
# Host path variants of one 131k tokenize_batch (GPUBPE_HOSTMODE: 3 = ids stored by the
# kernel into mapped pinned memory, 0 = device ids + D2H + host copy-out).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for M in ${MODES:-3 0}; do
  echo "== GPUBPE_HOSTMODE=$M $EXTRA"
  env $EXTRA GPUBPE_HOSTMODE=$M timeout 300 python tools/e2e_breakdown.py 2>&1 | head -4
  env $EXTRA GPUBPE_HOSTMODE=$M GPUBPE_HOSTTIME=1 timeout 120 python -c '
import sys; sys.path.insert(0,"."); sys.path.insert(0,"tools")
import fixtures, synth_corpus, paper_2603_02597_b200 as bpe
spec = fixtures.synth_sizes()["c1_131k"]; doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
W = 1 << 40
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=W, chunk_budget=W))
for _ in range(40): bpe.tokenize_batch([doc], tok)
' 2>&1 | grep encode_host | tail -20 | python -c '
import sys, re, statistics
rows = [list(map(float, re.findall(r"(\d+\.\d+)", l))) for l in sys.stdin]
names = ["stage+h2d enqueue", "encode enqueue", "sync wait", "copy-out"]
print("  medians (tokenize_batch):", ", ".join("%s %.1f us" % (n, statistics.median(r[i] for r in rows)) for i, n in enumerate(names)))'
done
