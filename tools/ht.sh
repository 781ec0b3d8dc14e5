# host-path timing lines (GPUBPE_HOSTTIME) of 60 tokenize_batch calls on the 131k sequence
cd ${GRAFT_REPO_ROOT:-/root/repo}
env ${EXTRA} python -c '
import sys; sys.path.insert(0,"."); sys.path.insert(0,"tools")
import fixtures, synth_corpus, paper_2603_02597_b200 as bpe
spec = fixtures.synth_sizes()["c1_131k"]; doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
W = 1 << 40
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=W, chunk_budget=W))
for _ in range(60): bpe.tokenize_batch([doc], tok)
' 2>&1 | grep -E "encode_impl|encode_host|timeline|overlap|sync:" | tail -${TAILN:-12}
