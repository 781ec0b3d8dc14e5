"""Breakdown of the device context build (Tokenizer.device_encoder on a fresh Tokenizer)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
torch.empty(1, device="cuda"); torch.cuda.synchronize()
import fixtures
import paper_2603_02597_b200 as bpe
from paper_2603_02597_b200.device import DeviceEncoder
from paper_2603_02597_b200.merge_table import rule_arrays
for rep in range(3):
    T = {}
    t = time.perf_counter()
    vocab_path, merges_path = fixtures.gpt2_paths()
    v = bpe.Vocab.from_file(vocab_path); T["Vocab.from_file"] = time.perf_counter() - t; t = time.perf_counter()
    from pathlib import Path
    rules = bpe.parse_merges(Path(merges_path).read_bytes(), v); T["parse_merges"] = time.perf_counter() - t; t = time.perf_counter()
    table = bpe.build_table(rules); T["build_table"] = time.perf_counter() - t; t = time.perf_counter()
    tok = bpe.Tokenizer(v, table); T["Tokenizer()"] = time.perf_counter() - t; t = time.perf_counter()
    arrs = rule_arrays(tok.table); T["rule_arrays"] = time.perf_counter() - t; t = time.perf_counter()
    vs = tok._vocab_strings(); T["_vocab_strings"] = time.perf_counter() - t; t = time.perf_counter()
    enc = DeviceEncoder(tok._base_ids, *arrs, *vs, device=0); torch.cuda.synchronize(); T["ctx_create (C)"] = time.perf_counter() - t; t = time.perf_counter()
    enc.set_vocab(*tok._decode_strings()); T["set_vocab"] = time.perf_counter() - t
    print(" | ".join("%s %.1f ms" % (k, 1e3 * x) for k, x in T.items()))
