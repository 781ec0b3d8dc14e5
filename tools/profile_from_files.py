import os, sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch; torch.empty(1, device="cuda")
import fixtures, paper_2603_02597_b200 as bpe
for i in range(3):
    t = time.perf_counter(); tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths()); print("from_files %.1f ms" % ((time.perf_counter() - t) * 1e3))
pr = cProfile.Profile(); pr.enable()
tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
pr.disable(); pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
