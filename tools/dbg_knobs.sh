cd $GRAFT_REPO_ROOT
for d in 0 1 2 4 7; do echo "== DEBUG=$d"; GPUBPE_DEBUG=$d timeout 300 python tools/perf.py --iters 20 --only c1_8k,c1_131k,corpus_256m 2>&1 | tail -3; done
