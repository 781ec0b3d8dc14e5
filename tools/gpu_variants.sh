#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for L in ${LIBS:-libgpubpe.so libgpubpe_nw24.so libgpubpe_nw16.so}; do echo "== $L"; GPUBPE_LIB=$L timeout 300 python tools/perf.py --iters 20 --only ${ONLY:-c1_8k,c1_131k,c3_1m,c2_4096x512,corpus_256m} 2>&1 | tail -6; done
