#!/bin/bash
# A/B timing of in-tree library builds (tools/build_rev.sh), interleaved:
#   LIBS="libgpubpe.so libprev.so" WL=c1_8k,c1_131k bash tools/ab.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2; do
  for L in ${LIBS:-libgpubpe.so libprev.so}; do
    echo "== $L (rep $rep)"
    GPUBPE_LIB=$L timeout 300 python tools/perf.py --iters ${ITERS:-30} --only ${WL:-c1_8k,c1_131k} 2>&1 | grep -v "^perf"
    if [ -n "$E2E" ]; then GPUBPE_LIB=$L timeout 300 python tools/e2e_breakdown.py 2>&1 | grep -E "tokenize_batch"; fi
  done
done
