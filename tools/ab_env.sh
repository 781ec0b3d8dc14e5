#!/bin/bash
# A/B timing of environment knobs on one build, interleaved:
#   ENVS="GPUBPE_PREFETCH=0 GPUBPE_PREFETCH=1" WL=c1_8k,c1_131k bash tools/ab_env.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2; do
  for E in ${ENVS}; do
    echo "== $E (rep $rep)"
    env $E timeout 300 python tools/perf.py --iters ${ITERS:-30} --only ${WL:-c1_8k,c1_131k} 2>&1 | grep -v "^perf"
    if [ -n "$E2E" ]; then env $E timeout 300 python tools/e2e_breakdown.py 2>&1 | grep -E "tokenize_batch"; fi
  done
done
