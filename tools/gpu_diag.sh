#!/bin/bash
# Latency diagnostics: CTA timelines and per-step tile cycles (stamps build), warm and L2-flushed.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-diag}
make -s -C paper_2603_02597_b200/csrc stamps > /dev/null 2>&1 || echo "stamps build failed"
for W in ${WORKLOADS:-c1_8k c1_131k}; do
  for F in "" 1; do
    echo "=== $W flush=${F:-0} (CTA timeline, release build)"
    FLUSH=$F timeout 120 python tools/dbg_cta.py $W 2>&1 | tail -6
    echo "=== $W flush=${F:-0} (tile steps, stamps build)"
    FLUSH=$F timeout 120 python tools/dbg_cycles.py $W 2>&1 | tail -16
  done
done > gpurun_out/diag_${TAG}.txt 2>&1
cat gpurun_out/diag_${TAG}.txt
