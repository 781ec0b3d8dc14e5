#!/bin/bash
# Iteration session: smoke, GPU parity tests, perf sweep.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 180 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
tail -3 gpurun_out/smoke_${TAG}.log
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 ${PYTEST_ARGS:--x} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -15 gpurun_out/pytest_${TAG}.log
timeout 600 python tools/perf.py --iters 20 ${PERF_ARGS} --json gpurun_out/perf_${TAG}.json > gpurun_out/perf_${TAG}.log 2>&1; echo "perf rc=$?" >> gpurun_out/perf_${TAG}.log
cat gpurun_out/perf_${TAG}.log
if [ -n "$DIAG" ]; then
  for W in $DIAG; do echo "== $W (L2 flushed)"; FLUSH=1 timeout 120 python tools/dbg_cta.py $W 2>&1 | tail -10; done > gpurun_out/diag_${TAG}.txt 2>&1
  cat gpurun_out/diag_${TAG}.txt
fi
if [ -n "$CYCLES" ]; then
  make -s -C paper_2603_02597_b200/csrc stamps > /dev/null 2>&1 || echo "stamps build failed"
  for W in $CYCLES; do echo "== $W tile steps (stamps build, L2 flushed)"; FLUSH=1 timeout 120 python tools/dbg_cycles.py $W 2>&1 | tail -16; done > gpurun_out/cycles_${TAG}.txt 2>&1
  cat gpurun_out/cycles_${TAG}.txt
fi
