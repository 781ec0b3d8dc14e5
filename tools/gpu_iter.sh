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
