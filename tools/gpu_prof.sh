#!/bin/bash
# Perf sweep + ncu evidence for k_encode.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 python tools/perf.py --iters 20 --json gpurun_out/perf_${TAG}.json > gpurun_out/perf_${TAG}.log 2>&1
echo "perf rc=$?" >> gpurun_out/perf_${TAG}.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 5 --warmup 3 --cpu-seconds 1 > gpurun_out/launches_bench_${TAG}.log 2>&1
for W in c1_131k corpus_256m; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -s 2 -c 1 \
    -o gpurun_out/prof_${TAG}_${W} -f python tools/perf.py --only $W --iters 1 --warmup 1 --no-flush > gpurun_out/ncu_${TAG}_${W}.log 2>&1
  echo "ncu $W rc=$?" >> gpurun_out/ncu_${TAG}_${W}.log
done
cat gpurun_out/perf_${TAG}.log
