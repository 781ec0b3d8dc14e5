#!/bin/bash
# Evidence pass: GPU tests, smoke, 1-GPU bench, perf sweep, launch list, ncu
# full captures of the timed launch.  Outputs in gpurun_out/ (TAG-suffixed).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-round}
cp paper_2603_02597_b200/libgpubpe.so gpurun_out/lib_${TAG}.so
nvidia-smi -L > gpurun_out/smi_${TAG}.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -2 gpurun_out/pytest_${TAG}.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_${TAG}.log
timeout 900 python tools/perf.py --iters 20 --json gpurun_out/perf_${TAG}.json > gpurun_out/perf_${TAG}.log 2>&1; echo "perf rc=$?" >> gpurun_out/perf_${TAG}.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 5 --warmup 3 --cpu-seconds 1 > gpurun_out/launches_bench_${TAG}.log 2>&1
for W in ${WORKLOADS:-c1_131k corpus_256m}; do
  GPUBPE_PROFILE_TIMED=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_encode -c 1 \
    -o gpurun_out/prof_${TAG}_${W} -f python tools/perf.py --only $W --iters 1 --warmup 1 --no-flush > gpurun_out/ncu_${TAG}_${W}.log 2>&1
done
cat gpurun_out/perf_${TAG}.log; tail -3 gpurun_out/bench_${TAG}.log | cut -c1-600; tail -2 gpurun_out/bench_ref_${TAG}.log | cut -c1-400
