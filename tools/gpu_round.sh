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
timeout 600 python bench.py --gpus 2 --steps 200 --warmup 5 --corpus-mb 1024 > gpurun_out/bench_g2_${TAG}.log 2>&1; echo "g2 rc=$?" >> gpurun_out/bench_g2_${TAG}.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_${TAG}.log
timeout 600 python bench.py --workload corpus_256m --steps 5 --warmup 3 > gpurun_out/bench_corpus_${TAG}.log 2>&1; echo "corpus rc=$?" >> gpurun_out/bench_corpus_${TAG}.log
timeout 900 python bench.py --workload corpus_10240m --steps 3 --warmup 3 > gpurun_out/bench_c4_${TAG}.log 2>&1; echo "c4 rc=$?" >> gpurun_out/bench_c4_${TAG}.log
timeout 900 python tools/perf.py --iters 20 --json gpurun_out/perf_${TAG}.json > gpurun_out/perf_${TAG}.log 2>&1; echo "perf rc=$?" >> gpurun_out/perf_${TAG}.log
timeout 300 python tools/perf.py --only rx_c1_131k,rx_c2_4096x512,rx_corpus_256m,decode_corpus_256m --iters 20 > gpurun_out/perf_rx_${TAG}.log 2>&1
PINNED_INPUT=1 timeout 300 python tools/e2e_stream.py 256 > gpurun_out/e2e_stream_${TAG}.log 2>&1
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown_${TAG}.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 5 --warmup 3 --cpu-seconds 1 > gpurun_out/launches_bench_${TAG}.log 2>&1
for W in ${WORKLOADS:-c1_131k corpus_256m}; do
  GPUBPE_PROFILE_TIMED=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_encode -c 1 \
    -o gpurun_out/prof_${TAG}_${W} -f python tools/perf.py --only $W --iters 1 --warmup 1 --no-flush > gpurun_out/ncu_${TAG}_${W}.log 2>&1
done
GPUBPE_PROFILE_TIMED=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_pretok -c 1 \
  -o gpurun_out/prof_${TAG}_pretok -f python tools/perf.py --only rx_corpus_256m --iters 1 --warmup 1 --no-flush > gpurun_out/ncu_${TAG}_pretok.log 2>&1
GPUBPE_PROFILE_TIMED=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_decode -c 1 \
  -o gpurun_out/prof_${TAG}_decode_corpus_256m -f python tools/perf.py --only decode_corpus_256m --iters 1 --warmup 1 --no-flush > gpurun_out/ncu_${TAG}_decode.log 2>&1
cat gpurun_out/perf_${TAG}.log; tail -3 gpurun_out/bench_${TAG}.log | cut -c1-600; tail -2 gpurun_out/bench_ref_${TAG}.log | cut -c1-400
