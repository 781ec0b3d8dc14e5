#!/bin/bash
# One ncu --set full capture of the timed k_encode launch of a workload (tools/perf.py).
#   TAG=x W=corpus_256m bash tools/ncu_one.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp paper_2603_02597_b200/libgpubpe.so gpurun_out/lib_${TAG}.so
GPUBPE_PROFILE_TIMED=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:${K:-k_encode} -c 1 \
  -o gpurun_out/prof_${TAG}_${W} -f python tools/perf.py --only $W --iters 1 --warmup 1 --no-flush > gpurun_out/ncu_${TAG}_${W}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}_${W}.log
