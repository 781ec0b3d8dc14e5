#!/bin/bash
# ncu evidence: launch list + full capture of k_encode on the named workloads.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp paper_2603_02597_b200/libgpubpe.so gpurun_out/lib_${TAG:-iter}.so
TAG=${TAG:-iter}
for W in ${WORKLOADS:-c1_131k corpus_256m}; do
  GPUBPE_PROFILE_TIMED=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_encode -c 1 \
    -o gpurun_out/prof_${TAG}_${W} -f python tools/perf.py --only $W --iters 1 --warmup 1 --no-flush > gpurun_out/ncu_${TAG}_${W}.log 2>&1
  echo "ncu $W rc=$?" >> gpurun_out/ncu_${TAG}_${W}.log
  tail -2 gpurun_out/ncu_${TAG}_${W}.log
done
