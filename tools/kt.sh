#!/bin/bash
# Per-kernel device times (ncu launch list, cold cache, serialised) of one perf.py
# workload for each library: LIBS="libgpubpe.so libprev.so" WL=rx_corpus_256m,rx_c2_4096x512 K=k_pretok bash tools/kt.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for W in ${WL//,/ }; do
for L in ${LIBS:-libgpubpe.so libprev.so}; do
  GPUBPE_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:${K:-k_} \
    --log-file gpurun_out/kt_$L.csv python tools/perf.py --only $W --iters ${ITERS:-5} --warmup 1 > /dev/null 2>&1
  python - "$L" "$W" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/kt_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
t = collections.defaultdict(list)
for r in rows[1:]:
    t[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) / 1e3)
for k, v in t.items():
    v.sort(); print(f"{sys.argv[2]:18s} {sys.argv[1]:16s} {k:24s} n={len(v):3d} median {v[len(v)//2]:9.1f} us  min {v[0]:9.1f}")
PY
done
done
