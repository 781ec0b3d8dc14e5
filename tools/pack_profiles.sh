#!/bin/bash
# Copy one evidence round (tools/gpu_round.sh TAG=...) from gpurun_out/ into profiles/.
set -e
cd "$(dirname "$0")/.."
TAG=${1:?tag}
python tools/ncu_summary.py $TAG c1_131k corpus_256m pretok decode_corpus_256m > /dev/null
for W in c1_131k corpus_256m; do
  python tools/ncu_lines.py gpurun_out/prof_${TAG}_$W.ncu-rep --kernel k_encode --top 40 --lib gpurun_out/lib_${TAG}.so > profiles/${TAG}_${W}_lines.txt 2>&1
done
python tools/ncu_lines.py gpurun_out/prof_${TAG}_pretok.ncu-rep --kernel k_pretok --top 30 --lib gpurun_out/lib_${TAG}.so > profiles/${TAG}_pretok_lines.txt 2>&1
[ -f gpurun_out/prof_${TAG}_decode_corpus_256m.ncu-rep ] && python tools/ncu_lines.py gpurun_out/prof_${TAG}_decode_corpus_256m.ncu-rep --kernel k_decode_rows --top 30 --lib gpurun_out/lib_${TAG}.so > profiles/${TAG}_decode_lines.txt 2>&1
grep -h "^{" gpurun_out/bench_${TAG}.log > profiles/${TAG}_bench.jsonl
grep -h "^{" gpurun_out/bench_ref_${TAG}.log > profiles/${TAG}_bench_reference.jsonl
grep -h "^{" gpurun_out/bench_corpus_${TAG}.log gpurun_out/bench_c4_${TAG}.log > profiles/${TAG}_bench_corpus.jsonl
cp gpurun_out/perf_${TAG}.log profiles/${TAG}_perf.txt
cp gpurun_out/perf_rx_${TAG}.log profiles/${TAG}_perf_rx_decode.txt
cp gpurun_out/pytest_${TAG}.log profiles/${TAG}_pytest_gpu.log
cp gpurun_out/smoke_${TAG}.log profiles/${TAG}_smoke.log
cp gpurun_out/e2e_stream_${TAG}.log profiles/${TAG}_e2e_stream.txt
cp gpurun_out/e2e_breakdown_${TAG}.log profiles/${TAG}_e2e_breakdown.txt
cp gpurun_out/launches_${TAG}.csv profiles/${TAG}_launches.csv
python - "$TAG" <<'PY'
import csv, collections, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"profiles/{tag}_launches.csv")))
hdr, data = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            data[d["Kernel Name"][:60]].append(float(d["Metric Value"].replace(",", "")))
tot = sum(sum(v) for v in data.values())
out = ["ncu --metrics gpu__time_duration.sum --clock-control none over `python bench.py --steps 5 --warmup 3 --cpu-seconds 1` (ns)",
       "cold-cache, serialised launches: compare shares, not absolutes; the fill kernel is the bench's L2 flush"]
for k, v in data.items():
    out.append(f"{k:60s} launches {len(v):5d}  total {sum(v):12.1f}  share {100*sum(v)/tot:5.1f}%  mean {sum(v)/len(v):10.1f}")
open(f"profiles/{tag}_launches_summary.txt", "w").write("\n".join(out) + "\n")
PY
ls profiles/ | grep "^${TAG}" | wc -l
