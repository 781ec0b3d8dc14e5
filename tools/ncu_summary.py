#!/usr/bin/env python3
"""Summarise k_encode ncu captures into profiles/ncu_summary.json (read by bench.py).

  python tools/ncu_summary.py TAG [WORKLOAD ...]

Reads gpurun_out/prof_<TAG>_<WORKLOAD>.ncu-rep (one --set full capture of the
timed launch, tools/gpu_ncu.sh) and records per workload: duration, DRAM bytes
read/written (the roofline `traffic`), instructions, issue activity, L2 hit
rate and the top stall reasons.  Also writes profiles/<TAG>_<WORKLOAD>.txt.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = {
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1}


def summarise(rep: Path) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, val = rows[0], rows[1], rows[2]
    out, stalls = {}, {}
    for i, n in enumerate(hdr):
        try:
            v = float(val[i])
        except ValueError:
            continue
        if n == "gpu__time_duration.sum":
            out["duration_us"] = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(units[i], 1.0)
        elif n in KEYS:
            out[KEYS[n]] = v * SCALE.get(units[i], 1)
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued") and v > 0:
            stalls[n.rsplit("stalled_", 1)[1]] = int(v)
    tot = sum(stalls.values()) or 1
    out["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    out["traffic_bytes"] = out.get("dram_read", 0) + out.get("dram_write", 0)
    return out


def main():
    tag, works = sys.argv[1], sys.argv[2:] or ["c1_131k", "corpus_256m"]
    prof = ROOT / "profiles"
    summ_p = prof / "ncu_summary.json"
    summ = json.loads(summ_p.read_text()) if summ_p.exists() else {}
    for w in works:
        rep = ROOT / "gpurun_out" / f"prof_{tag}_{w}.ncu-rep"
        if not rep.exists():
            print("missing", rep)
            continue
        s = summarise(rep)
        s["tag"] = tag
        summ[w] = s
        (prof / f"{tag}_{w}.txt").write_text(json.dumps(s, indent=1) + "\n")
        print(w, json.dumps(s))
    summ_p.write_text(json.dumps(summ, indent=1) + "\n")


if __name__ == "__main__":
    main()
