#!/usr/bin/env python3
"""Aggregate an ncu SASS source page by CUDA source line.

  python tools/ncu_lines.py REPORT.ncu-rep [--kernel k_encode] [--top 40]

ncu's CUDA-source view needs the source on the profiling box; the SASS view
does not.  This maps SASS offsets to file:line with `nvdisasm -g` on the cubin
inside libgpubpe.so (built with -lineinfo) and sums warp-stall samples and
executed instructions per line.
"""

from __future__ import annotations

import argparse
import csv
import io
import re
import subprocess
import tempfile
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2603_02597_b200" / "libgpubpe.so"


def line_map(kernel: str, lib: Path = LIB, template: str = "") -> dict[int, tuple[str, int]]:
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(lib).resolve())], cwd=tmp, check=True,
                   capture_output=True)
    out: dict[int, tuple[str, int]] = {}
    for cub in tmp.glob("*.cubin"):
        txt = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True).stdout
        inside, cur = False, None
        for ln in txt.splitlines():
            if ln.startswith(".text."):
                # exact kernel (k_decode must not match k_decode_rows) and, for a
                # template, the instantiation the report profiled
                inside = re.search(r"_Z\d+" + re.escape(kernel) + r"(?![a-z_])", ln) is not None and (
                    not template or template in ln)
                continue
            if not inside:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (Path(m.group(1)).name, int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and cur:
                out[int(m.group(1), 16)] = cur
        if out:
            break
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", default="k_encode")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--lib", default=str(LIB), help="the .so the report was captured with")
    ap.add_argument("--reasons", action="store_true", help="per-line stall reasons (no barrier)")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ci = {n: hdr.index(n) for n in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                     "Instructions Executed")}
    body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    base = int(body[0][ci["Address"]], 16)
    # which template instantiation the report holds (k_encode<true> / <false>)
    names = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv", "--metrics", "launch__grid_size"],
                           capture_output=True, text=True).stdout
    template = ("ILb1E" if ("<true>" in names or "<1>" in names) else
                "ILb0E" if ("<false>" in names or "<0>" in names) else "")
    lm = line_map(args.kernel, Path(args.lib), template)
    reason_cols = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
    reasons = defaultdict(lambda: defaultdict(int))
    samples, insts = defaultdict(int), defaultdict(int)
    tot_s = tot_i = 0
    for r in body:
        off = int(r[ci["Address"]], 16) - base
        key = lm.get(off, ("?", 0))
        s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(r[ci["Instructions Executed"]] or 0)
        if args.reasons:
            s = sum(int(r[hdr.index(c)] or 0) for c in reason_cols if c != "stall_barrier")
            for c in reason_cols:
                v = int(r[hdr.index(c)] or 0)
                if v and c != "stall_barrier":
                    reasons[key][c[6:]] += v
        samples[key] += s
        insts[key] += n
        tot_s += s
        tot_i += n
    src_cache: dict[str, list[str]] = {}

    def text(f, l):
        if f not in src_cache:
            p = ROOT / "paper_2603_02597_b200" / "csrc" / f
            src_cache[f] = p.read_text().splitlines() if p.exists() else []
        lines = src_cache[f]
        return lines[l - 1].strip()[:70] if 0 < l <= len(lines) else ""

    print(f"total stall samples {tot_s}, warp instructions {tot_i}")
    print(f"{'file:line':28s} {'stall%':>7s} {'inst%':>7s}  source")
    for key in sorted(samples, key=lambda k: -samples[k])[: args.top]:
        f, l = key
        extra = ""
        if args.reasons:
            top = sorted(reasons[key].items(), key=lambda kv: -kv[1])[:3]
            extra = "  [" + " ".join(f"{k}:{v}" for k, v in top) + "]"
        print(f"{f + ':' + str(l):28s} {100 * samples[key] / max(tot_s, 1):6.2f}% "
              f"{100 * insts[key] / max(tot_i, 1):6.2f}%  {text(f, l)}{extra}")


if __name__ == "__main__":
    main()
