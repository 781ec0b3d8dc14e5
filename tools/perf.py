#!/usr/bin/env python3
"""Device-time sweep of the encode kernel over the SURVEY §8(d) workloads.

  python tools/perf.py [--iters K] [--only name,...] [--memo 0|1] [--json out.json]

For each workload: input resident in HBM, W warm-ups, then K encodes each
preceded by an L2 flush (256 MiB write); CUDA events on the launching stream
around the encode only.  Prints p50 kernel time, tokens/s, input GB/s and the
HBM-roofline fraction of the algorithmic bytes (n_bytes + 4 n_ids + 16 (n_docs+1)).
Also the profiling driver for ncu (--iters 3 --no-flush).
"""

from __future__ import annotations

import argparse
import os
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

WHOLE = 1 << 40


def workloads():
    import numpy as np

    import fixtures
    import synth_corpus

    sizes = fixtures.synth_sizes()

    def single(name):
        spec = sizes[name]
        doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
        return np.frombuffer(doc, np.uint8), np.array([0, len(doc)], np.int64), spec["tokens_whole"]

    def batch(n_docs, doc_bytes, seed):
        pool = np.frombuffer(synth_corpus.english_bytes(n_docs * doc_bytes + (1 << 20), seed), np.uint8)
        offs = np.arange(n_docs + 1, dtype=np.int64) * doc_bytes
        return pool[: n_docs * doc_bytes].copy(), offs, None

    def corpus(mb):
        data, offs = synth_corpus.corpus_docs(mb << 20, seed=0)
        return data, offs, None

    def adversarial(kind, n):
        rng = np.random.default_rng(0)
        if kind == "digits":
            d = rng.integers(48, 58, n, dtype=np.uint8)
        elif kind == "letters":
            d = rng.integers(97, 123, n, dtype=np.uint8)
        else:
            d = np.full(n, {"newlines": 10, "aaaa": 97}[kind], np.uint8)
        return d, np.array([0, n], np.int64), None

    def giant_docs(n_docs, doc_bytes):  # every document one digit giant
        rng = np.random.default_rng(1)
        d = rng.integers(48, 58, n_docs * doc_bytes, dtype=np.uint8)
        return d, np.arange(0, n_docs * doc_bytes + 1, doc_bytes, dtype=np.int64), None

    return {
        "c1_8k": lambda: single("c1_8k"),
        "c1_32k": lambda: single("c1_32k"),
        "c1_131k": lambda: single("c1_131k"),
        "c3_1m": lambda: single("c3_1m"),
        "c2_4096x512": lambda: batch(4096, 2300, 5),
        "corpus_256m": lambda: corpus(256),
        "adv_digits_1m": lambda: adversarial("digits", 1 << 20),
        "adv_letters_1m": lambda: adversarial("letters", 1 << 20),
        "adv_newlines_1m": lambda: adversarial("newlines", 1 << 20),
        "adv_aaaa_1m": lambda: adversarial("aaaa", 1 << 20),
        "adv_digit_docs_1000x10k": lambda: giant_docs(1000, 10000),
        "adv_digits_64k": lambda: adversarial("digits", 1 << 16),
        "adv_digit_docs_64x10k": lambda: giant_docs(64, 10000),
        "adv_digit_docs_1000x6k": lambda: giant_docs(1000, 6000),
        "adv_digits_6k": lambda: giant_docs(1, 6000),
        "adv_digits_7k": lambda: giant_docs(1, 7000),
        "adv_digits_600": lambda: giant_docs(1, 600),
        "adv_digits_200": lambda: giant_docs(1, 200),
        "adv_digits_400": lambda: giant_docs(1, 400),
        "adv_digit_docs_100x400": lambda: giant_docs(100, 400),
        "adv_digit_docs_4096x400": lambda: giant_docs(4096, 400),
        "adv_digit_docs_4096x800": lambda: giant_docs(4096, 800),
        "adv_digit_docs_2048x2000": lambda: giant_docs(2048, 2000),
        "adv_digits_2k": lambda: giant_docs(1, 2000),
        "adv_digits_4k": lambda: giant_docs(1, 4000),
        "adv_digit_docs_16384x200": lambda: giant_docs(16384, 200),
    }


def decode_row(name, enc, flush, peak, args):
    """decode_<workload>: device decode of that workload's ids (ids in HBM,
    bytes out in HBM); alg bytes = 4 n_ids + n_bytes + 16 (n_seqs+1)."""
    import numpy as np
    import torch

    wl = workloads()[name[len("decode_"):]]
    data, offs, _ = wl()
    dev = torch.device("cuda", 0)
    d_data = torch.from_numpy(data.copy()).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    ids = torch.empty(max(data.size, 1), dtype=torch.int32, device=dev)
    ioffs = torch.empty(len(offs), dtype=torch.int64, device=dev)
    enc.encode_into(d_data, d_offs, ids, ioffs, 8192, 8192)
    n_ids = int(ioffs[-1].item())
    ids = ids[:n_ids]
    out = torch.empty(data.size + 64, dtype=torch.uint8, device=dev)
    oo = torch.empty_like(ioffs)
    for _ in range(args.warmup):
        enc.decode_into(ids, ioffs, out, oo)
    got = out[: data.size].cpu().numpy()
    bad = np.flatnonzero(got != data)
    if bad.size:
        b = int(bad[0])
        print(f"{name}: {bad.size} bytes differ, first at {b} of {data.size}: got {bytes(got[b-8:b+24])!r} "
              f"want {bytes(data[b-8:b+24])!r}", flush=True)
    assert not bad.size, "decode round trip"
    times = []
    prof = os.environ.get("GPUBPE_PROFILE_TIMED")
    if prof:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    for _ in range(args.iters):
        if not args.no_flush:
            flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        enc.decode_into(ids, ioffs, out, oo)  # includes its one sync for the error/size check
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    ms = statistics.median(times)
    b_alg = 4 * n_ids + data.size + 16 * len(offs)
    row = {"workload": name, "bytes": int(data.size), "ids": n_ids, "p50_ms": ms,
           "tokens_per_s": n_ids / ms * 1e3, "alg_GBps": b_alg / ms / 1e6, "frac": b_alg / ms / 1e6 / peak}
    print(f"{name:18s} {n_ids:>11,d} ids -> {data.size:>11,d} B  p50 {ms*1e3:9.1f} us  "
          f"{row['tokens_per_s']/1e9:7.3f} Gtok/s  alg {row['alg_GBps']:8.1f} GB/s  frac {row['frac']:.4f}", flush=True)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    ap.add_argument("--memo", type=int, default=1)
    ap.add_argument("--strict", type=int, default=0,
                    help="1: the engines take one merge per pass (as for a table that is not well-formed)")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--json", default="")
    args = ap.parse_args()

    import numpy as np
    import torch

    import fixtures
    import paper_2603_02597_b200 as bpe

    peaks_p = ROOT / "MEASURED_PEAKS.json"
    peak = json.loads(peaks_p.read_text())["hbm_gbs"] if peaks_p.exists() else 6650.0
    tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(), bpe.BlockConfig(max_seq_len=WHOLE, chunk_budget=WHOLE))
    enc = tok.device_encoder(0, memo=bool(args.memo), strict=bool(args.strict))
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    wl = workloads()
    names = args.only.split(",") if args.only else list(wl)
    rows = []
    for name in [n for n in names if n.startswith("decode_")]:
        rows.append(decode_row(name, enc, flush, peak, args))
    names = [n for n in names if not n.startswith("decode_")]
    for name in names:
        rx = name.startswith("rx_")  # GPT-2 regex pre-tokenization mode (ids differ: no check)
        enc.set_mode(1 if rx else 0)
        data, offs, want = wl[name[3:] if rx else name]()
        if rx:
            want = None
        n = int(data.size)
        d_data = torch.from_numpy(data.copy()).to(dev)
        d_offs = torch.from_numpy(offs).to(dev)
        out_ids = torch.empty(n, dtype=torch.int32, device=dev)
        out_offs = torch.empty(len(offs), dtype=torch.int64, device=dev)
        for _ in range(args.warmup):
            enc.encode_into(d_data, d_offs, out_ids, out_offs, WHOLE, WHOLE, stream)
        st = enc.query()
        n_ids = int(out_offs[-1].item())
        if want is not None:
            assert n_ids == want or os.environ.get("GPUBPE_DEBUG"), (name, n_ids, want)
        times = []
        prof = os.environ.get("GPUBPE_PROFILE_TIMED")  # ncu --profile-from-start off
        if prof:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        for _ in range(args.iters):
            if not args.no_flush:
                flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            enc.encode_into(d_data, d_offs, out_ids, out_offs, WHOLE, WHOLE, stream)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
        ms = statistics.median(times)
        b_alg = n + 4 * n_ids + 16 * len(offs)
        row = {"workload": name, "bytes": n, "docs": len(offs) - 1, "ids": n_ids, "p50_ms": ms,
               "min_ms": min(times), "tokens_per_s": n_ids / ms * 1e3, "in_GBps": n / ms / 1e6,
               "alg_GBps": b_alg / ms / 1e6, "frac": b_alg / ms / 1e6 / peak,
               "engine_passes": st["engine_passes"], "memo_hits": st["memo_hits"],
               "short_merges": st["short_merges"], "medium": st["medium_segments"],
               "giant": st["giant_segments"], "segments": st["n_segments"]}
        rows.append(row)
        print(f"{name:18s} {n:>11,d} B {len(offs)-1:>6d} docs {n_ids:>10,d} ids  p50 {ms*1e3:9.1f} us  "
              f"{row['tokens_per_s']/1e9:7.3f} Gtok/s  in {row['in_GBps']:8.1f} GB/s  "
              f"frac {row['frac']:.4f}  passes {st['engine_passes']}", flush=True)
        del d_data, d_offs, out_ids, out_offs
    if args.json:
        Path(args.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
