#!/usr/bin/env python3
"""Benchmark: GPT-2 BPE encode tokens/sec on a 131k-token sequence (B200).

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
One step = one encode of one synthetic 131,072-token English-like sequence
(configs[1] of BASELINE.json, the metric's workload), whole-sequence semantics
(P-whole: no fixed-offset chunking), input resident in HBM.  L2 is flushed
(256 MiB write) before every timed step, outside the step's events.  With
N > 1 every rank encodes its own sequence (replicas; weak scaling, no
collective on the data path); value = all ranks' tokens / max-over-ranks time.
`--gpus N` without torchrun spawns the N ranks itself (torch.distributed.run);
with more ranks than GPUs the ranks share GPUs round-robin and talk over gloo.

The line also carries: e2e (same metric through the public API,
tokenize_batch, with host bytes in and host ids out), roofline (k_encode,
the only kernel, HBM-bound), cpu_baseline (the CPU oracle port of the
reference's sequential engine on this host), clocks (NVML during the timed
region), gpu_launches, and "corpus": the C4 configuration (BASELINE.json
configs[4]) -- a synthetic corpus (default 10 GiB, --corpus-mb) sharded by
document across the N ranks (strong scaling: each rank generates and encodes
only its shard), device-resident whole-box tokens/s, its HBM roofline
(N x peak), end to end through the host API, and a multi-core CPU baseline.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

WORKLOAD = "c1_131k"
METRIC = "GPT-2 BPE encode tokens/sec at 131k-token seqs; p50 latency per sequence"
UNIT = "tokens/s"
WHOLE = 1 << 40  # max_seq_len = chunk_budget beyond any input: P-whole


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default=WORKLOAD)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--corpus-mb", type=int, default=10240,
                    help="size of the sharded-corpus leg (C4); 0 skips it")
    return ap.parse_args()


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` run directly (no torchrun): launch N ranks through
    torch.distributed.run on 127.0.0.1 with the same arguments; rank 0 prints
    the line.  Returns the launcher's exit code."""
    import socket
    import subprocess

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def load_workload(name: str):
    import fixtures
    import synth_corpus

    spec = fixtures.synth_sizes()[name]
    doc = synth_corpus.english_bytes(spec["n_bytes"], spec["seed"])
    return doc, spec


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # pragma: no cover - NVML is in the image
            self._nv = None
            self.error = str(exc)
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                get = getattr(self._nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self._nv.nvmlDeviceGetCurrentClocksThrottleReasons
                mask = get(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._nv:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self) -> dict:
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ shared


def workload_config(args, world: int, n_bytes: int, n_ids: int) -> dict:
    """The `config` both arms print (identical keys and values)."""
    return {"workload": args.workload, "bytes": int(n_bytes), "tokens": int(n_ids), "semantics": "P-whole",
            "docs_per_gpu": 1, "l2": "flushed (256 MiB write) before every step",
            "parallelism": f"replicas x{world}"}


def peaks() -> dict:
    f = ROOT / "MEASURED_PEAKS.json"
    return json.loads(f.read_text()) if f.exists() else {}


def ncu_summary(workload: str) -> dict:
    prof = ROOT / "profiles" / "ncu_summary.json"
    return json.loads(prof.read_text()).get(workload, {}) if prof.exists() else {}


# The paper's published number for this metric (BASELINE.md Table 1):
# GPU-Opt encodes a 131,072-token sequence in 53.4 ms on an RTX 4070, end to end
# (host text in, host ids out), so vs_baseline divides our end-to-end value by it.
PAPER_131K_TOKS = 131072 / 53.4e-3


# ------------------------------------------------------------------ reference arm


def as_shipped_reference(doc: bytes, seconds: float = 20.0) -> dict | None:
    """Context only: the as-shipped pure-Python reference (`lanebpe`, installed
    unmodified into baseline/_ref) through its public API, tokenize_batch(...,
    "sequential", workers=os.cpu_count()), on a prefix of the workload sized
    to ~`seconds` of CPU time.  None when baseline/_ref is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "lanebpe" / "__init__.py").exists():
        return None
    import fixtures

    sys.path.insert(0, str(ref))
    try:
        import lanebpe
    finally:
        sys.path.remove(str(ref))
    cores = os.cpu_count() or 1
    tok = lanebpe.Tokenizer.from_files(*fixtures.gpt2_paths(),
                                       lanebpe.BlockConfig(max_seq_len=WHOLE, chunk_budget=WHOLE))
    probe = doc[:4096]
    t0 = time.perf_counter()
    lanebpe.tokenize_batch([probe], tok, "sequential", workers=cores)
    rate = len(probe) / max(time.perf_counter() - t0, 1e-9)
    cut = int(min(len(doc), max(4096, rate * seconds)))
    sample = doc[:cut]
    t0 = time.perf_counter()
    res = lanebpe.tokenize_batch([sample], tok, "sequential", workers=cores)
    dt = time.perf_counter() - t0
    toks = len(res.token_ids[0])
    return {"value": toks / dt, "unit": UNIT, "cores": cores, "kind": "reference (as shipped, pure Python)",
            "sample": f"first {cut} of {len(doc)} bytes of {WORKLOAD} ({toks} ids), P-whole, one "
                      f"tokenize_batch call in {dt:.2f} s (one P-whole sequence is one chunk: one core works)",
            "lanebpe": str(ref)}


def run_reference(args, rank, world):
    """The reference arm: the reference's CPU path on this host's cores -- the
    oracle port (oracle/) of sequential_bpe + tokenize_batch (pinned to the
    reference's goldens; ~45x faster than the as-shipped Python, whose number
    rides along as `as_shipped` context).  Rank 0 only."""
    if rank != 0:
        return
    from oracle.oracle import OracleEncoder, default_threads, load_tables
    import fixtures
    import numpy as np

    doc, spec = load_workload(args.workload)
    orc = OracleEncoder.from_tables(load_tables(*fixtures.gpt2_paths()))
    threads = default_threads()
    data = np.frombuffer(doc, dtype=np.uint8)
    # size each step so the whole run stays within ~150 s
    t0 = time.perf_counter()
    ids, _, _ = orc.encode_packed(data, np.array([0, len(doc)]), WHOLE, WHOLE, threads)
    est = time.perf_counter() - t0
    n = len(doc)
    frac = min(1.0, 150.0 / max(1e-9, est * (args.steps + args.warmup)))
    cut = max(1024, int(n * frac))
    sample = data[:cut]
    offs = np.array([0, cut], dtype=np.int64)
    for _ in range(args.warmup):
        orc.encode_packed(sample, offs, WHOLE, WHOLE, threads)
    times, toks = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out, _, _ = orc.encode_packed(sample, offs, WHOLE, WHOLE, threads)
        times.append(time.perf_counter() - t0)
        toks = len(out)
    total = sum(times)
    value = toks * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / len(times),
        "p50_ms": 1000 * statistics.median(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8->u32", "data": "synthetic",
        "config": workload_config(args, world, n, len(ids)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"first {cut} of {n} bytes of {args.workload} per step; oracle port "
                                   "of engines.py:269-335 sequential_bpe through the batch pipeline with "
                                   f"{threads} threads (one P-whole sequence is one chunk, so one works)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["as_shipped"] = as_shipped_reference(doc)
    except Exception as exc:  # context only: never fail the arm
        line["as_shipped"] = {"error": str(exc)[:200]}
    print(json.dumps(line), flush=True)


def cpu_baseline(doc, seconds: float) -> dict:
    from oracle.oracle import OracleEncoder, load_tables
    import fixtures
    import numpy as np

    orc = OracleEncoder.from_tables(load_tables(*fixtures.gpt2_paths()))
    data = np.frombuffer(doc, dtype=np.uint8)
    offs = np.array([0, len(doc)], dtype=np.int64)
    times, toks = [], 0
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or not times:
        t0 = time.perf_counter()
        out, _, _ = orc.encode_packed(data, offs, WHOLE, WHOLE, 1)
        times.append(time.perf_counter() - t0)
        toks = len(out)
    return {"value": toks / statistics.median(times), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{len(times)} x whole {WORKLOAD} sequence ({len(doc)} B -> {toks} ids), P-whole, "
                      "oracle port of the reference sequential engine (engines.py:269-335), 1 thread, "
                      "median run"}


# ------------------------------------------------------------------ corpus (C4)


def corpus_leg(args, mb: int, rank, world, local, dist, steps: int, warmup: int) -> dict | None:
    """BASELINE.json configs[4]: a synthetic corpus of `mb` MiB (documents of
    log-uniform 1-64 KiB) sharded by document across the ranks -- each rank
    generates and encodes ONLY its byte-balanced shard (strong scaling, no
    collective on the data path; NCCL/gloo only for the barrier and the
    max-over-ranks time).  P-default semantics.  Returns rank 0's dict."""
    import numpy as np
    import torch

    import fixtures
    import synth_corpus
    import paper_2603_02597_b200 as bpe
    from paper_2603_02597_b200 import device as bpe_device

    data, offs, (d0, d1), n_docs_all = synth_corpus.corpus_shard(mb << 20, rank, world, seed=0)
    n = len(data)
    tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
    enc = tok.device_encoder(local)
    dev = torch.device("cuda", local)
    cfg = tok.config
    d_data = torch.from_numpy(data).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    out_ids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    out_offs = torch.empty(len(offs), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    enc.set_profiling(True)
    for _ in range(warmup):
        enc.encode_into(d_data, d_offs, out_ids, out_offs, cfg.max_seq_len, cfg.chunk_budget, stream)
    torch.cuda.synchronize()
    n_ids = int(out_offs[-1].item()) if d1 > d0 else 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    kern = []
    with ClockSampler(local) as clocks:
        ev[0].record(stream)
        for _ in range(steps):
            enc.encode_into(d_data, d_offs, out_ids, out_offs, cfg.max_seq_len, cfg.chunk_budget, stream)
        ev[1].record(stream)
        torch.cuda.synchronize()
        kern.append(enc.kernel_ms())  # the last launch's k_encode time
    ms = ev[0].elapsed_time(ev[1])
    enc.set_profiling(False)
    del d_data, out_ids
    torch.cuda.empty_cache()
    # end to end through the public host API: pinned host bytes in, host ids out
    # (gpubpe_encode_host; a shard this large streams through its two-slot pipeline)
    h_data = bpe.pinned_empty(n, local)
    h_data[:] = data
    e2e_steps = 2
    res = enc.encode_packed_host(h_data, offs, cfg.max_seq_len, cfg.chunk_budget)
    assert len(res[0]) == n_ids, (len(res[0]), n_ids)
    del res
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = enc.encode_packed_host(h_data, offs, cfg.max_seq_len, cfg.chunk_budget)
        del res
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    cpu = None
    if rank == 0:  # multi-core CPU baseline on a bounded sample of this corpus
        cpu = corpus_cpu_baseline(data, offs, n_ids / max(n, 1))
    t = torch.tensor([ms, e2e_s, float(n_ids), float(n)], dtype=torch.float64, device=dev)
    if dist:
        if dist.get_backend() == "gloo":
            t = t.cpu()
        tm = t[0:2].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        tot = t[2:4].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms, e2e_s, total_ids, total_bytes = float(tm[0]), float(tm[1]), int(tot[0]), int(tot[1])
    else:
        total_ids, total_bytes = n_ids, n
    if rank != 0:
        return None
    step_ms = ms / steps
    p = peaks()
    peak = float(p.get("hbm_gbs", 6650.0))
    b_alg = total_bytes + 4 * total_ids + 16 * (n_docs_all + 1)
    achieved = b_alg / (step_ms / 1e3) / 1e9
    return {
        "metric": "GPT-2 BPE encode tokens/sec, synthetic corpus sharded by document (whole box)",
        "value": total_ids / (step_ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "config": {"workload": f"corpus_{mb}m", "bytes": total_bytes, "docs": n_docs_all, "tokens": total_ids,
                   "semantics": "P-default", "l2": f"input {mb} MiB >> L2 (not flushed)",
                   "parallelism": f"documents sharded x{world} (each rank generates only its shard)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                     "frac": achieved / (peak * world), "traffic": ncu_summary(f"corpus_{mb}m").get("traffic_bytes"),
                     "kernel": "k_encode", "alg_bytes_per_step": b_alg, "k_encode_ms_last": kern[-1],
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs x {world} GPU(s)" if p else "fallback"},
        "e2e": {"value": total_ids / e2e_s, "unit": UNIT, "h2d_bytes_per_step": total_bytes + 8 * (n_docs_all + 1),
                "d2h_bytes_per_step": 4 * total_ids + 8 * (n_docs_all + 1), "steps": e2e_steps,
                "input": "pinned host bytes",
                "output": ("host ids, pooled pinned result buffer" if 4 * n <= bpe_device._POOLED_MAX
                           else "host ids, pageable result buffer (staged through pinned slots)"),
                "path": "encode_packed_host (gpubpe_encode_host), wall clock, max over ranks"},
        "cpu_baseline": cpu, "clocks": clocks.summary(), "gpu_launches": steps,
    }


def corpus_cpu_baseline(data, offs, ids_per_byte: float, sample_bytes: int = 48 << 20) -> dict:
    """The reference's pipeline (oracle port, one pthread per host core over
    whole documents: the multi-process best case of BASELINE.md section 3) on
    the first documents of this shard up to `sample_bytes`."""
    import numpy as np

    from oracle.oracle import OracleEncoder, default_threads, load_tables
    import fixtures

    k = int(np.searchsorted(offs, min(sample_bytes, int(offs[-1])), side="right")) - 1
    k = max(k, 1)
    sample, so = data[: int(offs[k])], offs[: k + 1]
    orc = OracleEncoder.from_tables(load_tables(*fixtures.gpt2_paths()))
    threads = default_threads()
    t0 = time.perf_counter()
    ids, _, _ = orc.encode_packed(sample, so, 8192, 8192, threads)
    dt = time.perf_counter() - t0
    return {"value": len(ids) / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {k} documents ({int(so[-1])} B -> {len(ids)} ids) of the corpus, P-default, oracle "
                      f"port of tokenize_batch + sequential_bpe with {threads} threads over documents, {dt:.2f} s; "
                      "whole-corpus time extrapolates linearly in bytes"}


# ------------------------------------------------------------------ our arm (standalone corpus line)


def run_corpus(args, rank, world, local, dist):
    """--workload corpus_<MB>m: the corpus leg as its own line."""
    mb = int(args.workload.split("_")[1].rstrip("m"))
    line = corpus_leg(args, mb, rank, world, local, dist, args.steps, args.warmup)
    if rank == 0:
        print(json.dumps(line), flush=True)


def issue_roofline(warp_inst, kernel_ms, device):
    """Warp instructions issued per second vs the SMs' issue peak (4 schedulers
    per SM, one instruction per cycle each, at the maximum SM clock)."""
    import torch

    if not warp_inst or not kernel_ms:
        return None
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    try:
        import pynvml

        pynvml.nvmlInit()
        mhz = pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(device), pynvml.NVML_CLOCK_SM)
    except Exception:
        mhz = 1965
    peak = sms * 4 * mhz * 1e6
    achieved = warp_inst / (kernel_ms / 1e3)
    return {"achieved": achieved, "peak": peak, "unit": "warp-instructions/s", "frac": achieved / peak,
            "warp_instructions_per_launch": warp_inst, "source": "profiles/ncu_summary.json"}


def init_dist(world: int, local: int):
    """One process per GPU; with more ranks than GPUs (a one-GPU box running
    --gpus N) ranks share GPUs round-robin and the process group is gloo
    (NCCL cannot put two ranks on one GPU).  Returns (dist or None, device)."""
    import torch

    ndev = torch.cuda.device_count()
    shared = world > ndev or bool(os.environ.get("GPUBPE_BENCH_SHARE_GPU"))
    if shared:
        local %= ndev
    torch.cuda.set_device(local)
    if world == 1:
        return None, local, shared
    import torch.distributed as dist

    if shared or os.environ.get("GPUBPE_BENCH_BACKEND") == "gloo":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist, local, shared


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch

    import paper_2603_02597_b200 as bpe
    import fixtures

    dist, local, shared = init_dist(world, local)
    if args.workload.startswith("corpus"):
        run_corpus(args, rank, world, local, dist)
        if dist:
            dist.destroy_process_group()
        return
    doc, spec = load_workload(args.workload)
    tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths(),
                                   bpe.BlockConfig(max_seq_len=WHOLE, chunk_budget=WHOLE))
    enc = tok.device_encoder(local)
    dev = torch.device("cuda", local)
    n = len(doc)
    d_data = torch.frombuffer(bytearray(doc), dtype=torch.uint8).to(dev)
    d_offs = torch.tensor([0, n], dtype=torch.int64, device=dev)
    out_ids = torch.empty(n, dtype=torch.int32, device=dev)
    out_offs = torch.empty(2, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        enc.encode_into(d_data, d_offs, out_ids, out_offs, WHOLE, WHOLE, stream)

    # correctness of the measured configuration
    step()
    st = enc.query()
    n_ids = int(out_offs[1].item())
    assert n_ids == spec["tokens_whole"], (n_ids, spec["tokens_whole"])
    import hashlib

    digest = hashlib.sha256(out_ids[:n_ids].cpu().numpy().astype("<u4").tobytes()).hexdigest()
    assert digest == spec["sha_whole"], "device ids differ from the reference digest"

    enc.set_profiling(True)
    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kern = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev0[i].record(stream)
            step()
            ev1[i].record(stream)
            kern.append(enc.kernel_ms())  # syncs on this step only
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    enc.set_profiling(False)
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    total_ms = sum(step_ms)
    # context only (not the metric): the same kernel with the tables warm in L2
    # (no flush between steps), min(steps, 200) back-to-back launches
    enc.set_profiling(True)
    warm = []
    for _ in range(min(args.steps, 200)):
        step()
        warm.append(enc.kernel_ms())
    enc.set_profiling(False)

    # e2e through the public API: host bytes in, host ids out
    for _ in range(3):
        bpe.tokenize_batch([doc], tok)
    e2e_t = []
    for _ in range(min(args.steps, 100)):
        t0 = time.perf_counter()
        r = bpe.tokenize_batch([doc], tok)
        e2e_t.append(time.perf_counter() - t0)
        assert len(r.token_ids[0]) == n_ids
        del r  # the caller is done with the ids: their pooled buffer is reused
    e2e_p50 = statistics.median(e2e_t)
    e2e_p90 = sorted(e2e_t)[int(0.9 * (len(e2e_t) - 1))]
    if dist:
        t = torch.tensor([total_ms, e2e_p50], dtype=torch.float64, device=dev)
        if dist.get_backend() == "gloo":
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_p50 = float(t[0]), float(t[1])
    value = world * n_ids * args.steps / (total_ms / 1000.0)
    ms_per_step = total_ms / args.steps
    e2e = {"value": world * n_ids / e2e_p50, "unit": UNIT, "h2d_bytes_per_step": n + 16,
           "d2h_bytes_per_step": 4 * n_ids + 16, "p50_ms": 1000 * e2e_p50, "p90_ms": 1000 * e2e_p90,
           "api": "tokenize_batch",
           "timing": "wall clock per call, p50 of min(steps, 100), max over ranks"}
    corpus = None
    if args.corpus_mb:
        corpus = corpus_leg(args, args.corpus_mb, rank, world, local, dist, steps=3, warmup=3)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    t_tile = statistics.mean(kern) / 1000.0
    b_alg = n + 4 * n_ids + 16 * 2  # bytes in + ids out + offsets in/out
    p = peaks()
    peak = float(p.get("hbm_gbs", 6650.0))
    achieved = b_alg / t_tile / 1e9
    # DRAM bytes of one k_encode launch on this workload, from the committed
    # `ncu --set full` capture (profiles/ncu_summary.json, tools/ncu_summary.py)
    summ = ncu_summary(args.workload)
    cpu = cpu_baseline(doc, args.cpu_seconds) if world == 1 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "p50_ms": statistics.median(step_ms), "p90_ms": sorted(step_ms)[int(0.9 * (len(step_ms) - 1))],
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": e2e["value"] / (world * PAPER_131K_TOKS) if args.workload == "c1_131k" else None,
        "vs_baseline_source": ("end-to-end tokens/s per GPU over BASELINE.md Table 1's paper GPU-Opt, 131K tokens "
                               "in 53.4 ms end to end on an RTX 4070 (2.45 M tok/s)") if args.workload == "c1_131k" else None,
        "dtype": "u8->u32",
        "data": "synthetic",
        "config": workload_config(args, world, n, n_ids),
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": summ.get("traffic_bytes"), "kernel": "k_encode",
                     "alg_bytes_per_launch": b_alg, "kernel_ms": statistics.mean(kern),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst)" if p else "fallback",
                     # the binding ceiling of this integer kernel: warp-instruction issue
                     # (ncu smsp__inst_executed.sum per launch / the live kernel time)
                     "issue": issue_roofline(summ.get("warp_instructions"), statistics.mean(kern), local)},
        "kernel_ms": {"k_encode": statistics.mean(kern), "k_encode_p50": statistics.median(kern),
                      "k_encode_warm_l2_p50": statistics.median(warm),
                      "warm_l2": "context only: no flush between launches (tables and input in L2)"},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "gpu_launches": args.steps,
        "device_stats": st,
        "wall_s": wall,
        "ranks_share_gpus": shared,
        "corpus": corpus,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
