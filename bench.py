#!/usr/bin/env python3
"""Benchmark: GPT-2 BPE encode tokens/sec on a 131k-token sequence (B200).

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
One step = one encode of one synthetic 131,072-token English-like sequence
(configs[1] of BASELINE.json, the metric's workload), whole-sequence semantics
(P-whole: no fixed-offset chunking), input resident in HBM.  L2 is flushed
(256 MiB write) before every timed step, outside the step's events.  With
N > 1 (torchrun), every rank encodes its own sequence (replicas; weak scaling,
no collective on the data path); value = all ranks' tokens / max-over-ranks time.

The line also carries: e2e (same metric through the public API,
tokenize_batch, with host bytes in and host ids out), roofline (k_encode,
the only kernel, HBM-bound), cpu_baseline (the CPU oracle port of the
reference's sequential engine on this host), clocks (NVML during the timed
region) and gpu_launches.
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
    return ap.parse_args()


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


# ------------------------------------------------------------------ reference arm


def run_reference(args, rank, world):
    """The reference's CPU path on this host: the oracle port (oracle/) of
    sequential_bpe + tokenize_batch (the reference is pure Python and cannot
    travel to this box; the port is pinned to its goldens)."""
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
        "config": {"workload": args.workload, "bytes": int(cut), "semantics": "P-whole",
                   "tokens_per_step": int(toks)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"first {cut} of {n} bytes of {args.workload} per step; oracle port "
                                   "of engines.py:269-335 sequential_bpe (one P-whole sequence is one "
                                   f"chunk, so 1 of {threads} threads works)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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


# ------------------------------------------------------------------ our arm


def run_corpus(args, rank, world, local, dist):
    """--workload corpus_<MB>m: one synthetic corpus sharded by documents across
    the ranks (multigpu.shard_batch, byte-balanced; strong scaling), P-default
    semantics, device-resident inputs; value = all ids / max-over-ranks time."""
    import numpy as np
    import torch

    import fixtures
    import synth_corpus
    import paper_2603_02597_b200 as bpe
    from paper_2603_02597_b200 import multigpu

    mb = int(args.workload.split("_")[1].rstrip("m"))
    data, offs = synth_corpus.corpus_docs(mb << 20, seed=0)
    d0, d1 = multigpu.shard_batch(offs, world)[rank]
    lo, hi = int(offs[d0]), int(offs[d1])
    tok = bpe.Tokenizer.from_files(*fixtures.gpt2_paths())
    enc = tok.device_encoder(local)
    dev = torch.device("cuda", local)
    d_data = torch.from_numpy(np.ascontiguousarray(data[lo:hi])).to(dev)
    d_offs = torch.from_numpy(offs[d0:d1 + 1] - lo).to(dev)
    out_ids = torch.empty(max(hi - lo, 1), dtype=torch.int32, device=dev)
    out_offs = torch.empty(d1 - d0 + 1, dtype=torch.int64, device=dev)
    cfg = tok.config
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        enc.encode_into(d_data, d_offs, out_ids, out_offs, cfg.max_seq_len, cfg.chunk_budget, stream)
    torch.cuda.synchronize()
    n_ids = int(out_offs[-1].item()) if d1 > d0 else 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            enc.encode_into(d_data, d_offs, out_ids, out_offs, cfg.max_seq_len, cfg.chunk_budget, stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del d_data, out_ids
    # end to end through the public host API: host bytes in, host ids out
    # (gpubpe_encode_host; large shards stream through its two-slot pipeline)
    h_data = bpe.pinned_empty(hi - lo, local)  # the shard's bytes in pinned host memory
    h_data[:] = data[lo:hi]
    h_offs = np.ascontiguousarray(offs[d0:d1 + 1] - lo)
    e2e_steps = max(1, min(args.steps, 3))
    res = enc.encode_packed_host(h_data, h_offs, cfg.max_seq_len, cfg.chunk_budget)
    assert len(res[0]) == n_ids, (len(res[0]), n_ids)
    del res
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = enc.encode_packed_host(h_data, h_offs, cfg.max_seq_len, cfg.chunk_budget)
        del res
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([ms, n_ids, e2e_s], dtype=torch.float64, device=dev)
    if dist:
        tm = t[0::2].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ids_all = t[1:2].clone()
        dist.all_reduce(ids_all, op=dist.ReduceOp.SUM)
        ms, e2e_s, total_ids = float(tm[0].item()), float(tm[1].item()), int(ids_all.item())
    else:
        total_ids = n_ids
    if rank == 0:
        line = {
            "metric": "GPT-2 BPE encode tokens/sec, synthetic corpus sharded by document",
            "value": total_ids * args.steps / (ms / 1000.0), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8->u32",
            "data": "synthetic",
            "config": {"workload": args.workload, "bytes": int(offs[-1]), "docs": len(offs) - 1,
                       "semantics": "P-default", "l2": f"input {mb} MiB > L2 (not flushed)",
                       "parallelism": f"documents sharded x{world}"},
            "clocks": clocks.summary(), "gpu_launches": args.steps,
            "roofline": corpus_roofline(args, offs, total_ids, ms / args.steps, world, local),
            "e2e": {"value": total_ids * e2e_steps / e2e_s, "unit": "tokens/s",
                    "h2d_bytes_per_step": int(offs[-1]) + 8 * len(offs),
                    "d2h_bytes_per_step": 4 * total_ids + 8 * len(offs),
                    "steps": e2e_steps, "input": "pinned host bytes",
                    "path": "encode_packed_host (gpubpe_encode_host), wall clock, max over ranks"},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()



def corpus_roofline(args, offs, total_ids, kernel_ms, world, device):
    """HBM roofline of one corpus step (all ranks' bytes over the max-over-ranks
    time, per GPU peak x world) and, for the captured workload, the issue roofline."""
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0)) * world
    b_alg = int(offs[-1]) + 4 * total_ids + 16 * len(offs)
    achieved = b_alg / (kernel_ms / 1e3) / 1e9
    summ = {}
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        summ = json.loads(prof.read_text()).get(args.workload, {})
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": summ.get("traffic_bytes"), "kernel": "k_encode", "alg_bytes_per_launch": b_alg,
            "kernel_ms": kernel_ms,
            "peak_source": ("MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback") + f" x {world} GPU(s)",
            "issue": issue_roofline(summ.get("warp_instructions"), kernel_ms, device) if world == 1 else None}


# The paper's published number for this metric (BASELINE.md Table 1):
# GPU-Opt encodes a 131,072-token sequence in 53.4 ms on an RTX 4070.
PAPER_131K_TOKS = 131072 / 53.4e-3


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


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch

    import paper_2603_02597_b200 as bpe
    import fixtures

    if os.environ.get("GPUBPE_BENCH_SHARE_GPU"):  # test only: several ranks on one GPU
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("GPUBPE_BENCH_BACKEND", "nccl")  # gloo: test of the rank logic only
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if args.workload.startswith("corpus"):
        run_corpus(args, rank, world, local, dist)
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
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * n_ids * args.steps / (total_ms / 1000.0)
    ms_per_step = total_ms / args.steps
    k_tile = kern
    t_tile = statistics.mean(k_tile) / 1000.0
    b_alg = n + 4 * n_ids + 16 * 2  # bytes in + ids out + offsets in/out
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = b_alg / t_tile / 1e9
    # DRAM bytes of one k_encode launch on this workload, from the committed
    # `ncu --set full` capture (profiles/ncu_summary.json, tools/ncu_summary.py)
    traffic = None
    warp_inst = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        summ = json.loads(prof.read_text()).get(args.workload, {})
        traffic = summ.get("traffic_bytes")
        warp_inst = summ.get("warp_instructions")

    # e2e through the public API: host bytes in, host ids out
    e2e = None
    if rank == 0 or True:
        for _ in range(3):
            bpe.tokenize_batch([doc], tok)
        e2e_t = []
        for _ in range(min(args.steps, 100)):
            t0 = time.perf_counter()
            r = bpe.tokenize_batch([doc], tok)
            e2e_t.append(time.perf_counter() - t0)
            assert len(r.token_ids[0]) == n_ids
            del r  # the caller is done with the ids: their pooled buffer is reused
        e2e = {"value": world * n_ids / statistics.median(e2e_t), "unit": UNIT,
               "h2d_bytes_per_step": n + 16, "d2h_bytes_per_step": 4 * n_ids + 16,
               "p50_ms": 1000 * statistics.median(e2e_t), "api": "tokenize_batch"}
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = cpu_baseline(doc, args.cpu_seconds) if world == 1 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "p50_ms": statistics.median(step_ms), "p90_ms": sorted(step_ms)[int(0.9 * (len(step_ms) - 1))],
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / PAPER_131K_TOKS if args.workload == "c1_131k" else None,
        "vs_baseline_source": ("BASELINE.md Table 1: paper GPU-Opt, 131K tokens in 53.4 ms on an RTX 4070 "
                               "(2.45 M tok/s, one sequence per GPU)") if args.workload == "c1_131k" else None,
        "dtype": "u8->u32",
        "data": "synthetic",
        "config": {"workload": args.workload, "bytes": n, "tokens": n_ids, "semantics": "P-whole",
                   "docs_per_gpu": 1, "l2": "flushed (256 MiB write) before every step",
                   "parallelism": f"replicas x{world}"},
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": "k_encode",
                     "alg_bytes_per_launch": b_alg, "kernel_ms": statistics.mean(k_tile),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst)" if peaks else "fallback",
                     # the binding ceiling of this integer kernel: warp-instruction issue
                     # (ncu smsp__inst_executed.sum per launch / the live kernel time)
                     "issue": issue_roofline(warp_inst, statistics.mean(k_tile), local)},
        "kernel_ms": {"k_encode": statistics.mean(k_tile), "k_encode_p50": statistics.median(k_tile)},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "gpu_launches": args.steps,
        "device_stats": st,
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
