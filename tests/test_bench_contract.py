"""bench.py's contract: the reference arm's JSON line on CPU (the driver's
keys), and on the GPU box `python bench.py --gpus 2` without torchrun --
it spawns the ranks itself (sharing the one GPU over gloo when the box has
fewer GPUs than ranks), rank 0 prints one line with n_gpus = 2 and the corpus
leg sharded across both ranks, with the reference arm's config keys."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, env=env, cwd=ROOT)


def test_reference_arm_line_has_the_contract_keys():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["unit"] == line["unit"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["config"]["workload"] == "c1_131k"


def test_reference_arm_other_ranks_exit_quietly():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"],
             {"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def _line(out: str) -> dict:
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out[-3000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_gpus_2_spawns_ranks_and_shards_the_corpus():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "20", "--warmup", "3",
           "--corpus-mb", "64", "--cpu-seconds", "1"]
    proc = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = _line(proc.stdout)
    assert line["n_gpus"] == 2 and line["steps"] == 20 and line["value"] > 0
    assert line["e2e"]["value"] > 0 and line["roofline"]["frac"] > 0
    c = line["corpus"]
    assert c["n_gpus"] == 2 and c["scaling"] == "strong" and c["config"]["workload"] == "corpus_64m"
    assert c["e2e"]["value"] > 0 and c["roofline"]["peak"] == 2 * line["roofline"]["peak"]
    ref = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert ref.returncode == 0, ref.stderr[-3000:]
    rline = _line(ref.stdout)
    assert rline["impl"] == "reference" and set(rline["config"]) == set(line["config"])
    assert {k: v for k, v in rline["config"].items() if k != "parallelism"} == \
        {k: v for k, v in line["config"].items() if k != "parallelism"}
