"""Access to the committed fixtures (tests/golden/) without /root/reference.

The GPT-2 tables are committed gzip-compressed; `gpt2_paths()` expands them
once per process into a temporary directory and returns plain file paths, so
the reference-shaped API `Tokenizer.from_files(vocab, merges)` can be used
unchanged on the GPU box.
"""

from __future__ import annotations

import gzip
import json
import tempfile
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"


@lru_cache(maxsize=1)
def gpt2_paths() -> tuple[Path, Path]:
    d = Path(tempfile.mkdtemp(prefix="gpt2_tables_"))
    out = []
    for name in ("vocab.json", "merges.txt"):
        p = d / name
        p.write_bytes(gzip.decompress((GOLDEN / "gpt2" / (name + ".gz")).read_bytes()))
        out.append(p)
    return out[0], out[1]


def gz_text(name: str) -> bytes:
    return gzip.decompress((GOLDEN / name).read_bytes())


def prose_samples() -> list[bytes]:
    return gz_text("prose_corpus.txt.gz").rstrip(b"\n").split(b"\n")


def batch_fixture() -> list[bytes]:
    return gz_text("batch_fixture.txt.gz").rstrip(b"\n").split(b"\n")


def csr(npz, ids_key="ids", offs_key="offs") -> list[np.ndarray]:
    ids, offs = npz[ids_key], npz[offs_key]
    return [ids[offs[i] : offs[i + 1]] for i in range(len(offs) - 1)]


def golden_prose() -> list[np.ndarray]:
    return csr(np.load(GOLDEN / "golden_prose.npz"))


def batch_fixture_ids() -> list[np.ndarray]:
    return csr(np.load(GOLDEN / "batch_fixture_ids.npz"))


def mixed_cases():
    """(docs, {config_name: (max_seq_len, chunk_budget, expected list)})."""
    z = np.load(GOLDEN / "mixed_cases.npz")
    data, offs = z["data"], z["offs"]
    docs = [data[offs[i] : offs[i + 1]].tobytes() for i in range(len(offs) - 1)]
    cfgs = {}
    for k in z.files:
        if k.startswith("cfg_"):
            name = k[4:]
            msl, cb = (int(x) for x in z[k])
            cfgs[name] = (msl, cb, csr(z, f"ids_{name}", f"offs_{name}"))
    return docs, cfgs


def known_answers() -> dict:
    return json.loads((GOLDEN / "known_answers.json").read_text())


def synth_sizes() -> dict:
    return json.loads((GOLDEN / "synth_sizes.json").read_text())
