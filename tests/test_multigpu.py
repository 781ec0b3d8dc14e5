"""Multi-GPU sharding (paper_2603_02597_b200/multigpu.py) on CPU.

The sharding and gather logic is host code; here the per-rank "engine" is
the CPU oracle (test infrastructure), so the world-size-2 gloo run checks
that sharded encoding concatenates to exactly the single-process result.
"""

import os
import random

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import fixtures
from paper_2603_02597_b200 import multigpu
from paper_2603_02597_b200.chunker import pack_texts


def junction_bits(tables) -> np.ndarray:
    """J restated from the oracle tables (same definition as ctx.cu): the
    (last byte of left operand, first byte of right operand) of every rule."""
    from oracle.oracle import byte_symbols

    inv = {c: i for i, c in enumerate(byte_symbols())}
    strs = {}
    for sym, i in tables.symbol_to_id.items():
        try:
            strs[i] = bytes(inv[c] for c in sym)
        except KeyError:
            pass
    bits = np.zeros(2048, dtype=np.uint32)
    for l, r in zip(tables.left, tables.right):
        if l in strs and r in strs:
            k = (strs[l][-1] << 8) | strs[r][0]
            bits[k >> 5] |= np.uint32(1 << (k & 31))
    return bits


def test_shard_batch_covers_every_document_once():
    rng = np.random.default_rng(3)
    for n_docs in (0, 1, 2, 7, 100):
        lens = rng.integers(0, 5000, n_docs)
        offs = np.zeros(n_docs + 1, np.int64)
        offs[1:] = np.cumsum(lens)
        for world in (1, 2, 3, 8):
            sh = multigpu.shard_batch(offs, world)
            assert len(sh) == world and sh[0][0] == 0 and sh[-1][1] == n_docs
            assert all(a <= b for a, b in sh) and all(sh[i][1] == sh[i + 1][0] for i in range(world - 1))
            if n_docs >= 50:
                per = [offs[b] - offs[a] for a, b in sh]
                assert max(per) <= offs[-1] / world + lens.max() + 1


def test_concat_results_roundtrip():
    parts = [(np.array([1, 2, 3], np.uint32), np.array([0, 2, 3])),
             (np.array([], np.uint32), np.array([0, 0])),
             (np.array([4, 5], np.uint32), np.array([0, 2]))]
    ids, offs = multigpu.concat_results(parts)
    assert ids.tolist() == [1, 2, 3, 4, 5] and offs.tolist() == [0, 2, 3, 3, 5]


@pytest.mark.parametrize("msl,cb", [(1 << 40, 1 << 40), (8192, 8192), (5000, 3000)])
def test_split_points_are_exact(oracle, oracle_tables, msl, cb):
    jb = junction_bits(oracle_tables)
    docs = [b"".join(fixtures.prose_samples()[:12]), bytes(random.Random(2).choice(b"ab c1\n") for _ in range(20000))]
    for doc in docs:
        want = oracle.encode_docs([doc], msl, cb)[0]
        for world in (2, 3, 5):
            pts = multigpu.split_points(doc, world, jb, msl, cb)
            assert pts[0] == 0 and pts[-1] == len(doc) and pts == sorted(pts)
            shards = multigpu.split_document(doc, world, jb, msl, cb)
            assert b"".join(b"".join(s) for s in shards) == doc
            got = [ids for s in shards if s for ids in oracle.encode_docs(s, msl, cb)]
            got = np.concatenate(got) if got else np.empty(0, np.uint32)
            assert np.array_equal(got, want), (world, pts)


def _worker(rank, world, port, docs, msl, cb, q, device=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    data, offs = pack_texts(docs)
    if device:  # the CUDA engine of this rank's GPU (ranks share GPUs round-robin on a small box)
        import torch

        import paper_2603_02597_b200 as bpe

        gpu = rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        enc = bpe.Tokenizer.from_files(*fixtures.gpt2_paths()).device_encoder(gpu)

        def encode(d, o):
            ids, oo, _, _ = enc.encode_packed_host(d, o, msl, cb)
            return np.array(ids), oo
    else:
        from oracle.oracle import OracleEncoder, load_tables

        orc = OracleEncoder.from_tables(load_tables(*fixtures.gpt2_paths()))

        def encode(d, o):  # stands in for DeviceEncoder.encode_packed_host on this rank's GPU
            ids, oo, _ = orc.encode_packed(d, o, msl, cb, 1)
            return ids, oo

    res = multigpu.encode_sharded(data, offs, encode, rank, world)
    if rank == 0:
        q.put((res[0].tolist(), res[1].tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("device", [False, pytest.param(True, marks=pytest.mark.gpu)])
def test_gloo_world2_sharded_encode_matches_single(oracle, device):
    """world 2 over gloo: the per-rank engine is the C oracle on CPU, or the
    CUDA engine (DeviceEncoder) when a GPU is present (-m gpu)."""
    docs = fixtures.prose_samples()[:30] + [b"", b"hello world", b" between", b"x" * 20000]
    msl, cb = 8192, 8192
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random(os.getpid() + device).randrange(2000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, docs, msl, cb, q, device)) for r in range(2)]
    for p in ps:
        p.start()
    ids, offs = q.get(timeout=240)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.encode_docs(docs, msl, cb)
    got = [ids[offs[i]:offs[i + 1]] for i in range(len(docs))]
    assert [w.tolist() for w in want] == got
