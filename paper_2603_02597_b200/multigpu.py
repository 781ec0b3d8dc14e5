"""Multi-GPU sharding of an encode: one process per GPU, no collective on the
data path.

Documents are independent in the reference (chunker.py:139-179 encodes each
input on its own), so a batch shards by contiguous document ranges balanced
by bytes.  A single document can be split too, at a position that is a cut in
the reference's own semantics, so no merge ever spans the split:

* P-default documents longer than max_seq_len are encoded by the reference as
  independent chunk_budget-sized chunks (chunker.py:42-53,139-144); a piece of
  such a document is handed to the encoder as its list of chunks, each a
  document of its own (no chunk exceeds max_seq_len, so none is re-cut);
* otherwise a split is taken at a byte pair outside the junction set J (no
  rule joins a token ending in byte x to one starting with byte y, so no merge
  can span x|y).

Each rank encodes its shard on its own GPU (the single-GPU engine), copies
its ids to the host, and rank 0 concatenates them in rank order.  The only
cross-rank traffic is that final gather (torch.distributed, gloo or NCCL),
which is not part of the measured device path.
"""

from __future__ import annotations

import numpy as np


def shard_batch(doc_offs: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous document ranges [d0, d1) per rank with about equal bytes.

    Every document goes to exactly one rank; ranks may be empty when there
    are fewer documents than ranks.
    """
    offs = np.asarray(doc_offs, dtype=np.int64)
    n_docs = len(offs) - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    total = int(offs[-1]) if n_docs > 0 else 0
    bounds = [0]
    for r in range(1, world):
        target = total * r // world
        # first document starting at or after the byte target (never before the previous bound)
        d = int(np.searchsorted(offs[:n_docs], target, side="left")) if n_docs > 0 else 0
        bounds.append(max(bounds[-1], min(d, n_docs)))
    bounds.append(n_docs)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def split_points(data: bytes, world: int, junction_bits: np.ndarray, max_seq_len: int,
                 chunk_budget: int) -> list[int]:
    """Byte positions 0 = p_0 <= p_1 <= ... <= p_world = len(data) at which one
    document can be cut without changing its encoding: chunk boundaries when
    the document is chunked (len > max_seq_len), else junction misses.

    junction_bits: uint32[2048] bitmap, bit (x << 8 | y) set iff some rule joins
    a token ending in byte x to a token starting with byte y (the device
    context's table, DeviceEncoder.junction_bits()).
    """
    n = len(data)
    pts = [0]
    b = np.frombuffer(data, dtype=np.uint8)
    for r in range(1, world):
        target = max(pts[-1], n * r // world)
        if n > max_seq_len:
            p = min(n, -(-target // chunk_budget) * chunk_budget)
        elif target == 0 or target >= n:
            p = min(target, n)
        else:
            k = (b[target - 1:n - 1].astype(np.uint32) << 8) | b[target:n].astype(np.uint32)
            hit = np.flatnonzero(((junction_bits[k >> 5] >> (k & 31)) & 1) == 0)
            p = target + int(hit[0]) if hit.size else n
        pts.append(max(pts[-1], p))
    pts.append(n)
    return pts


def split_document(data: bytes, world: int, junction_bits: np.ndarray, max_seq_len: int,
                   chunk_budget: int) -> list[list[bytes]]:
    """Per rank, the documents to encode (in order) so that concatenating all
    ranks' ids reproduces the encoding of `data` under (max_seq_len,
    chunk_budget): pieces of a chunked document as their chunks, otherwise the
    junction-cut pieces themselves."""
    pts = split_points(data, world, junction_bits, max_seq_len, chunk_budget)
    out = []
    for r in range(world):
        lo, hi = pts[r], pts[r + 1]
        if len(data) > max_seq_len:
            out.append([data[c:min(c + chunk_budget, hi)] for c in range(lo, hi, chunk_budget)])
        else:
            out.append([data[lo:hi]] if hi > lo else [])
    return out


def concat_results(parts: list[tuple[np.ndarray, np.ndarray]]) -> tuple[np.ndarray, np.ndarray]:
    """Rank-ordered (ids, offs) CSR pieces -> one CSR (ids, offs)."""
    ids = [p[0] for p in parts]
    offs = [np.asarray(p[1], dtype=np.int64) for p in parts]
    out_ids = np.concatenate(ids) if ids else np.empty(0, np.uint32)
    out_offs = [np.zeros(1, np.int64)]
    base = 0
    for o in offs:
        if len(o) > 1:
            out_offs.append(o[1:] + base)
        base += int(o[-1]) if len(o) else 0
    return out_ids.astype(np.uint32, copy=False), np.concatenate(out_offs)


def encode_sharded(data: np.ndarray, doc_offs: np.ndarray, encode, rank: int, world: int, group=None):
    """Encode this rank's share of a packed batch and gather on rank 0.

    encode(data, offs) -> (ids uint32[], offs int64[]) runs the single-GPU
    engine (DeviceEncoder.encode_packed_host on this rank's GPU).  Returns the
    full (ids, offs) CSR on rank 0 and None elsewhere.  With world == 1 no
    process group is needed.
    """
    d0, d1 = shard_batch(doc_offs, world)[rank]
    offs = np.asarray(doc_offs, dtype=np.int64)
    lo, hi = int(offs[d0]), int(offs[d1])
    part = encode(np.ascontiguousarray(data[lo:hi]), offs[d0:d1 + 1] - lo)
    if world == 1:
        return part
    import torch.distributed as dist

    gathered = [None] * world if rank == 0 else None
    dist.gather_object((np.asarray(part[0]), np.asarray(part[1])), gathered, dst=0, group=group)
    if rank != 0:
        return None
    return concat_results(gathered)
