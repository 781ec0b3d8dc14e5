"""Engine configuration and work counters.

`BlockConfig` and `PassCounters` keep the reference's fields and validation
(/root/reference/pkg/src/lanebpe/engines.py:40-65 and :77-97).  On the device
`lane_count` has no effect (the reference documents it as scheduling-only);
`max_seq_len` / `chunk_budget` keep their meaning as the chunking semantics of
the batch path.  PassCounters.passes is the number of merges, i.e. input bytes
minus output ids, the identity the reference's acceptance gate checks
(test_acceptance.py:363-376).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class BlockConfig:
    lane_count: int = 256
    max_seq_len: int = 8192
    chunk_budget: int | None = None

    def __post_init__(self):
        if self.chunk_budget is None:
            object.__setattr__(self, "chunk_budget", self.max_seq_len)
        if self.lane_count < 1:
            raise ValueError(f"lane_count must be >= 1, got {self.lane_count}")
        if self.max_seq_len < 2:
            raise ValueError(f"max_seq_len must be >= 2, got {self.max_seq_len}")
        if not 2 <= self.chunk_budget <= self.max_seq_len:
            raise ValueError(
                f"chunk_budget must be in [2, max_seq_len={self.max_seq_len}], got {self.chunk_budget}")


@dataclass
class PassCounters:
    passes: int = 0
    lookups: int = 0
    compaction_moves: int = 0
    buffer_allocations: int = 0

    def merge_from(self, other: "PassCounters") -> None:
        self.passes += other.passes
        self.lookups += other.lookups
        self.compaction_moves += other.compaction_moves
        self.buffer_allocations += other.buffer_allocations


# ---------------------------------------------------------------- token level
#
# The reference's engine entry points work on token ids (not bytes):
# sequential_bpe (engines.py:269-335) and run_block_engine (:338-403).  Here
# both run the exact device engine over the ids (gpubpe_merge_tokens, one CTA
# per run of ids the table covers; ids no rule mentions never merge and stay
# in place) and return the reference's result; their counters follow from
# the result (see each function).

def token_seq(ids):
    """A token-id sequence as a 1-D uint32 array (engines.py:100-105)."""
    import numpy as np

    arr = np.asarray(ids, dtype=np.uint32)
    if arr.ndim != 1:
        raise ValueError(f"expected a 1-D sequence, got shape {arr.shape}")
    return arr


class _TableDevice:
    """Device context + producer map of one PackedPairTable (kept for the last
    few tables used; the table object is held so its id stays unique)."""

    def __init__(self, table):
        import numpy as np

        from .device import DeviceEncoder
        from .merge_table import rule_arrays

        self.table = table
        left, right, rank, new = rule_arrays(table)
        self.n_ids = int(max(left.max(initial=0), right.max(initial=0), new.max(initial=0))) + 1
        self.enc = DeviceEncoder(np.zeros(256, np.uint32), left, right, rank, new, memo=False)
        # token -> (left, right, rank) of the first rule producing it
        self.prod = {}
        for a, b, k, c in zip(left.tolist(), right.tolist(), rank.tolist(), new.tolist()):
            self.prod.setdefault(c, (a, b, k))

    def merge(self, ids):
        """Exact greedy BPE fixpoint of ids on the device."""
        import numpy as np
        import torch

        from . import _native

        known = ids < self.n_ids
        # maximal runs of covered ids (ids outside the table are separators)
        edges = np.flatnonzero(np.diff(np.r_[0, known.view(np.int8), 0]))
        starts, ends = edges[0::2], edges[1::2]
        merged, offs, counts = None, None, None
        if len(starts):
            flat = np.concatenate([ids[s:e] for s, e in zip(starts, ends)]) if len(starts) > 1 else ids[starts[0]:ends[0]]
            offs = np.zeros(len(starts) + 1, np.uint64)
            np.cumsum(ends - starts, out=offs[1:].view(np.int64))
            with torch.cuda.device(self.enc.device):
                d_in = torch.from_numpy(np.ascontiguousarray(flat).view(np.int32)).cuda(self.enc.device)
                d_out = torch.empty_like(d_in)
                counts = np.zeros(len(starts), np.uint64)
                s = torch.cuda.current_stream(self.enc.device)
                rc = self.enc._lib.gpubpe_merge_tokens(self.enc._h, d_in.data_ptr(), offs.ctypes.data, len(starts),
                                                       d_out.data_ptr(), counts.ctypes.data, s.cuda_stream)
                _native.check(rc, self.enc._h, "gpubpe_merge_tokens")
                merged = d_out.cpu().numpy().view(np.uint32)
        pieces, prev = [], 0
        for k, (s0, e0) in enumerate(zip(starts, ends)):
            pieces.append(ids[prev:s0])  # uncovered ids in between
            o = int(offs[k])
            pieces.append(merged[o:o + int(counts[k])])
            prev = e0
        pieces.append(ids[prev:])
        out = np.concatenate(pieces).astype(np.uint32, copy=False) if pieces else ids[:0].copy()
        return out

    def spine(self, top: int, leaf: int, side: int) -> int:
        """Merges on one spine of top's tree down to the input id leaf (side 0:
        left operands, 1: right operands)."""
        n, t = 0, top
        while t != leaf and t in self.prod:
            t = self.prod[t][side]
            n += 1
        return n

    def trace(self, ids, out) -> list[int]:
        """Ranks of the merges in application order: each output id's tree above
        the input ids it covers, ranks sorted (a well-formed table merges in
        non-decreasing rank order)."""
        ranks, pos = [], 0

        def expand(t):
            nonlocal pos
            if pos < len(ids) and t == int(ids[pos]):
                pos += 1
                return
            a, b, k = self.prod[t]
            ranks.append(k)
            expand(a)
            expand(b)

        for t in out.tolist():
            expand(t)
        return sorted(ranks)


_TABLES: list = []


def _table_device(table) -> _TableDevice:
    for td in _TABLES:
        if td.table is table:
            return td
    td = _TableDevice(table)
    _TABLES.insert(0, td)
    del _TABLES[4:]
    return td


def _check_trace(td: _TableDevice):
    st = td.enc.query()
    if not st["well_formed"]:
        raise NotImplementedError("merge traces are reconstructed for well-formed tables only "
                                  "(every rule using a token ranks above the rule producing it)")


def sequential_bpe(tokens, table, trace: list | None = None):
    """Greedy lowest-rank / leftmost BPE of token ids to a fixpoint
    (engines.py:269-335), on the device.  Returns (ids, PassCounters) with the
    reference's counters: passes = merges; lookups = the n - 1 initial probes
    plus one per neighbour of every merge (a merge on the left spine of the
    first output token has no left neighbour, one on the right spine of the
    last has no right one); no compaction moves or pool buffers."""
    ids = token_seq(tokens)
    counters = PassCounters()
    n = len(ids)
    if n < 2:
        return ids.copy(), counters
    td = _table_device(table)
    out = td.merge(ids)
    m = n - len(out)
    counters.passes = m
    counters.lookups = (n - 1) + 2 * m - td.spine(int(out[0]), int(ids[0]), 0) - td.spine(int(out[-1]), int(ids[-1]), 1)
    if trace is not None and m:
        _check_trace(td)
        trace.extend(td.trace(ids, out))
    return out, counters


def run_block_engine(tokens, table, config: BlockConfig | None = None, variant: str = "optimized",
                     trace: list | None = None):
    """The lane-engine entry point (engines.py:338-403) on the device: the same
    result as sequential_bpe, with the reference lane model's counters (one
    merge per pass; every pass evaluates all cur_len - 1 pairs, the final one
    finding none while at least two ids remain; cur_len - 1 compaction moves
    per merge; two pool buffers).  SequenceTooLong above config.max_seq_len."""
    from .errors import SequenceTooLong

    if variant not in ("baseline", "optimized"):
        raise ValueError(f"unknown variant {variant!r}")
    config = config if config is not None else BlockConfig()
    ids = token_seq(tokens)
    n = len(ids)
    counters = PassCounters()
    if n > config.max_seq_len:
        raise SequenceTooLong(f"length {n} exceeds max_seq_len {config.max_seq_len}")
    if n < 2:
        return ids.copy(), counters
    td = _table_device(table)
    out = td.merge(ids)
    m = n - len(out)
    counters.passes = m
    counters.buffer_allocations = 2
    counters.compaction_moves = sum(n - k - 1 for k in range(m))
    last = n - m  # length after the final merge: one more (empty) evaluation if >= 2
    counters.lookups = sum(L - 1 for L in range(last if last >= 2 else last + 1, n + 1))
    if trace is not None and m:
        _check_trace(td)
        trace.extend(td.trace(ids, out))
    return out, counters
