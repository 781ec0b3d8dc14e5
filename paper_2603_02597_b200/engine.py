"""Engine configuration and work counters.

`BlockConfig` and `PassCounters` keep the reference's fields and validation
(/root/reference/pkg/src/lanebpe/engines.py:40-65 and :77-97).  On the device
`lane_count` has no effect (the reference documents it as scheduling-only);
`max_seq_len` / `chunk_budget` keep their meaning as the chunking semantics of
the batch path.  PassCounters.passes is the number of merges, i.e. input bytes
minus output ids, the identity the reference's acceptance gate checks
(test_acceptance.py:363-376).

The token-level entry points below (sequential_bpe, run_block_engine,
eval_pairs, compact_scan, compact_double_buffer, inject_compaction_fault)
keep the reference's signatures and results and run on the device.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np


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


@dataclass(frozen=True)
class PairCandidate:
    """Winning pair of one evaluation pass (engines.py:68-74)."""

    pos: int
    rank: int
    new_token: int


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
# sequential_bpe (engines.py:269-335) and run_block_engine (:338-403), plus the
# lane engine's single steps eval_pairs (:133-168) and the two compactions
# (:171-217).  All of them run on the device here: the exact engine of
# tokens.cu (gpubpe_merge_tokens_ex: one CTA per sequence), k_eval_pairs,
# k_compact_*.  Ids are mapped to the device context's internal ids first:
# ids no rule mentions become the context's inert sentinel (they can never
# merge) and are restored in order afterwards; tables with ids >= 2^24 are
# densely renumbered.  There is no CPU engine behind any of these names.

def token_seq(ids):
    """A token-id sequence as a 1-D uint32 array (engines.py:100-105)."""
    import numpy as np

    arr = np.asarray(ids, dtype=np.uint32)
    if arr.ndim != 1:
        raise ValueError(f"expected a 1-D sequence, got shape {arr.shape}")
    return arr


_TRACE_RANK = 0xFFFFFFFF
_TRACE_LAST = 1 << 32
_TRACE_FIRST = 1 << 33


class _TableDevice:
    """Device context of one PackedPairTable (kept for the last few tables
    used; the table object is held so its id stays unique)."""

    WIDE = 1 << 24

    def __init__(self, table):
        import numpy as np

        from .device import DeviceEncoder
        from .merge_table import rule_arrays

        self.table = table
        left, right, rank, new = rule_arrays(table)
        ids = np.unique(np.concatenate([left, right, new])) if left.size else np.zeros(0, np.uint32)
        self.ext = ids if ids.size and int(ids[-1]) >= self.WIDE else None
        if self.ext is not None:  # dense internal ids 0..len-1
            left, right, new = (np.searchsorted(ids, x).astype(np.uint32) for x in (left, right, new))
            self.sentinel = len(ids)
        else:
            self.sentinel = int(ids[-1]) + 1 if ids.size else 1
        self.enc = DeviceEncoder(np.zeros(256, np.uint32), left, right, rank, new, memo=False)
        self.well_formed = bool(self.enc.query()["well_formed"])

    # -- id mapping
    def to_internal(self, ids):
        """(internal uint32 ids, mask of ids outside the table or None)."""
        import numpy as np

        if self.ext is None:
            out = ids.copy()
            outside = ids >= self.sentinel
            if outside.any():
                out[outside] = self.sentinel
                return out, outside
            return out, None
        idx = np.searchsorted(self.ext, ids)
        hit = idx < len(self.ext)
        hit[hit] = self.ext[idx[hit]] == ids[hit]
        out = np.where(hit, idx, self.sentinel).astype(np.uint32)
        return out, (None if hit.all() else ~hit)

    def to_external(self, out, ids, outside):
        if self.ext is not None:
            keep = out != self.sentinel
            res = out.copy()
            res[keep] = self.ext[out[keep]]
            out = res
        if outside is not None:  # inert ids never merge: they come back in order
            out = out.copy()
            out[out == self.sentinel] = ids[outside]
        return out

    def device_ids(self, internal):
        import torch

        dev = torch.device("cuda", self.enc.device)
        return torch.from_numpy(internal.view(np.int32) if internal.size else np.zeros(1, np.int32)).to(dev)

    # -- engine
    def merge(self, ids, fault: bool = False):
        """Exact greedy BPE fixpoint of ids on the device -> (out, merge
        records): each record is (pass << 34) | (at position 0 << 33) | (right
        token last << 32) | rank, merges in pass order (tokens.cu)."""
        import torch

        from . import _native

        internal, outside = self.to_internal(ids)
        n = len(ids)
        with torch.cuda.device(self.enc.device):
            d_in = self.device_ids(internal)
            d_out = torch.empty_like(d_in)
            d_trace = torch.empty(max(n, 1), dtype=torch.int64, device=d_in.device)
            offs = np.array([0, n], np.uint64)
            counts = np.zeros(1, np.uint64)
            s = torch.cuda.current_stream(self.enc.device)
            rc = self.enc._lib.gpubpe_merge_tokens_ex(self.enc._h, d_in.data_ptr(), offs.ctypes.data, 1,
                                                      d_out.data_ptr(), counts.ctypes.data, d_trace.data_ptr(),
                                                      0 if fault else -1, s.cuda_stream)
            _native.check(rc, self.enc._h, "gpubpe_merge_tokens_ex")
            cnt = int(counts[0])
            out = d_out[:cnt].cpu().numpy().view(np.uint32)
            rec = d_trace[: n - cnt].cpu().numpy().view(np.uint64)
        return self.to_external(out, ids, outside), rec

    def trace(self, rec) -> list[int]:
        """The reference's merge-rank trace from the device's merge records:
        in application order when every pass merged one pair (tables that are
        not well-formed run strict passes), sorted by rank otherwise (a
        well-formed table merges in non-decreasing rank order)."""
        ranks = (rec & np.uint64(_TRACE_RANK)).astype(np.int64)
        if self.well_formed:
            ranks = np.sort(ranks, kind="stable")
        return ranks.tolist()

    def eval_pairs(self, ids):
        import torch

        from . import _native

        internal, _ = self.to_internal(ids)
        res = np.zeros(3, np.uint64)
        with torch.cuda.device(self.enc.device):
            d_in = self.device_ids(internal)
            s = torch.cuda.current_stream(self.enc.device)
            rc = self.enc._lib.gpubpe_eval_pairs(self.enc._h, d_in.data_ptr(), len(ids), res.ctypes.data,
                                                 s.cuda_stream)
            _native.check(rc, self.enc._h, "gpubpe_eval_pairs")
        if int(res[0]) == (1 << 64) - 1:
            return None
        new = int(res[2])
        if self.ext is not None:
            new = int(self.ext[new])
        return PairCandidate(int(res[0]), int(res[1]), new)

    def lookup_keys(self, keys):
        """(hit bool[m], vals uint64[m]) of packed keys, probed on the device."""
        import torch

        from . import _native

        m = len(keys)
        keys = np.asarray(keys, dtype=np.uint64)
        left = (keys >> np.uint64(32)).astype(np.uint32)
        right = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        il, ol = self.to_internal(left)
        ir, orr = self.to_internal(right)
        ik = (il.astype(np.uint64) << np.uint64(32)) | ir.astype(np.uint64)
        ik[keys == np.uint64(0xFFFFFFFFFFFFFFFF)] = np.uint64(0xFFFFFFFFFFFFFFFF)  # the sentinel key
        with torch.cuda.device(self.enc.device):
            dev = torch.device("cuda", self.enc.device)
            d_k = torch.from_numpy(ik.view(np.int64) if m else np.zeros(1, np.int64)).to(dev)
            d_hit = torch.empty(max(m, 1), dtype=torch.uint8, device=dev)
            d_val = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
            s = torch.cuda.current_stream(self.enc.device)
            rc = self.enc._lib.gpubpe_lookup_keys(self.enc._h, d_k.data_ptr(), m, d_hit.data_ptr(),
                                                  d_val.data_ptr(), s.cuda_stream)
            _native.check(rc, self.enc._h, "gpubpe_lookup_keys")
            hit = d_hit[:m].cpu().numpy().astype(bool)
            vals = d_val[:m].cpu().numpy().view(np.uint64)
        if self.ext is not None and hit.any():
            nw = self.ext[(vals[hit] >> np.uint64(32)).astype(np.int64)].astype(np.uint64)
            vals[hit] = (nw << np.uint64(32)) | (vals[hit] & np.uint64(0xFFFFFFFF))
        return hit, vals


_TABLES: list = []
_TABLES_LOCK = threading.Lock()


def _table_device(table) -> _TableDevice:
    with _TABLES_LOCK:
        for td in _TABLES:
            if td.table is table:
                return td
        td = _TableDevice(table)
        _TABLES.insert(0, td)
        del _TABLES[4:]
        return td


# Fault injection for divergence testing (engines.py:247-266): when armed, the
# next block-engine run in this thread corrupts one pass on the device.
_fault_armed = threading.local()


@contextmanager
def inject_compaction_fault():
    """Arm a one-shot compaction fault for engine runs in this thread: the
    next run_block_engine shifts one pass's merge position by one slot inside
    the device engine (tokens.cu, EngineExt.fault)."""
    _fault_armed.flag = True
    try:
        yield
    finally:
        _fault_armed.flag = False


def _take_fault() -> bool:
    if getattr(_fault_armed, "flag", False):
        _fault_armed.flag = False
        return True
    return False


def sequential_bpe(tokens, table, trace: list | None = None):
    """Greedy lowest-rank / leftmost BPE of token ids to a fixpoint
    (engines.py:269-335), on the device.  Returns (ids, PassCounters) with the
    reference's counters: passes = merges; lookups = the n - 1 initial probes
    plus one per neighbour of every merge (the device marks merges at the
    sequence's start / end, which lack one); no compaction moves or pool
    buffers."""
    ids = token_seq(tokens)
    counters = PassCounters()
    n = len(ids)
    if n < 2:
        return ids.copy(), counters
    td = _table_device(table)
    out, rec = td.merge(ids)
    m = n - len(out)
    counters.passes = m
    first = int(np.count_nonzero(rec & np.uint64(_TRACE_FIRST)))
    last = int(np.count_nonzero(rec & np.uint64(_TRACE_LAST)))
    counters.lookups = (n - 1) + 2 * m - first - last
    if trace is not None:
        trace.extend(td.trace(rec))
    return out, counters


def run_block_engine(tokens, table, config: BlockConfig | None = None, variant: str = "optimized",
                     trace: list | None = None):
    """The lane-engine entry point (engines.py:338-403) on the device: the same
    result as sequential_bpe, with the reference lane model's counters (one
    merge per pass; every pass evaluates all cur_len - 1 pairs, the final one
    finding none while at least two ids remain; cur_len - 1 compaction moves
    per merge; two pool buffers).  SequenceTooLong above config.max_seq_len.
    An armed inject_compaction_fault is taken here and applied by the device
    engine."""
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
    out, rec = td.merge(ids, fault=_take_fault())
    m = n - len(out)
    counters.passes = m
    counters.buffer_allocations = 2
    counters.compaction_moves = sum(n - k - 1 for k in range(m))
    last = n - m  # length after the final merge: one more (empty) evaluation if >= 2
    counters.lookups = sum(L - 1 for L in range(last if last >= 2 else last + 1, n + 1))
    if trace is not None:
        trace.extend(td.trace(rec))
    return out, counters


def eval_pairs(tokens, table, config: BlockConfig | None = None, counters: PassCounters | None = None,
               scratch=None):
    """Lowest-rank adjacent pair, leftmost on ties (engines.py:133-168), found
    by one device pass (k_eval_pairs: every pair probed, block argmin).
    Returns a PairCandidate or None; counts len - 1 lookups.  config and
    scratch are accepted for signature compatibility (the result does not
    depend on the lane count)."""
    ids = token_seq(tokens)
    n = len(ids)
    if n < 2:
        return None
    if counters is not None:
        counters.lookups += n - 1
    return _table_device(table).eval_pairs(ids)


def _compact(tokens, best_pos: int, new_token: int, out, method: int):
    import torch

    from . import _native
    from .device import _require_cuda
    from .errors import OutOfRange

    src = token_seq(tokens)
    n = len(src)
    if not 0 <= best_pos < n - 1:
        raise OutOfRange(f"best_pos {best_pos} not a pair position in length {n}")
    _require_cuda()
    lib = _native.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    d_in = torch.from_numpy(src.view(np.int32)).to(dev)
    d_out = torch.empty(n - 1, dtype=torch.int32, device=dev)
    rc = lib.gpubpe_compact(d_in.data_ptr(), n, int(best_pos), int(new_token) & 0xFFFFFFFF, d_out.data_ptr(),
                            method, torch.cuda.current_stream().cuda_stream)
    _native.check(rc, None, "gpubpe_compact")
    res = d_out.cpu().numpy().view(np.uint32)
    if out is None:
        return res
    result = out[: n - 1]
    result[:] = res
    return result


def compact_scan(tokens, best_pos: int, new_token: int, out=None):
    """One merge by removal flags + exclusive prefix sum + scatter
    (engines.py:171-194), on the device (k_compact_scan).  OutOfRange unless
    best_pos addresses a pair; `out` (>= len - 1 entries) receives the result."""
    return _compact(tokens, best_pos, new_token, out, 1)


def compact_double_buffer(tokens, best_pos: int, new_token: int, out=None):
    """One merge by direct index mapping into a second buffer
    (engines.py:197-217), on the device (k_compact_direct)."""
    return _compact(tokens, best_pos, new_token, out, 0)
