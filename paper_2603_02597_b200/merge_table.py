"""Merge rules and the packed pair table (host side, construction time).

Mirrors /root/reference/pkg/src/lanebpe/merge_table.py:
  * `parse_merges` (:88-116): rank = 0-based rule line, an initial '#' line is a
    header, new_token = vocab[left_sym + right_sym], MalformedLine/UnknownSymbol;
  * `PackedPairTable` / `build_table` (:140-278): key (left<<32)|right, value
    (new<<32)|rank, murmur3 fmix64, power-of-two linear probing at <= 50% load,
    empty key 2**64-1, DuplicatePair / ReservedKey.  Slots are laid out exactly
    as the reference lays them out (same hash, same insertion order), so a
    table built by either package can be handed to the other.

The device never probes this table: the context (device.py) re-packs the rules
into its own L2-resident layout (csrc/ctx.cu).  `rule_arrays()` recovers the
rules from any object with the reference's `keys` / `values` / `count` fields.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .byte_codec import Vocab
from .errors import DuplicatePair, MalformedLine, ReservedKey, UnknownSymbol

U32_MASK = 0xFFFF_FFFF
U64_MASK = 0xFFFF_FFFF_FFFF_FFFF
EMPTY_KEY = U64_MASK
_M1 = 0xFF51_AFD7_ED55_8CCD
_M2 = 0xC4CE_B9FE_1A85_EC53


def pack_key(left: int, right: int) -> int:
    return (left << 32) | right


def pack_value(new_token: int, rank: int) -> int:
    return (new_token << 32) | rank


def unpack_value(value: int) -> tuple[int, int]:
    return value >> 32, value & U32_MASK


def fmix64(x: int) -> int:
    """murmur3 fmix64 (merge_table.py:49-57), the table's slot hash."""
    x &= U64_MASK
    x = ((x ^ (x >> 33)) * _M1) & U64_MASK
    x = ((x ^ (x >> 33)) * _M2) & U64_MASK
    return x ^ (x >> 33)


def fmix64_array(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64).copy()
    _mix64_inplace(x, np.empty_like(x))
    return x


def _mix64_inplace(x: np.ndarray, tmp: np.ndarray) -> None:
    """fmix64 of a uint64 array in place, with caller scratch (merge_table.py:68-77)."""
    np.right_shift(x, np.uint64(33), out=tmp)
    np.bitwise_xor(x, tmp, out=x)
    np.multiply(x, np.uint64(_M1), out=x)
    np.right_shift(x, np.uint64(33), out=tmp)
    np.bitwise_xor(x, tmp, out=x)
    np.multiply(x, np.uint64(_M2), out=x)
    np.right_shift(x, np.uint64(33), out=tmp)
    np.bitwise_xor(x, tmp, out=x)


# the reference's private names for the same functions (merge_table.py:49-66)
_mix64 = fmix64


def _mix64_np(x: np.ndarray) -> np.ndarray:
    return fmix64_array(x)


@dataclass(frozen=True)
class MergeRule:
    left: int
    right: int
    rank: int
    new_token: int


def parse_merges(merges_text, vocab: Vocab) -> list[MergeRule]:
    if isinstance(merges_text, (bytes, bytearray)):
        merges_text = merges_text.decode("utf-8")
    lines = merges_text.splitlines()
    skip = 1 if lines and lines[0].startswith("#") else 0
    ids = vocab.symbol_to_id
    rules = []
    for rank, line in enumerate(lines[skip:]):
        lineno = rank + skip + 1
        parts = line.split(" ")
        if len(parts) != 2 or not all(parts):
            raise MalformedLine(f"line {lineno}: expected two symbols, got {line!r}")
        a, b = parts
        missing = next((s for s in (a, b, a + b) if s not in ids), None)
        if missing is not None:
            raise UnknownSymbol(f"line {lineno}: symbol {missing!r} not in vocabulary")
        rules.append(MergeRule(ids[a], ids[b], rank, ids[a + b]))
    return rules


# line breaks str.splitlines() honours besides "\n" (UTF-8): such texts take the host parser
_OTHER_BREAKS = (b"\r", b"\x0b", b"\x0c", b"\x1c", b"\x1d", b"\x1e", b"\xc2\x85", b"\xe2\x80\xa8", b"\xe2\x80\xa9")


def _symbol_csr(vocab: Vocab):
    """UTF-8 of every vocabulary symbol as CSR (bytes, offsets) with the ids."""
    syms = list(vocab.symbol_to_id)
    n = len(syms)
    ids = np.fromiter(vocab.symbol_to_id.values(), dtype=np.uint32, count=n)
    cps = np.frombuffer("".join(syms).encode("utf-32-le", "surrogatepass"), dtype=np.uint32)
    width = 1 + (cps >= 0x80).astype(np.int64) + (cps >= 0x800) + (cps >= 0x10000)
    lens = np.fromiter(map(len, syms), dtype=np.int64, count=n)
    offs = np.zeros(n + 1, dtype=np.uint64)
    if cps.size:
        seg_end = np.cumsum(lens)
        csum = np.r_[0, np.cumsum(width)]
        offs[1:] = csum[seg_end]
    blob = np.frombuffer("".join(syms).encode("utf-8", "surrogatepass"), dtype=np.uint8)
    return blob, offs, ids


def parse_merges_device(merges_text, vocab: Vocab, device: int = 0):
    """parse_merges on the GPU (build.cu): (left, right,
    rank, new) uint32 arrays in rank order.  Any input the reference would
    reject is re-parsed by parse_merges so that exactly its exception (type and
    message) is raised; texts with line breaks other than "\n" also take the
    host parser (str.splitlines semantics).  Returns None for those."""
    import ctypes

    from . import _native

    if not isinstance(merges_text, (bytes, bytearray)):
        return None  # str input: the host parser (exact str semantics)
    text = bytes(merges_text)
    text.decode("utf-8")  # the reference decodes first: UnicodeDecodeError as there
    if any(b in text for b in _OTHER_BREAKS):
        return None
    arr = np.frombuffer(text, dtype=np.uint8)
    nl = np.flatnonzero(arr == 10).astype(np.uint64)
    starts = np.r_[np.uint64(0), nl + np.uint64(1)].astype(np.uint64)
    ends = np.r_[nl, np.uint64(len(text))].astype(np.uint64)
    if text.endswith(b"\n") or not text:  # splitlines: no empty last line
        starts, ends = starts[:-1], ends[:-1]
    if len(starts) and text[int(starts[0]):int(starts[0]) + 1] == b"#":
        starts, ends = starts[1:], ends[1:]
    n = len(starts)
    left = np.empty(n, np.uint32)
    right = np.empty(n, np.uint32)
    new = np.empty(n, np.uint32)
    status = np.zeros(n, np.uint8)
    blob, offs, ids = _symbol_csr(vocab)
    lib = _native.load()

    def ptr(a):
        return ctypes.c_void_p(a.ctypes.data) if a.size else None

    rc = lib.gpubpe_parse_merges(int(device), ptr(blob), ptr(offs), ptr(ids), len(ids), ptr(arr), len(text),
                                 ptr(starts), ptr(ends), n, ptr(left), ptr(right), ptr(new), ptr(status))
    _native.check(rc, None, "gpubpe_parse_merges")
    if status.any():
        parse_merges(text, vocab)  # raises the reference's error for the first bad line
        raise AssertionError("device merges parser rejected a line the host parser accepts")
    return left, right, np.arange(n, dtype=np.uint32), new


class ProbeScratch:
    """Reusable result buffers for repeated vectorised probes up to a fixed
    width (merge_table.py:119-137).  lookup_keys_into returns views of
    `hit` / `vals`; the other fields keep the reference's layout."""

    __slots__ = ("width", "idx", "tmp", "slots", "vals", "hit", "aux", "res")

    def __init__(self, width: int):
        self.width = width
        self.idx = np.empty(width, dtype=np.uint64)
        self.tmp = np.empty(width, dtype=np.uint64)
        self.slots = np.empty(width, dtype=np.uint64)
        self.vals = np.empty(width, dtype=np.uint64)
        self.hit = np.empty(width, dtype=bool)
        self.aux = np.empty(width, dtype=bool)
        self.res = np.empty(width, dtype=bool)


class PackedPairTable:
    """Open-addressing pair table with the reference's exact slot layout.
    `lookup` is the scalar host probe (construction / tests); the vectorised
    probes `lookup_keys_into` / `lookup_pairs` run on the device against the
    table's device context (engine._table_device, k_lookup_keys)."""

    __slots__ = ("keys", "values", "capacity", "count", "_mask")

    def __init__(self, keys: np.ndarray, values: np.ndarray, count: int):
        self.keys = keys
        self.values = values
        self.capacity = len(keys)
        self.count = count
        self._mask = self.capacity - 1

    def lookup(self, left: int, right: int):
        key = pack_key(left, right)
        if key == EMPTY_KEY:
            return None
        i = fmix64(key) & self._mask
        while True:
            k = int(self.keys[i])
            if k == key:
                return unpack_value(int(self.values[i]))
            if k == EMPTY_KEY:
                return None
            i = (i + 1) & self._mask

    def lookup_keys_into(self, probe_keys: np.ndarray, scratch: ProbeScratch):
        """Probe many packed keys at once (merge_table.py:170-230) on the device.
        Returns views (hit, values) of width len(probe_keys) into scratch;
        values are meaningful only where hit is True, and both views are
        overwritten by the next call.  The empty-slot key is always a miss."""
        from .engine import _table_device

        m = len(probe_keys)
        hit = scratch.hit[:m]
        vals = scratch.vals[:m]
        if m == 0:
            return hit, vals
        h, v = _table_device(self).lookup_keys(probe_keys)
        hit[:] = h
        vals[:] = v
        return hit, vals

    def lookup_pairs(self, left: np.ndarray, right: np.ndarray):
        """Vectorised probe (merge_table.py:232-243), on the device:
        (found bool[], new_tokens u64[], ranks u64[])."""
        n = len(left)
        keys = (np.asarray(left).astype(np.uint64) << np.uint64(32)) | np.asarray(right).astype(np.uint64)
        hit, vals = self.lookup_keys_into(keys, ProbeScratch(n))
        return hit, vals >> np.uint64(32), vals & np.uint64(U32_MASK)


def build_table(rules) -> PackedPairTable:
    count = len(rules)
    cap = 1
    while cap < 2 * count:
        cap <<= 1
    mask = cap - 1
    keys = [EMPTY_KEY] * cap
    vals = [0] * cap
    packed = [pack_key(r.left, r.right) for r in rules]
    homes = (fmix64_array(np.array(packed, dtype=np.uint64)) & np.uint64(mask)).tolist() if rules else []
    for rule, key, i in zip(rules, packed, homes):
        if key == EMPTY_KEY:
            raise ReservedKey(f"pair ({rule.left}, {rule.right}) packs to the empty-slot sentinel")
        while keys[i] != EMPTY_KEY:
            if keys[i] == key:
                raise DuplicatePair(
                    f"pair ({rule.left}, {rule.right}) already inserted at rank "
                    f"{vals[i] & U32_MASK}, duplicated at rank {rule.rank}")
            i = (i + 1) & mask
        keys[i] = key
        vals[i] = pack_value(rule.new_token, rule.rank)
    return PackedPairTable(np.array(keys, dtype=np.uint64), np.array(vals, dtype=np.uint64), count)


def rule_arrays(table) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """(left, right, rank, new) uint32 arrays recovered from a packed table,
    ordered by rank.  Works for this package's and the reference's tables."""
    keys = np.asarray(table.keys, dtype=np.uint64)
    vals = np.asarray(table.values, dtype=np.uint64)
    used = keys != np.uint64(EMPTY_KEY)
    k, v = keys[used], vals[used]
    order = np.argsort(v & np.uint64(U32_MASK), kind="stable")
    k, v = k[order], v[order]
    return ((k >> np.uint64(32)).astype(np.uint32), (k & np.uint64(U32_MASK)).astype(np.uint32),
            (v & np.uint64(U32_MASK)).astype(np.uint32), (v >> np.uint64(32)).astype(np.uint32))
