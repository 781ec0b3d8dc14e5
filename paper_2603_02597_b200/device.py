"""Device context: one per (tokenizer, GPU).  Wraps the C ABI of libgpubpe.so.

`DeviceEncoder` owns the device tables (pair table, rl/rr, junction bitmap,
memo) and the encode workspace.  Inputs and outputs are torch tensors only at
this boundary; the kernels see raw pointers.  There is no CPU path: every
method raises DeviceError when CUDA or the extension is unavailable.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native
from .errors import DeviceError, DuplicatePair, UnknownTokenId

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def _require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise DeviceError("the GPT-2 BPE engine needs a CUDA device (no CPU fallback)")


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


class _Lease:
    """A pooled host buffer lent to result arrays (PEP 688): numpy views of it
    keep it alive, and when the last one is released the buffer goes back to
    the pool instead of to the allocator."""

    __slots__ = ("buf", "pool")

    def __init__(self, buf: np.ndarray, pool: "_HostPool"):
        self.buf, self.pool = buf, pool

    def __buffer__(self, flags):
        return memoryview(self.buf)

    def __release_buffer__(self, view):
        try:
            self.pool.put(self.buf)
        except Exception:  # interpreter shutdown: nothing left to recycle into
            pass


class _PinnedBlock:
    """Owner of one gpubpe_host_alloc block (freed with the last reference)."""

    __slots__ = ("ptr", "lib")

    def __init__(self, ptr: int, lib):
        self.ptr, self.lib = ptr, lib

    def __del__(self):
        try:
            self.lib.gpubpe_host_free(ctypes.c_void_p(self.ptr))
        except Exception:
            pass


def _size_class(nbytes: int) -> int:
    """Power-of-two classes up to 1 GiB, then whole GiB (a 43 GB result of a
    10 GiB corpus shard must not pin 64 GiB)."""
    if nbytes <= 1 << 30:
        return 1 << max(20, int(nbytes - 1).bit_length())
    return -(-nbytes // (1 << 30)) << 30


def _pinned_limit() -> int:
    """Largest result buffer kept in pinned memory: a quarter of physical RAM
    split over the processes of this node (LOCAL_WORLD_SIZE), at least 8 GiB.
    Results beyond it are pageable, and the streamed native path stages
    their ids through its pinned slots (one host copy more)."""
    try:
        ram = os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError, AttributeError):  # pragma: no cover
        ram = 0
    lws = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1))
    return max(8 << 30, ram // (4 * lws))


class _HostPool:
    """Recycled result buffers: pinned and device-mapped (gpubpe_host_alloc),
    so the device writes the ids straight into them and nothing is copied out
    on the host; reused across calls, so neither pinning nor page faults are
    paid per call.  A buffer returns here when its last result array dies."""

    def __init__(self, keep: int = 4):
        self._free: dict[tuple[int, bool], list[np.ndarray]] = {}
        self._keep = keep
        self._lock = threading.Lock()
        self.pinned_max = _pinned_limit()

    def _pop(self, key):
        with self._lock:
            lst = self._free.get(key)
            return lst.pop() if lst else None

    def take(self, nbytes: int, lib, device: int) -> np.ndarray:
        cls = _size_class(nbytes)
        buf = self._pop((cls, True))
        if buf is not None:
            return buf
        p = ctypes.c_void_p()
        if lib.gpubpe_host_alloc(device, cls, ctypes.byref(p)) == _native.OK and p.value:
            raw = (ctypes.c_uint8 * cls).from_address(p.value)
            raw._owner = _PinnedBlock(p.value, lib)  # freed when the last view of raw dies
            return np.frombuffer(raw, dtype=np.uint8)
        return self.take_pageable(nbytes)  # pinned memory exhausted: the encode copies out

    def take_pageable(self, nbytes: int) -> np.ndarray:
        """A plain host buffer (for results too large to pin), recycled like the
        pinned ones so its pages are faulted in once, not on every call."""
        cls = _size_class(nbytes)
        buf = self._pop((cls, False))
        return buf if buf is not None else np.empty(cls, dtype=np.uint8)

    def put(self, buf: np.ndarray, _carray=ctypes.Array) -> None:
        # (_carray: bound at definition, as module globals may be gone when the last
        # result array dies at interpreter shutdown)
        key = (buf.size, isinstance(buf.base, _carray))  # pinned blocks are views of a ctypes array
        with self._lock:
            if buf.size > (256 << 20):
                # one large buffer of each kind at most: a run of calls whose sizes
                # land in different GiB classes must not pin several of them
                for k in [k for k in self._free if k[0] > (256 << 20) and k[1] == key[1] and k != key]:
                    del self._free[k]
            lst = self._free.setdefault(key, [])
            if len(lst) < (self._keep if buf.size <= (256 << 20) else 1):
                lst.append(buf)

    def array(self, buf: np.ndarray, dtype, count: int) -> np.ndarray:
        return np.frombuffer(_Lease(buf, self), dtype=dtype, count=count)


_RESULTS = _HostPool()
_POOLED_MAX = _RESULTS.pinned_max


def _result_buffer(nbytes: int, lib, device: int) -> np.ndarray:
    """The result buffer of one host encode: pinned up to _POOLED_MAX bytes."""
    nbytes = max(int(nbytes), 4)
    return (_RESULTS.take(nbytes, lib, device) if nbytes <= _POOLED_MAX
            else _RESULTS.take_pageable(nbytes))


def _hostlist():
    try:
        from . import _hostlist as hl  # csrc/hostlist.c, built in-tree with libgpubpe.so
    except ImportError as exc:
        raise DeviceError(f"host helper _hostlist not built ({exc}); run make -C csrc") from exc
    return hl


def bytes_ptrs_lens(parts: list) -> tuple[np.ndarray, np.ndarray]:
    """uint64 data addresses and lengths of a list of `bytes` objects (kept
    alive by the caller), read through the CPython C API in one call."""
    n = len(parts)
    ptrs = np.empty(n, dtype=np.uint64)
    lens = np.empty(n, dtype=np.uint64)
    if n:
        _hostlist().ptrs_lens(parts if type(parts) is list else list(parts), ptrs.ctypes.data, lens.ctypes.data)
    return ptrs, lens


def bytes_ptrs(parts: list) -> np.ndarray:
    """uint64 data addresses of a list of `bytes` objects (kept alive by the caller)."""
    return bytes_ptrs_lens(parts)[0]


def pinned_empty(nbytes: int, device: int = 0) -> np.ndarray:
    """uint8[nbytes] in pinned, device-mapped host memory (gpubpe_host_alloc),
    freed when the last view dies.  Input batches held here skip the staging
    copy of encode_packed_host / tokenize paths (the DMA reads them directly)."""
    _require_cuda()
    lib = _native.load()
    p = ctypes.c_void_p()
    rc = lib.gpubpe_host_alloc(int(device), max(int(nbytes), 1), ctypes.byref(p))
    if rc != _native.OK or not p.value:
        raise DeviceError(f"gpubpe_host_alloc({nbytes}) failed ({rc})")
    raw = (ctypes.c_uint8 * max(int(nbytes), 1)).from_address(p.value)
    raw._owner = _PinnedBlock(p.value, lib)
    return np.frombuffer(raw, dtype=np.uint8, count=int(nbytes))


class DeviceEncoder:
    """Device-resident tables for one merge table on one GPU."""

    def __init__(self, base_ids, left, right, rank, new, vocab_ids=None, vocab_blob=None,
                 vocab_offs=None, device: int | None = None, memo: bool = True,
                 strict: bool = False, host_tables: bool = False):
        _require_cuda()
        lib = _native.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        arrs = [np.ascontiguousarray(x, dtype=np.uint32) for x in (left, right, rank, new)]
        base = np.ascontiguousarray(base_ids, dtype=np.uint32)
        if vocab_ids is None:
            vocab_ids = np.empty(0, np.uint32)
            vocab_blob = np.empty(0, np.uint8)
            vocab_offs = np.zeros(1, np.uint64)
        vids = np.ascontiguousarray(vocab_ids, dtype=np.uint32)
        vblob = np.ascontiguousarray(vocab_blob, dtype=np.uint8)
        voffs = np.ascontiguousarray(vocab_offs, dtype=np.uint64)
        flags = ((0 if memo else _native.F_NO_MEMO) | (_native.F_STRICT if strict else 0)
                 | (_native.F_HOST_TABLES if host_tables else 0))
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            rc = lib.gpubpe_ctx_create(self.device, _ptr(base), *[_ptr(a) for a in arrs],
                                       len(arrs[0]), _ptr(vids), _ptr(vblob), _ptr(voffs),
                                       len(vids), flags, ctypes.byref(h))
        if rc != _native.OK:
            msg = lib.gpubpe_last_error(h).decode() if h.value else ""
            if h.value:
                lib.gpubpe_ctx_destroy(h)
            if rc == _native.ETABLE:
                raise DuplicatePair(msg)
            _native.check(rc, None, f"gpubpe_ctx_create: {msg}")
        self._h = h
        self._lib = lib
        self._lock = threading.RLock()  # decode_host -> decode_into re-enters
        self._pinned: dict[str, torch.Tensor] = {}

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.gpubpe_ctx_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ device API

    def encode_into(self, data: "torch.Tensor", doc_offs: "torch.Tensor", out_ids: "torch.Tensor",
                    out_offs: "torch.Tensor", max_seq_len: int, chunk_budget: int,
                    stream=None) -> None:
        """Enqueue one encode on `stream` (default: current).  All tensors on
        this device: data uint8[n], doc_offs int64[n_docs+1], out_ids
        int32[>= n], out_offs int64[n_docs+1].  Asynchronous."""
        n = data.numel()
        n_docs = doc_offs.numel() - 1
        if n_docs < 0:
            raise ValueError("doc_offs must hold n_docs + 1 entries")
        if out_ids.numel() < n or out_offs.numel() != n_docs + 1:
            raise ValueError("output tensors too small")
        for t, dt in ((data, torch.uint8), (doc_offs, torch.int64), (out_ids, torch.int32),
                      (out_offs, torch.int64)):
            if t.dtype != dt or not t.is_cuda or not t.is_contiguous() or t.device.index != self.device:
                raise ValueError(f"expected contiguous {dt} on cuda:{self.device}, got {t.dtype} {t.device}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self._lib.gpubpe_encode(self._h, data.data_ptr(), n, doc_offs.data_ptr(), n_docs,
                                     int(max_seq_len), int(chunk_budget), out_ids.data_ptr(),
                                     out_offs.data_ptr(), s.cuda_stream)
        _native.check(rc, self._h, "gpubpe_encode")

    # ------------------------------------------------------------ decode

    def set_vocab(self, ids: np.ndarray, blob: np.ndarray, offs: np.ndarray) -> None:
        """Byte strings of every decodable id (CSR) for the device decode."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        blob = np.ascontiguousarray(blob, dtype=np.uint8)
        offs = np.ascontiguousarray(offs, dtype=np.uint64)
        rc = self._lib.gpubpe_set_vocab(self._h, _ptr(ids), _ptr(blob), _ptr(offs), len(ids))
        _native.check(rc, self._h, "gpubpe_set_vocab")

    def decode_into(self, ids: "torch.Tensor", id_offs, out: "torch.Tensor", out_offs, stream=None) -> int:
        """Device CSR of ids -> device CSR of bytes; returns the bytes written.
        id_offs/out_offs: int64 [n_seqs+1] tensors, or None for one sequence.
        Raises UnknownTokenId, or ValueError when `out` is too small or a
        tensor has the wrong dtype / layout / device (ids int32 or uint32,
        out uint8, offsets int64; out 16-byte aligned)."""
        n = ids.numel()
        n_seqs = 0 if id_offs is None else id_offs.numel() - 1
        checks = [(ids, (torch.int32, torch.uint32)), (out, (torch.uint8,))]
        if n_seqs:
            checks += [(id_offs, (torch.int64,)), (out_offs, (torch.int64,))]
        for t, dts in checks:
            if t.dtype not in dts or not t.is_cuda or not t.is_contiguous() or t.device.index != self.device:
                raise ValueError(f"expected contiguous {dts} on cuda:{self.device}, got {t.dtype} {t.device}")
        if out.data_ptr() % 16:
            raise ValueError("decode_into: out must be 16-byte aligned")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        nb, bad = ctypes.c_uint64(0), ctypes.c_uint64(0)
        with self._lock:
            rc = self._decode_call(ids, n, id_offs, n_seqs, out, out_offs, nb, bad, s)
        if rc == _native.EINVAL and bad.value != (1 << 64) - 1:
            raise UnknownTokenId(f"id {int(ids[bad.value].item()) & 0xFFFFFFFF} at index {bad.value} "
                                 "not in vocabulary")
        if rc == _native.ERANGE:
            raise ValueError(f"decode output needs {nb.value} bytes, capacity {out.numel()}")
        _native.check(rc, self._h, "gpubpe_decode")
        return int(nb.value)

    def _decode_call(self, ids, n, id_offs, n_seqs, out, out_offs, nb, bad, s):
        return self._lib.gpubpe_decode(self._h, ids.data_ptr(), n, id_offs.data_ptr() if n_seqs else None,
                                     n_seqs, out.data_ptr(), out.numel(),
                                     out_offs.data_ptr() if n_seqs else None, ctypes.byref(nb),
                                     ctypes.byref(bad), s.cuda_stream)

    def decode_host(self, seqs) -> list[bytes]:
        """list of id sequences -> list of byte strings, decoded on the device."""
        arrs = [np.asarray(x, dtype=np.int64).ravel() for x in seqs]
        for a in arrs:
            if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
                bad = int(a[(a < 0) | (a > 0xFFFFFFFF)][0])
                raise UnknownTokenId(f"id {bad} not in vocabulary")
        offs = np.zeros(len(arrs) + 1, dtype=np.int64)
        if arrs:
            offs[1:] = np.cumsum([a.size for a in arrs])
        flat = np.concatenate(arrs).astype(np.uint32) if arrs else np.empty(0, np.uint32)
        with self._lock, torch.cuda.device(self.device):
            dev = torch.device("cuda", self.device)
            d_ids = torch.from_numpy(flat.view(np.int32) if flat.size else np.zeros(1, np.int32)).to(dev)
            d_offs = torch.from_numpy(offs).to(dev)
            d_oo = torch.empty_like(d_offs)
            cap = 8 * max(int(flat.size), 1) + 64
            for _ in range(2):
                d_out = torch.empty(cap, dtype=torch.uint8, device=dev)
                try:
                    nb = self.decode_into(d_ids[: flat.size], d_offs, d_out, d_oo)
                    break
                except ValueError as exc:  # capacity: re-run with the size the device asked for
                    cap = int(str(exc).split()[3]) + 64
            else:  # pragma: no cover
                raise DeviceError("decode capacity retry failed")
            out = d_out[:nb].cpu().numpy().tobytes()
            oo = d_oo.cpu().numpy()
        return [out[oo[i]:oo[i + 1]] for i in range(len(arrs))]

    def junction_bits(self) -> np.ndarray:
        """uint32[2048] junction bitmap (bit x << 8 | y: some rule joins x|y)."""
        out = np.zeros(2048, dtype=np.uint32)
        _native.check(self._lib.gpubpe_junction_bits(self._h, _ptr(out)), self._h, "junction_bits")
        return out

    def set_profiling(self, on: bool) -> None:
        _native.check(self._lib.gpubpe_set_profiling(self._h, int(on)), self._h, "set_profiling")

    def kernel_ms(self) -> float:
        """Duration (ms) of the encode kernel of the last profiled encode."""
        arr = (ctypes.c_float * 1)()
        _native.check(self._lib.gpubpe_kernel_ms(self._h, arr, 1), self._h, "kernel_ms")
        return float(arr[0])

    def query(self, stream=None) -> dict:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        st = _native.Stats()
        rc = self._lib.gpubpe_query(self._h, s.cuda_stream, ctypes.byref(st))
        _native.check(rc, self._h, "gpubpe_query")
        return st.as_dict()

    def encode_tensors(self, data, doc_offs, max_seq_len: int, chunk_budget: int):
        """Device CSR in -> device CSR out: (ids int32[total], offsets int64[n_docs+1]).
        Synchronises once (to learn the total)."""
        with self._lock, torch.cuda.device(self.device):
            n_docs = doc_offs.numel() - 1
            out_ids = torch.empty(max(data.numel(), 1), dtype=torch.int32, device=data.device)
            out_offs = torch.empty(n_docs + 1, dtype=torch.int64, device=data.device)
            self.encode_into(data, doc_offs, out_ids, out_offs, max_seq_len, chunk_budget)
            st = self.query()
            total = int(out_offs[-1].item()) if n_docs >= 0 and data.numel() else 0
            return out_ids[:total], out_offs, st

    def lookup_pairs(self, left: np.ndarray, right: np.ndarray):
        """(new uint32[], rank uint32[]) from the device table; rank 2**32-1 = miss."""
        with self._lock, torch.cuda.device(self.device):
            l = torch.from_numpy(np.ascontiguousarray(left, np.uint32).view(np.int32)).cuda()
            r = torch.from_numpy(np.ascontiguousarray(right, np.uint32).view(np.int32)).cuda()
            nw = torch.empty_like(l)
            rk = torch.empty_like(l)
            s = torch.cuda.current_stream()
            rc = self._lib.gpubpe_lookup_pairs(self._h, l.data_ptr(), r.data_ptr(), l.numel(),
                                               nw.data_ptr(), rk.data_ptr(), s.cuda_stream)
            _native.check(rc, self._h, "gpubpe_lookup_pairs")
            return nw.cpu().numpy().view(np.uint32), rk.cpu().numpy().view(np.uint32)

    # ------------------------------------------------------------ host API

    def set_mode(self, mode: int) -> None:
        """_native.MODE_DEFAULT or MODE_GPT2_REGEX (loads the class table on first use)."""
        if mode == _native.MODE_GPT2_REGEX and not getattr(self, "_pretok", False):
            from .pretok import N_CPS, gpt2_classes

            cls = gpt2_classes()
            _native.check(self._lib.gpubpe_set_pretok(self._h, _ptr(cls), N_CPS), self._h, "set_pretok")
            self._pretok = True
        _native.check(self._lib.gpubpe_set_mode(self._h, int(mode)), self._h, "set_mode")

    def encode_list_host(self, parts: list, max_seq_len: int, chunk_budget: int, mode: int = 0):
        """A batch of separate `bytes` documents -> host CSR (ids, offs, stats,
        engine_ms), gathered straight into the pinned staging buffer by the
        native side (gpubpe_encode_host_gather): no join on the Python side."""
        ptrs, lens = bytes_ptrs_lens(parts)  # TypeError unless every item is bytes
        return self.encode_ptrs_host(ptrs, lens, max_seq_len, chunk_budget, mode)

    def encode_ptrs_host(self, ptrs: np.ndarray, lens: np.ndarray, max_seq_len: int, chunk_budget: int,
                         mode: int = 0):
        """Documents given as host (address, length) pairs -- e.g. the chunks
        of longer documents -- gathered into pinned staging by the native
        side; the caller keeps the memory alive.  Same results as
        encode_list_host."""
        ptrs = np.ascontiguousarray(ptrs, dtype=np.uint64)
        lens = np.ascontiguousarray(lens, dtype=np.uint64)
        n_docs = len(lens)
        n = int(lens.sum())
        buf = _result_buffer(4 * n, self._lib, self.device)
        ids = buf.view(np.uint32)
        out_offs = np.zeros(n_docs + 1, dtype=np.int64)
        n_ids = ctypes.c_uint64(0)
        ms = ctypes.c_float(0.0)
        with self._lock, torch.cuda.device(self.device):
            if mode != _native.MODE_DEFAULT:
                self.set_mode(mode)
            s = torch.cuda.current_stream(self.device)
            try:
                rc = self._lib.gpubpe_encode_host_gather(self._h, _ptr(ptrs), _ptr(lens), n_docs, int(max_seq_len),
                                                         int(chunk_budget), _ptr(ids), _ptr(out_offs),
                                                         ctypes.byref(n_ids), ctypes.byref(ms), s.cuda_stream)
            finally:
                if mode != _native.MODE_DEFAULT:
                    self.set_mode(_native.MODE_DEFAULT)
            _native.check(rc, self._h, "gpubpe_encode_host_gather")
            st = self.query(s)
        return _RESULTS.array(buf, np.uint32, n_ids.value), out_offs, st, float(ms.value)

    def encode_bytes_host(self, doc: bytes, max_seq_len: int, chunk_budget: int):
        """One document (`bytes`) -> (ids uint32[], offs int64[units + 1], stats,
        engine_ms), default mode: the latency path as one C call
        (csrc/hostlist.c encode_one: the document's own buffer, its chunk
        offsets when len > max_seq_len, gpubpe_encode_host with the GIL
        released, gpubpe_query).  The current CUDA stream of this device."""
        n = len(doc)
        units = 1 if n <= max_seq_len else -(-n // int(chunk_budget))
        buf = _result_buffer(4 * n, self._lib, self.device)
        out_offs = np.empty(units + 1, dtype=np.int64)
        hl = _hostlist()
        if not getattr(hl, "_bound", False):
            hl.bind(ctypes.cast(self._lib.gpubpe_encode_host, ctypes.c_void_p).value,
                    ctypes.cast(self._lib.gpubpe_query, ctypes.c_void_p).value)
            hl._bound = True
        with self._lock:
            rc, n_ids, ms, st = hl.encode_one(self._h.value, doc, int(max_seq_len), int(chunk_budget),
                                              buf.ctypes.data, out_offs.ctypes.data, units,
                                              torch._C._cuda_getCurrentRawStream(self.device))
        _native.check(rc, self._h, "gpubpe_encode_host")
        return (_RESULTS.array(buf, np.uint32, n_ids), out_offs, _native.stats_dict(st), ms)

    def encode_packed_host(self, data: np.ndarray, offs: np.ndarray, max_seq_len: int,
                           chunk_budget: int, mode: int = 0):
        """Host CSR in -> host CSR out through gpubpe_encode_host (pinned
        staging, H2D, encode, D2H in one native call).  Returns (ids
        uint32[], offs int64[], stats, engine_ms)."""
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        n = int(data.size)
        n_docs = int(offs.size) - 1
        # large batches stream through the native pipeline, part by part: into
        # this buffer directly when pinned, else through its pinned slots
        buf = _result_buffer(4 * n, self._lib, self.device)
        ids = buf.view(np.uint32)
        out_offs = np.zeros(max(n_docs + 1, 1), dtype=np.int64)
        n_ids = ctypes.c_uint64(0)
        ms = ctypes.c_float(0.0)
        with self._lock, torch.cuda.device(self.device):
            if mode != _native.MODE_DEFAULT:
                self.set_mode(mode)
            s = torch.cuda.current_stream(self.device)
            try:
                rc = self._lib.gpubpe_encode_host(self._h, _ptr(data), n, _ptr(offs), n_docs,
                                                  int(max_seq_len), int(chunk_budget), _ptr(ids),
                                                  _ptr(out_offs), ctypes.byref(n_ids), ctypes.byref(ms),
                                                  s.cuda_stream)
            finally:
                if mode != _native.MODE_DEFAULT:
                    self.set_mode(_native.MODE_DEFAULT)
            _native.check(rc, self._h, "gpubpe_encode_host")
            st = self.query(s)
        return _RESULTS.array(buf, np.uint32, n_ids.value), out_offs[: n_docs + 1], st, float(ms.value)
