"""Host result-buffer pool of the host API (paper_2603_02597_b200/device.py):
size classes, the pinned-size limit, and the bound on pooled large buffers."""
import ctypes

import numpy as np

from paper_2603_02597_b200 import device


def test_size_classes():
    assert device._size_class(1) == 1 << 20
    assert device._size_class((1 << 20) + 1) == 2 << 20
    assert device._size_class(1 << 30) == 1 << 30
    # above 1 GiB: whole GiB, so a 43 GB result of a 10 GiB corpus shard pins 40 GiB, not 64
    assert device._size_class((1 << 30) + 1) == 2 << 30
    assert device._size_class(42_949_672_960 + 1) == 41 << 30


def test_pinned_limit_scales_with_local_ranks(monkeypatch):
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    one = device._pinned_limit()
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    eight = device._pinned_limit()
    assert one >= 8 << 30 and eight >= 8 << 30 and eight <= one


def test_pool_recycles_and_bounds_large_buffers():
    pool = device._HostPool()
    a = pool.take_pageable(3 << 20)
    assert a.size == 4 << 20
    pool.put(a)
    assert pool.take_pageable(3 << 20) is a  # recycled, pages already faulted in
    big1 = np.empty(300 << 20, np.uint8)
    big2 = np.empty(301 << 20, np.uint8)
    pool.put(big1)
    pool.put(big2)  # a second large class evicts the first
    assert [k for k in pool._free if k[0] > (256 << 20)] == [(big2.size, False)]
    raw = (ctypes.c_uint8 * 64)()
    pinned = np.frombuffer(raw, np.uint8)
    pool.put(pinned)  # pinned blocks (views of a ctypes array) are keyed apart
    assert (64, True) in pool._free
    # results handed out as views return their buffer when the last view dies
    buf = pool.take_pageable(1 << 20)
    view = pool.array(buf, np.uint32, 10)
    del view
    assert pool.take_pageable(1 << 20) is buf
