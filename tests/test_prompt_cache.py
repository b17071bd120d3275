"""Prompt-id-keyed shared cloud KV: host logic of
PromptKVCache over a PageAllocator — the reference's lookup/store semantics
(cloud.cpp:104-114: miss -> None, store is an emplace so the first entry
wins), plus what the B200 pool adds: session references, eviction that never
frees pages under a live session, and LRU make_room."""
import threading

import numpy as np
import pytest

from paper_2504_11729_b200._capi import InvalidArgument, OutOfMemory
from paper_2504_11729_b200.prompt_cache import PromptKVCache
from paper_2504_11729_b200.splice import PageAllocator


def _cache(n=16, P=64):
    a = PageAllocator(n)
    return PromptKVCache(allocator=a, page_tokens=P), a


def test_lookup_store_emplace():
    c, a = _cache()
    assert c.lookup(7) is None
    p = a.alloc(3)
    e = c.store(7, 150, p)
    a.release(p)                      # the producer drops its reference; the cache keeps one
    assert a.free_pages == 13 and 7 in c and len(c) == 1
    q = a.alloc(3)
    e2 = c.store(7, 150, q)           # emplace: existing entry wins
    assert e2 is e and np.array_equal(e2.pages, p)
    a.release(q)
    assert a.free_pages == 13
    hit = c.lookup(7)
    assert hit is e and all(a.refcount(int(x)) == 2 for x in p)
    c.release(hit)
    assert all(a.refcount(int(x)) == 1 for x in p)
    with pytest.raises(InvalidArgument):
        c.store(8, 200, a.alloc(1))   # 200 tokens need 4 pages


def test_evict_keeps_pages_of_live_sessions():
    c, a = _cache()
    p = a.alloc(2)
    c.store(1, 128, p)
    a.release(p)
    s = c.lookup(1)                   # a live session
    assert c.evict(1) and 1 not in c
    assert a.free_pages == 14         # still held by the session
    c.release(s)
    assert a.free_pages == 16
    assert not c.evict(1)


def test_make_room_lru_skips_busy_entries():
    c, a = _cache(n=8)
    ents = []
    for pid in range(4):
        p = a.alloc(2)
        ents.append(c.store(pid, 128, p))
        a.release(p)
    assert a.free_pages == 0
    busy = c.lookup(0)                # 0 is in use (and becomes most recent)
    c.lookup(1) and c.release(ents[1])  # touch 1 -> LRU order is 2, 3, 0, 1
    c.make_room(4)
    assert 2 not in c and 3 not in c and 0 in c and 1 in c
    with pytest.raises(OutOfMemory):
        c.make_room(7)                # 1 is idle and goes, 0 is busy: only 6 pages possible
    c.release(busy)


def test_concurrent_lookups_balance():
    c, a = _cache()
    p = a.alloc(4)
    c.store(3, 256, p)
    a.release(p)

    def worker():
        for _ in range(200):
            e = c.lookup(3)
            c.release(e)

    ts = [threading.Thread(target=worker) for _ in range(8)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert all(a.refcount(int(x)) == 1 for x in p)
