"""Prompt-id-keyed shared cloud KV.

The reference cloud keeps, per registered prompt id, the prompt's per-layer
KV segments once computed and serves later sessions from them
(CloudServer::lookup_cache / store_cache, /root/reference/proj/core/src/
cloud.cpp:104-114; used by serve_stream at :147-154; the map is
``std::map<uint32_t, shared_ptr<const vector<KVSegment>>>`` behind a mutex,
cloud.hpp:75-93). ``store`` is an emplace — an existing entry is kept.

Here an entry is a page list in the per-layer HBM pools (one shared page
numbering, ``PageAllocator``): every session's splice table references those
pages instead of copying the segments, which is exactly the shared-prefix
layout config 5 runs on (the planner detects the shared first segment and
takes the cascade path). ``lookup`` retains the pages for the session
(``release`` drops them), so an entry can be evicted — unlike the reference,
which never evicts — without pulling pages from under a live session.
"""
from __future__ import annotations

import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from ._capi import InvalidArgument, OutOfMemory


@dataclass(frozen=True)
class CachedPrompt:
    prompt_id: int
    seq_len: int
    pages: np.ndarray  # int32 page ids (same ids in every layer pool)


class PromptKVCache:
    """Prompt-id -> shared cloud-prompt pages over ``pools`` (one per layer,
    sharing one PageAllocator) or over a bare allocator (host logic only)."""

    def __init__(self, pools=None, allocator=None, page_tokens: int | None = None):
        if pools:
            allocator = pools[0].allocator
            page_tokens = pools[0].page_tokens
            for p in pools:
                if p.allocator is not allocator or p.page_tokens != page_tokens:
                    raise InvalidArgument("PromptKVCache: layer pools must share one allocator "
                                          "and page size")
        if allocator is None or page_tokens is None:
            raise InvalidArgument("PromptKVCache: pools or (allocator, page_tokens) required")
        self.pools = list(pools or [])
        self.allocator = allocator
        self.page_tokens = page_tokens
        self._mu = threading.RLock()
        self._entries: OrderedDict[int, CachedPrompt] = OrderedDict()  # LRU order
        self._sessions: dict[int, int] = {}

    # ----------------------------------------------------- reference API --
    def lookup(self, prompt_id: int) -> CachedPrompt | None:
        """cloud.cpp:104-108. A hit retains the pages for the caller's session."""
        with self._mu:
            e = self._entries.get(prompt_id)
            if e is None:
                return None
            self._entries.move_to_end(prompt_id)
            self.allocator.retain(e.pages)
            self._sessions[prompt_id] += 1
            return e

    def store(self, prompt_id: int, seq_len: int, pages) -> CachedPrompt:
        """cloud.cpp:110-114 (emplace): the cache takes a reference to
        ``pages``; if the id is already cached the existing entry wins and is
        returned (the caller keeps its own pages)."""
        pages = np.ascontiguousarray(pages, dtype=np.int32)
        if pages.size < -(-seq_len // self.page_tokens):
            raise InvalidArgument(f"PromptKVCache.store: {seq_len} tokens need "
                                  f"{-(-seq_len // self.page_tokens)} pages, got {pages.size}")
        with self._mu:
            e = self._entries.get(prompt_id)
            if e is not None:
                return e
            self.allocator.retain(pages)
            e = CachedPrompt(prompt_id, int(seq_len), pages.copy())
            self._entries[prompt_id] = e
            self._sessions[prompt_id] = 0
            return e

    # ------------------------------------------------------------ B200 ----
    def release(self, entry: CachedPrompt) -> None:
        """A session that got ``entry`` from lookup() is done with it."""
        with self._mu:
            if self._sessions.get(entry.prompt_id, 0) > 0:
                self._sessions[entry.prompt_id] -= 1
            self.allocator.release(entry.pages)

    def evict(self, prompt_id: int) -> bool:
        """Drops the cache's reference; pages return to the pool when the last
        session using them releases. False if not cached."""
        with self._mu:
            e = self._entries.pop(prompt_id, None)
            if e is None:
                return False
            self._sessions.pop(prompt_id, None)
            self.allocator.release(e.pages)
            return True

    def make_room(self, n_pages: int) -> None:
        """Evicts least-recently-used entries without live sessions until
        ``n_pages`` are free; OutOfMemory if that is impossible."""
        with self._mu:
            for pid in list(self._entries):
                if self.allocator.free_pages >= n_pages:
                    break
                if self._sessions.get(pid, 0) == 0:
                    e = self._entries.pop(pid)
                    self._sessions.pop(pid, None)
                    self.allocator.release(e.pages)
            if self.allocator.free_pages < n_pages:
                raise OutOfMemory(f"PromptKVCache: {n_pages} pages needed, "
                                  f"{self.allocator.free_pages} free after eviction")

    def reserve(self, n_pages: int) -> np.ndarray:
        """make_room + alloc under one lock: no other thread can take the
        pages that eviction freed before this caller allocates them."""
        with self._mu:
            self.make_room(n_pages)
            return self.allocator.alloc(n_pages)

    def ingest(self, prompt_id: int, frames, handle=None, stream=None) -> CachedPrompt:
        """Stores a prompt whose per-layer KV arrives as EPKV kv frames (one
        per layer pool, layer order — the cloud's serve_stream output,
        cloud.cpp:155-172): pages are allocated once (LRU eviction if needed),
        each frame is decoded into its layer's pool (ep_kv_ingest_frame), and
        the entry is stored. If the id is cached meanwhile, that entry wins."""
        if len(frames) != len(self.pools):
            raise InvalidArgument(f"PromptKVCache.ingest: {len(frames)} frames for "
                                  f"{len(self.pools)} layers")
        hit = self.lookup(prompt_id)
        if hit is not None:
            self.release(hit)
            return hit
        pages = None
        seq_len = None
        kept = False  # our pages became the stored entry
        try:
            for layer, (pool, frame) in enumerate(zip(self.pools, frames)):
                if pages is None:
                    seq_len = _frame_seq_len(frame)
                    pages = self.reserve(-(-seq_len // self.page_tokens))
                info = pool.ingest_frame(frame, pages, handle=handle, stream=stream)
                if info.seq_len != seq_len:
                    raise InvalidArgument("PromptKVCache.ingest: sequence length changed between "
                                          "layers (edge.cpp:150-152)")
                if info.layer != layer:
                    raise InvalidArgument(f"PromptKVCache.ingest: frame for layer {info.layer} "
                                          f"arrived out of order, expected {layer}")
            e = self.store(prompt_id, seq_len, pages)
            kept = e.pages is not pages and np.array_equal(e.pages, pages)
            return e
        finally:
            if pages is not None:
                if not kept:
                    # the pages go back to the free list while ingest kernels
                    # may still be writing them: wait for the stream first
                    _sync(stream)
                self.allocator.release(pages)  # the entry (if stored) holds its own reference

    def __contains__(self, prompt_id: int) -> bool:
        with self._mu:
            return prompt_id in self._entries

    def __len__(self) -> int:
        with self._mu:
            return len(self._entries)


def _sync(stream) -> None:
    import torch
    if stream is None:
        torch.cuda.current_stream().synchronize()
    elif hasattr(stream, "synchronize"):
        stream.synchronize()
    else:
        torch.cuda.synchronize()


def _frame_seq_len(frame) -> int:
    """seq_len field of a kv frame (payload offset 6, wire.cpp:98-104)."""
    head = bytes(np.asarray(frame[:24].cpu() if hasattr(frame, "cpu") else frame[:24],
                            dtype=np.uint8).tobytes())
    if len(head) < 24:
        raise InvalidArgument("PromptKVCache.ingest: frame shorter than a kv frame header")
    return int.from_bytes(head[16:20], "little")
