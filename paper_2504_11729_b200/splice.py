"""Device-resident paged KV store and splice tables.

The reference keeps, per session and per layer, an ordered list of fp64
``KVSegment`` s (cloud -> edge -> generated, gapless positions;
/root/reference/proj/core/include/edgeprompt/cache.hpp:11-61,
src/cache.cpp:25-103) and copies the whole generated segment on every decoded
token (cache.cpp:55-80). Here:

* ``KVPool``      — one HBM page pool per layer: K and V as
  ``[num_pages][n_kv_heads][page_tokens][d_head]`` (bf16 or fp32). A page is
  one contiguous ``page_tokens x d_head`` tile per kv-head, so the decode
  kernel streams it with a single bulk-async copy. Pages are refcounted, so a
  cloud-prompt segment is written once and referenced by every request's
  splice table (config 5).
* ``SpliceTable`` — per-request ordered segment descriptors (``ep_segment``)
  over pool pages, with the reference's append invariants (gapless positions,
  origin order, atomic validation) and O(1) token append into the trailing
  generated segment's last page.
* ``SplicedAttention`` — an ``ep_plan`` over (pool, table): the K1+K2 launch.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import InvalidArgument, KVPoolDesc, check, lib
from .attention import Handle, default_handle

ORIGIN_CLOUD, ORIGIN_EDGE, ORIGIN_GENERATED = 0, 1, 2  # SegmentOrigin (cache.hpp:11)
_ORIGIN_NAMES = {0: "cloud", 1: "edge", 2: "generated"}

SEGMENT_DTYPE = np.dtype([("origin", "<i4"), ("len", "<i4"), ("pos_offset", "<i8"),
                          ("page_off", "<i8")])
assert SEGMENT_DTYPE.itemsize == C.sizeof(_capi.Segment)


def _torch():
    import torch
    return torch


def dtype_code(dtype) -> int:
    torch = _torch()
    if dtype in ("bf16", torch.bfloat16):
        return _capi.EP_BF16
    if dtype in ("f32", "fp32", torch.float32):
        return _capi.EP_F32
    raise _capi.Unsupported(f"KV dtype {dtype!r}: expected bf16 or fp32")


class PageAllocator:
    """Refcounted page ids of a pool (or of several per-layer pools that share
    one page numbering: a page id then names the same slot in every layer)."""

    def __init__(self, num_pages: int):
        self.num_pages = num_pages
        self._free = list(range(num_pages - 1, -1, -1))
        self._ref = np.zeros(num_pages, dtype=np.int32)

    def alloc(self, n: int) -> np.ndarray:
        if n > len(self._free):
            raise _capi.OutOfMemory(f"KVPool: {n} pages requested, {len(self._free)} free")
        pages = np.array([self._free.pop() for _ in range(n)], dtype=np.int32)
        self._ref[pages] = 1
        return pages

    def retain(self, pages) -> None:
        self._ref[np.asarray(pages)] += 1

    def release(self, pages) -> None:
        for p in np.asarray(pages).tolist():
            if self._ref[p] <= 0:
                raise InvalidArgument(f"PageAllocator: page {p} released more often than retained")
            self._ref[p] -= 1
            if self._ref[p] == 0:
                self._free.append(p)

    def refcount(self, page: int) -> int:
        return int(self._ref[page])

    @property
    def free_pages(self) -> int:
        return len(self._free)


class KVPool:
    """Paged K/V pool in HBM for one layer (ep_kv_pool)."""

    def __init__(self, num_pages: int, n_kv_heads: int, d_head: int, page_tokens: int = 64,
                 dtype="bf16", device: int | None = None, k=None, v=None,
                 allocator: PageAllocator | None = None):
        torch = _torch()
        self.code = dtype_code(dtype)
        self.tdtype = torch.bfloat16 if self.code == _capi.EP_BF16 else torch.float32
        self.num_pages, self.n_kv_heads, self.d_head = num_pages, n_kv_heads, d_head
        self.page_tokens = page_tokens
        shape = (num_pages, n_kv_heads, page_tokens, d_head)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.k = k if k is not None else torch.zeros(shape, dtype=self.tdtype, device=dev)
        self.v = v if v is not None else torch.zeros(shape, dtype=self.tdtype, device=dev)
        assert tuple(self.k.shape) == shape and tuple(self.v.shape) == shape
        if allocator is not None and allocator.num_pages != num_pages:
            raise InvalidArgument("KVPool: shared allocator has a different page count")
        self.allocator = allocator or PageAllocator(num_pages)

    # --------------------------------------------------------- allocator --
    def alloc(self, n: int) -> np.ndarray:
        return self.allocator.alloc(n)

    def retain(self, pages) -> None:
        self.allocator.retain(pages)

    def release(self, pages) -> None:
        self.allocator.release(pages)

    @property
    def free_pages(self) -> int:
        return self.allocator.free_pages

    # ------------------------------------------------------------ writes --
    def write(self, pages, k, v, start: int = 0) -> None:
        """Scatter token rows k/v [len][n_kv_heads][d_head] into ``pages``,
        starting at token slot ``start`` of the first page."""
        torch = _torch()
        n = int(k.shape[0])
        if n == 0:
            return
        t = torch.arange(start, start + n, device=self.k.device)
        pg = torch.as_tensor(np.asarray(pages, dtype=np.int64), device=self.k.device)
        pidx = pg[t // self.page_tokens]
        sidx = t % self.page_tokens
        self.k[pidx, :, sidx, :] = k.to(self.tdtype)
        self.v[pidx, :, sidx, :] = v.to(self.tdtype)

    def ingest_frame(self, frame, pages, handle: Handle | None = None, stream=None):
        """Decodes one EPKV kv frame (the reference's encode_frame bytes,
        wire.cpp:70-136) straight into ``pages`` (ep_kv_ingest_frame): frame
        token t -> pages[t // page_tokens], slot t % page_tokens, values rounded
        to the pool dtype. ``frame``: bytes / uint8 numpy (pageable, staged),
        a pinned uint8 CPU tensor (read in place by the kernel) or a uint8
        CUDA tensor. Returns the frame info (session_id, layer, seq_len, ...).
        Raises WireError (``.kind``) for malformed frames like decode_frame."""
        torch = _torch()
        handle = handle or default_handle(self.k.device.index or 0)
        if isinstance(frame, (bytes, bytearray)):
            frame = np.frombuffer(frame, dtype=np.uint8)
        if isinstance(frame, np.ndarray):
            frame = np.ascontiguousarray(frame, dtype=np.uint8)
            ptr, nbytes = frame.ctypes.data, frame.size
        else:
            assert frame.dtype == torch.uint8 and frame.is_contiguous()
            ptr, nbytes = frame.data_ptr(), frame.numel()
        if isinstance(pages, torch.Tensor) and pages.is_cuda:
            pt = pages.to(torch.int32).contiguous()
        else:
            pt = torch.as_tensor(np.asarray(pages, dtype=np.int32), device=self.k.device)
        self._ingest_keep = (frame, pt)
        info = _capi.KVFrameInfo()
        pd = self.desc()
        rc = lib().ep_kv_ingest_frame(handle.ptr, C.byref(pd), ptr, nbytes, pt.data_ptr(),
                                      int(pt.numel()), C.byref(info), _stream(stream))
        if rc == _capi.EP_EWIRE:
            err = _capi.WireError("ep_kv_ingest_frame: " + lib().ep_last_error().decode())
            err.kind = int(info.wire_error)
            raise err
        check(rc, "ep_kv_ingest_frame")
        return info

    def ingest_frame_async(self, frame, pages, handle: Handle | None = None, stream=None):
        """ingest_frame for a device-resident frame without a host sync
        (ep_kv_ingest_frame_async): the header is checked by the kernel and a
        failure surfaces at the next ``ingest_poll``. Host frames and frames
        whose length does not fit the pool's head shape fail immediately."""
        torch = _torch()
        handle = handle or default_handle(self.k.device.index or 0)
        assert isinstance(frame, torch.Tensor) and frame.dtype == torch.uint8 and frame.is_contiguous()
        if isinstance(pages, torch.Tensor) and pages.is_cuda:
            pt = pages.to(torch.int32).contiguous()
        else:
            pt = torch.as_tensor(np.asarray(pages, dtype=np.int32), device=self.k.device)
        self._ingest_keep = (frame, pt)
        pd = self.desc()
        rc = lib().ep_kv_ingest_frame_async(handle.ptr, C.byref(pd), frame.data_ptr(), frame.numel(),
                                            pt.data_ptr(), int(pt.numel()), _stream(stream))
        if rc == _capi.EP_EWIRE:
            raise _capi.WireError("ep_kv_ingest_frame_async: " + lib().ep_last_error().decode())
        check(rc, "ep_kv_ingest_frame_async")

    @staticmethod
    def ingest_poll(handle: Handle | None = None, stream=None):
        """Synchronises ``stream`` and raises the first deferred kv frame
        failure since the last poll (WireError with ``.kind`` and ``.info``,
        or InvalidArgument); returns None when every frame was valid."""
        handle = handle or default_handle()
        info = _capi.KVFrameInfo()
        rc = lib().ep_kv_ingest_poll(handle.ptr, _stream(stream), C.byref(info))
        if rc == _capi.EP_EWIRE:
            err = _capi.WireError("ep_kv_ingest_poll: " + lib().ep_last_error().decode())
            err.kind = int(info.wire_error)
            err.info = info
            raise err
        check(rc, "ep_kv_ingest_poll")

    def desc(self) -> KVPoolDesc:
        return KVPoolDesc(self.code, self.n_kv_heads, self.d_head, self.page_tokens,
                          self.num_pages, self.k.data_ptr(), self.v.data_ptr())

    def host_raw(self):
        """(k, v) as numpy (fp32 or raw-bf16 uint16) for the CPU oracle."""
        torch = _torch()
        if self.code == _capi.EP_BF16:
            return (self.k.view(torch.int16).cpu().numpy().view(np.uint16),
                    self.v.view(torch.int16).cpu().numpy().view(np.uint16))
        return self.k.cpu().numpy(), self.v.cpu().numpy()


@dataclass
class SegmentRef:
    origin: int
    pos_offset: int
    length: int
    pages: np.ndarray  # int32 page ids

    @property
    def end_position(self) -> int:
        return self.pos_offset + self.length


class SpliceTable:
    """Ordered segment lists for a batch of requests (SegmentedCache analogue)."""

    def __init__(self, batch: int, page_tokens: int = 64):
        self.page_tokens = page_tokens
        self.requests: list[list[SegmentRef]] = [[] for _ in range(batch)]
        self.q_pos = np.zeros(batch, dtype=np.int64)

    @property
    def batch(self) -> int:
        return len(self.requests)

    def end_position(self, b: int) -> int:
        segs = self.requests[b]
        return segs[-1].end_position if segs else 0

    def append(self, b: int, origin: int, pos_offset: int, length: int, pages) -> None:
        """SegmentedCache::append invariants (cache.cpp:25-53), validated
        before any mutation."""
        pages = np.asarray(pages, dtype=np.int32)
        end = self.end_position(b)
        # A request's first segment may start past 0: a rank of the split-KV
        # path holds a contiguous window of the global cache (splitkv.py).
        if self.requests[b] and pos_offset != end:
            raise InvalidArgument(f"SpliceTable.append: segment starts at {pos_offset}, "
                                  f"cache ends at {end}")
        if length <= 0:
            raise InvalidArgument("SpliceTable.append: empty segment")
        need = -(-length // self.page_tokens)
        if pages.size < need:
            raise InvalidArgument(f"SpliceTable.append: {length} tokens need {need} pages, "
                                  f"got {pages.size}")
        segs = self.requests[b]
        if segs and origin < segs[-1].origin:
            raise InvalidArgument("SpliceTable.append: origin order must be (cloud, edge, "
                                  "generated)")
        segs.append(SegmentRef(origin, pos_offset, length, pages[:need].copy()))

    def append_generated_tokens(self, b: int, n: int, pool: KVPool | None = None):
        """Grows the trailing generated segment by n tokens (cache.cpp:55-80)
        without copying: new tokens go to the last page's free slots or a fresh
        page. Returns (pages, start_slot) where the caller writes the K/V rows."""
        segs = self.requests[b]
        pos = self.end_position(b)
        P = self.page_tokens
        if not segs or segs[-1].origin != ORIGIN_GENERATED:
            if pool is None:
                raise InvalidArgument("append_generated_tokens: pool needed for a new page")
            pages = pool.alloc(-(-n // P))
            segs.append(SegmentRef(ORIGIN_GENERATED, pos, n, pages))
            return pages, 0
        g = segs[-1]
        start = g.length % P
        have = g.pages.size * P - g.length
        if n > have:
            if pool is None:
                raise InvalidArgument("append_generated_tokens: pool needed for a new page")
            extra = pool.alloc(-(-(n - have) // P))
            g.pages = np.concatenate([g.pages, extra])
        first = g.length // P
        g.length += n
        return g.pages[first:], start

    def check_consistent(self) -> str:
        """cache.cpp:82-103 restricted to one layer: gapless, origin order."""
        for b, segs in enumerate(self.requests):
            pos, last = None, -1
            for s in segs:
                if pos is not None and s.pos_offset != pos:
                    return f"request {b}: gap in position coverage"
                if s.origin < last:
                    return f"request {b}: origin order violated"
                pos, last = s.end_position, s.origin
        return ""

    def arrays(self):
        """(seg_indptr int64 [B+1], segs SEGMENT_DTYPE, page_table int32)."""
        indptr = np.zeros(self.batch + 1, dtype=np.int64)
        recs = []
        pages = []
        off = 0
        for b, segs in enumerate(self.requests):
            for s in segs:
                recs.append((s.origin, s.length, s.pos_offset, off))
                pages.append(s.pages)
                off += s.pages.size
            indptr[b + 1] = len(recs)
        segs_arr = np.array(recs, dtype=SEGMENT_DTYPE) if recs else np.zeros(0, SEGMENT_DTYPE)
        pt = np.concatenate(pages).astype(np.int32) if pages else np.zeros(1, np.int32)
        return indptr, segs_arr, np.ascontiguousarray(pt)


class SpliceCache:
    """ep_cache — SegmentedCache (cache.hpp:30-61, cache.cpp:16-103) as the
    library's own host object for a batch of sessions over paged KV: per
    layer and request an ordered segment list {origin, pos_offset, len,
    pages}. Plans read it directly (SplicedAttention.from_cache), so growing
    every session by one token per step costs a C++ rebuild, not Python."""

    def __init__(self, n_layers: int, batch: int, page_tokens: int = 64):
        c = C.c_void_p()
        check(lib().ep_cache_create(n_layers, batch, page_tokens, C.byref(c)), "ep_cache_create")
        self._c = c
        self.n_layers, self.batch, self.page_tokens = n_layers, batch, page_tokens

    @property
    def ptr(self):
        return self._c

    def end_position(self, b: int) -> int:
        return int(lib().ep_cache_end_position(self._c, b))

    def append(self, b: int, origin: int, pos_offset: int, length: int, pages, layer: int = -1) -> None:
        """SegmentedCache::append (cache.cpp:25-53), validated then applied;
        layer = -1: every layer (shared page ids)."""
        pg = np.ascontiguousarray(pages, dtype=np.int32)
        check(lib().ep_cache_append(self._c, layer, b, origin, pos_offset, length,
                                    pg.ctypes.data if pg.size else None, int(pg.size)), "ep_cache_append")

    def append_generated(self, n_tokens, new_pages=None, out=None):
        """append_generated_token (cache.cpp:55-80) for the batch: request b
        grows by n_tokens[b]; new_pages [B][max_new] supplies pages when the
        last page is full. Returns (dst_page, dst_slot, pages_used); out =
        (dst_page, dst_slot) int32 arrays to fill (e.g. pinned staging)."""
        n = np.ascontiguousarray(n_tokens, dtype=np.int32)
        assert n.size == self.batch
        npg = (np.ascontiguousarray(new_pages, dtype=np.int32).reshape(self.batch, -1)
               if new_pages is not None else np.zeros((self.batch, 0), np.int32))
        if out is not None:
            dst_page, dst_slot = out
        else:
            dst_page = np.zeros(max(1, int(n.sum())), np.int32)
            dst_slot = np.zeros_like(dst_page)
        used = np.zeros(self.batch, np.int32)
        check(lib().ep_cache_append_generated(self._c, n.ctypes.data, npg.ctypes.data if npg.size else None,
                                              int(npg.shape[1]), dst_page.ctypes.data, dst_slot.ctypes.data,
                                              used.ctypes.data), "ep_cache_append_generated")
        k = int(n.sum())
        return dst_page[:k], dst_slot[:k], used

    def truncate(self, b: int, n_tokens: int) -> np.ndarray:
        """Drops the last n_tokens generated tokens of request b (rejected
        drafts); returns the pages no longer used."""
        rel = np.zeros(max(1, -(-n_tokens // self.page_tokens) + 1), np.int32)
        nr = C.c_int32()
        check(lib().ep_cache_truncate(self._c, b, n_tokens, rel.ctypes.data, C.byref(nr)), "ep_cache_truncate")
        return rel[:nr.value].copy()

    def check_consistent(self) -> str:
        """cache.cpp:82-103: '' when consistent, else the reason."""
        rc = lib().ep_cache_check_consistent(self._c)
        return "" if rc == 0 else lib().ep_last_error().decode()

    def arrays(self, layer: int = 0):
        """(seg_indptr, segs, page_table) of one layer (ep_plan_create layout)."""
        ns, npg = C.c_int64(), C.c_int64()
        check(lib().ep_cache_layer_arrays(self._c, layer, None, None, 0, None, 0, C.byref(ns), C.byref(npg)),
              "ep_cache_layer_arrays")
        indptr = np.zeros(self.batch + 1, np.int64)
        segs = np.zeros(max(1, ns.value), SEGMENT_DTYPE)
        pt = np.zeros(max(1, npg.value), np.int32)
        check(lib().ep_cache_layer_arrays(self._c, layer, indptr.ctypes.data, segs.ctypes.data, segs.size,
                                          pt.ctypes.data, pt.size, C.byref(ns), C.byref(npg)),
              "ep_cache_layer_arrays")
        return indptr, segs[:ns.value], pt[:npg.value]

    def close(self):
        if getattr(self, "_c", None) is not None and self._c.value:
            lib().ep_cache_destroy(self._c)
        self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SplicedAttention:
    """ep_plan over (pool, table): spliced attention for every request."""

    def __init__(self, pool: KVPool, table: SpliceTable, n_q_heads: int, n_q: int = 1,
                 handle: Handle | None = None):
        self.pool, self.table = pool, table
        self.n_q_heads, self.n_q = n_q_heads, n_q
        self.handle = handle or default_handle(pool.k.device.index or 0)
        self._keep = None
        indptr, segs, pt = table.arrays()
        self._keep = (indptr, segs, pt, np.ascontiguousarray(table.q_pos, dtype=np.int64))
        plan = C.c_void_p()
        pd = pool.desc()
        check(lib().ep_plan_create(self.handle.ptr, C.byref(pd), n_q_heads, n_q, table.batch,
                                   indptr.ctypes.data, segs.ctypes.data, pt.ctypes.data,
                                   self._keep[3].ctypes.data, 0, C.byref(plan)),
              "ep_plan_create")
        self.plan = plan

    @classmethod
    def from_cache(cls, pool: KVPool, cache: SpliceCache, n_q_heads: int, n_q: int = 1, layer: int = 0,
                   handle: Handle | None = None) -> "SplicedAttention":
        """Plan straight from an ep_cache (ep_plan_create_cache): request b's
        queries are its last n_q positions. update_from_cache() re-plans after
        the cache grew (one C++ rebuild + an async upload per step)."""
        self = cls.__new__(cls)
        self.pool, self.table, self.cache, self.layer = pool, None, cache, layer
        self.n_q_heads, self.n_q = n_q_heads, n_q
        self.handle = handle or default_handle(pool.k.device.index or 0)
        self._keep = None
        plan = C.c_void_p()
        pd = pool.desc()
        check(lib().ep_plan_create_cache(self.handle.ptr, C.byref(pd), cache.ptr, layer, n_q_heads, n_q,
                                         C.byref(plan)), "ep_plan_create_cache")
        self.plan = plan
        return self

    def update_from_cache(self, stream=None) -> None:
        check(lib().ep_plan_update_cache(self.plan, self.cache.ptr, self.layer, self.n_q, _stream(stream)),
              "ep_plan_update_cache")

    @property
    def batch(self) -> int:
        return self.table.batch if self.table is not None else self.cache.batch

    def update(self, stream=None) -> None:
        """Re-plan after the table changed (ep_plan_update, stream-ordered)."""
        indptr, segs, pt = self.table.arrays()
        self._keep = (indptr, segs, pt, np.ascontiguousarray(self.table.q_pos, dtype=np.int64))
        check(lib().ep_plan_update(self.plan, indptr.ctypes.data, segs.ctypes.data,
                                   pt.ctypes.data, self._keep[3].ctypes.data,
                                   _stream(stream)), "ep_plan_update")

    def info(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().ep_plan_info(self.plan, C.byref(a), C.byref(b), C.byref(c)), "ep_plan_info")
        return a.value, b.value, c.value

    def __call__(self, q, o=None, lse=None, o_dtype=None, stream=None):
        """q [B][n_q][Hq][d] (bf16/fp32 CUDA tensor) -> (o, lse)."""
        torch = _torch()
        B, d = self.batch, self.pool.d_head
        if tuple(q.shape) != (B, self.n_q, self.n_q_heads, d) or not q.is_contiguous():
            raise InvalidArgument(f"SplicedAttention: q must be contiguous "
                                  f"[{B}][{self.n_q}][{self.n_q_heads}][{d}]")
        if o is None:
            o = torch.empty(q.shape, dtype=o_dtype or q.dtype, device=q.device)
        if lse is None:
            lse = torch.empty((B, self.n_q, self.n_q_heads), dtype=torch.float32, device=q.device)
        pd = self.pool.desc()
        check(lib().ep_spliced_attention(self.handle.ptr, self.plan, C.byref(pd),
                                         dtype_code(q.dtype), q.data_ptr(), dtype_code(o.dtype),
                                         o.data_ptr(), lse.data_ptr() if lse is not False else None,
                                         _stream(stream)), "ep_spliced_attention")
        return o, lse

    def close(self):
        if getattr(self, "plan", None):
            lib().ep_plan_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SplicedPrefill:
    """Prefill attention over (pool, table) on the tensor cores
    (ep_plan_create_prefill): the last n_new[b] tokens of request b attend
    causally to everything up to themselves — the cloud-prompt prefill
    (n_new = whole prompt) and the edge prefill against a cloud segment
    (edge.cpp:148-164) alike. The new tokens' K/V must already be written into
    the table's pages. q / o: [sum n_new][n_q_heads][d] token-major."""

    def __init__(self, pool: KVPool, table: SpliceTable, n_q_heads: int, n_new,
                 handle: Handle | None = None):
        self.pool, self.table, self.n_q_heads = pool, table, n_q_heads
        self.handle = handle or default_handle(pool.k.device.index or 0)
        self.n_new = np.ascontiguousarray(np.asarray(n_new, dtype=np.int32).reshape(table.batch))
        self.n_tokens = int(self.n_new.sum())
        indptr, segs, pt = table.arrays()
        self._keep = (indptr, segs, pt, self.n_new)
        plan = C.c_void_p()
        pd = pool.desc()
        check(lib().ep_plan_create_prefill(self.handle.ptr, C.byref(pd), n_q_heads, table.batch,
                                           indptr.ctypes.data, segs.ctypes.data, pt.ctypes.data,
                                           self.n_new.ctypes.data, C.byref(plan)),
              "ep_plan_create_prefill")
        self.plan = plan

    def __call__(self, q, o=None, lse=None, o_dtype=None, stream=None):
        """q [sum n_new][Hq][d] (bf16/fp32 CUDA tensor) -> (o, lse)."""
        torch = _torch()
        d = self.pool.d_head
        if tuple(q.shape) != (self.n_tokens, self.n_q_heads, d) or not q.is_contiguous():
            raise InvalidArgument(f"SplicedPrefill: q must be contiguous "
                                  f"[{self.n_tokens}][{self.n_q_heads}][{d}]")
        if o is None:
            o = torch.empty(q.shape, dtype=o_dtype or q.dtype, device=q.device)
        if lse is None:
            lse = torch.empty((self.n_tokens, self.n_q_heads), dtype=torch.float32, device=q.device)
        pd = self.pool.desc()
        check(lib().ep_spliced_attention(self.handle.ptr, self.plan, C.byref(pd),
                                         dtype_code(q.dtype), q.data_ptr(), dtype_code(o.dtype),
                                         o.data_ptr(), lse.data_ptr() if lse is not False else None,
                                         _stream(stream)), "ep_spliced_attention")
        return o, lse

    def info(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().ep_plan_info(self.plan, C.byref(a), C.byref(b), C.byref(c)), "ep_plan_info")
        return a.value, b.value, c.value

    def close(self):
        if getattr(self, "plan", None):
            lib().ep_plan_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream(stream):
    if stream is None:
        return _torch().cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)
