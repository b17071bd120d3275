"""Host mirror of the reference decoder API over ``ep_model`` (include/ep/ep_model.h).

Same names and argument meaning as
/root/reference/proj/core/include/edgeprompt/model.hpp:

* ``ModelConfig``                                     (model.hpp:15-25)
* ``init_model(config)`` -> ``Model`` (+ ``weight_sum``) (model.hpp:41-64)
* ``SegmentedCache`` (per-session splice table)        (cache.hpp:30-61)
* ``prefill(model, tokens, origin, pos_offset, cache)`` -> ``PrefillResult``
* ``decode_step(model, cache, last_token)`` -> ``DecodeResult``
* ``decode_greedy`` / ``generate_monolithic`` / ``generate_split``
* ``decode_batch`` — one decode step for many sessions in one forward pass.

The weights, the per-layer KV page pools and every activation stay in HBM;
a decode step moves one token id in and one token id (+ logits on request)
out. ``PrefillResult`` returns the new segment WITHOUT appending it, like the
reference (the caller does ``cache.append(res.segments)``). Errors:
``InvalidArgument`` where the reference throws ``std::invalid_argument`` or
``std::out_of_range`` (unknown token ids, positions past max_positions).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import InvalidArgument, KVPoolDesc, ModelConfigDesc, check, lib
from .attention import Handle, default_handle
from .splice import (ORIGIN_CLOUD, ORIGIN_EDGE, ORIGIN_GENERATED, SEGMENT_DTYPE, PageAllocator,
                     SegmentRef)

__all__ = ["ModelConfig", "Model", "init_model", "SegmentedCache", "PrefillResult",
           "DecodeResult", "prefill", "decode_step", "decode_batch", "decode_greedy", "generate_batch",
           "generate_monolithic", "generate_split", "ORIGIN_CLOUD", "ORIGIN_EDGE",
           "ORIGIN_GENERATED"]


def _torch():
    import torch
    return torch


@dataclass
class ModelConfig:
    """ModelConfig (model.hpp:15-25)."""
    n_layers: int = 2
    n_heads: int = 2
    d_model: int = 8
    vocab_size: int = 32
    max_positions: int = 512
    init_seed: int = 1

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads

    def validate(self) -> None:
        """model.cpp:42-50."""
        if min(self.n_layers, self.n_heads, self.d_model, self.vocab_size,
               self.max_positions) <= 0:
            raise InvalidArgument("ModelConfig: all dimensions must be positive")
        if self.d_model % self.n_heads:
            raise InvalidArgument(f"ModelConfig: d_model {self.d_model} not divisible by "
                                  f"n_heads {self.n_heads}")


_DT = {"f64": _capi.EP_F64, "f32": _capi.EP_F32, "bf16": _capi.EP_BF16}


class Model:
    """init_model (model.cpp:82-102) on the device: weights + one KV page pool
    per layer (all layers share the page numbering, so one splice table per
    session addresses every layer).

    dtype "f64" keeps the reference's precision; "f32" is the serving
    precision of BASELINE config 1 (kv_dtype "f32" or "bf16")."""

    def __init__(self, config: ModelConfig, *, dtype: str = "f64", kv_dtype: str | None = None,
                 num_pages: int | None = None, page_tokens: int = 64,
                 handle: Handle | None = None, device: int = 0):
        config.validate()
        self.config = config
        self.dtype = dtype
        self.kv_dtype = kv_dtype or dtype
        self.page_tokens = page_tokens
        if num_pages is None:
            num_pages = 4 * (-(-config.max_positions // page_tokens)) + 8
        self.num_pages = num_pages
        self.handle = handle or default_handle(device)
        self.device = self.handle.device
        desc = ModelConfigDesc(config.n_layers, config.n_heads, config.d_model,
                               config.vocab_size, config.max_positions, _DT[dtype],
                               config.init_seed & ((1 << 64) - 1))
        m = C.c_void_p()
        check(lib().ep_model_create(self.handle.ptr, C.byref(desc), _DT[self.kv_dtype],
                                    page_tokens, num_pages, C.byref(m)), "init_model")
        self._m = m
        self.pages = PageAllocator(num_pages)
        torch = _torch()
        self.tdtype = torch.float64 if dtype == "f64" else torch.float32

    @property
    def ptr(self) -> C.c_void_p:
        return self._m

    def weight_sum(self) -> float:
        """Model::weight_sum (model.cpp:52-67)."""
        out = C.c_double()
        check(lib().ep_model_weight_sum(self._m, C.byref(out)), "weight_sum")
        return out.value

    def kv_pool(self, layer: int) -> KVPoolDesc:
        d = KVPoolDesc()
        check(lib().ep_model_kv_pool(self._m, layer, C.byref(d)), "kv_pool")
        return d

    def weight_ptr(self, name: str, layer: int = 0):
        p, n = C.c_void_p(), C.c_size_t()
        check(lib().ep_model_weight(self._m, name.encode(), layer, C.byref(p), C.byref(n)),
              "weight")
        return p.value, n.value

    def last_attention_path(self) -> str:
        return {1: "spliced", 2: "generic", 3: "persistent"}.get(
            lib().ep_model_last_attention_path(self._m), "none")

    def forward(self, tables, n_new, tokens, *, want_logits=True, want_hidden=False,
                stream=None, out=None):
        """ep_model_forward over a batch of splice tables (one per request):
        the last n_new[b] tokens of request b are new. Returns (next token ids
        [B] int32 cuda tensor, logits [B][V] or None, hidden or None).
        out: optional (next, logits) device tensors to write into."""
        torch = _torch()
        B = len(tables)
        indptr, segs, pt = _batch_arrays(tables)
        nn = np.ascontiguousarray(n_new, dtype=np.int32)
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        if tok.size != int(nn.sum()):
            raise InvalidArgument("forward: len(tokens) != sum(n_new)")
        dev = f"cuda:{self.device}"
        if out is not None:
            nxt, logits = out
        else:
            nxt = torch.empty(B, dtype=torch.int32, device=dev)
            logits = (torch.empty((B, self.config.vocab_size), dtype=self.tdtype, device=dev)
                      if want_logits else None)
        hidden = (torch.empty((int(nn.sum()), self.config.d_model), dtype=self.tdtype,
                              device=dev) if want_hidden else None)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().ep_model_forward(self._m, B, indptr.ctypes.data, segs.ctypes.data,
                                     pt.ctypes.data, nn.ctypes.data, tok.ctypes.data,
                                     hidden.data_ptr() if hidden is not None else None,
                                     logits.data_ptr() if logits is not None else None,
                                     nxt.data_ptr(), s.cuda_stream), "forward")
        return nxt, logits, hidden

    def verify(self, tables, n_new, tokens, *, want_logits=False, stream=None):
        """ep_model_verify: per request the last n_new[b] positions hold
        [last, d1..dk] (tokens, request-major). Returns (targets [sum n_new]
        int32, n_accepted [B] int32, logits [sum n_new][V] or None) as cuda
        tensors."""
        torch = _torch()
        B = len(tables)
        indptr, segs, pt = _batch_arrays(tables)
        nn = np.ascontiguousarray(n_new, dtype=np.int32)
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        if tok.size != int(nn.sum()):
            raise InvalidArgument("verify: len(tokens) != sum(n_new)")
        dev = f"cuda:{self.device}"
        tgt = torch.empty(int(nn.sum()), dtype=torch.int32, device=dev)
        nacc = torch.empty(B, dtype=torch.int32, device=dev)
        logits = (torch.empty((int(nn.sum()), self.config.vocab_size), dtype=self.tdtype, device=dev)
                  if want_logits else None)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().ep_model_verify(self._m, B, indptr.ctypes.data, segs.ctypes.data, pt.ctypes.data,
                                    nn.ctypes.data, tok.ctypes.data,
                                    logits.data_ptr() if logits is not None else None,
                                    tgt.data_ptr(), nacc.data_ptr(), s.cuda_stream), "verify")
        return tgt, nacc, logits

    def generate(self, tables, n_steps: int, first_tokens, *, stream=None):
        """ep_model_generate: the last n_steps positions of every table are
        decoded on the device (one CUDA graph per step, replayed). Returns
        [B][n_steps] greedy tokens."""
        torch = _torch()
        B = len(tables)
        indptr, segs, pt = _batch_arrays(tables)
        first = np.ascontiguousarray(first_tokens, dtype=np.int32)
        out = np.zeros((B, n_steps), dtype=np.int32)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().ep_model_generate(self._m, B, indptr.ctypes.data, segs.ctypes.data,
                                      pt.ctypes.data, n_steps, first.ctypes.data, out.ctypes.data,
                                      s.cuda_stream), "generate")
        return out.tolist()

    def close(self) -> None:
        if getattr(self, "_m", None):
            lib().ep_model_destroy(self._m)
            self._m = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_model(config: ModelConfig, **kw) -> Model:
    return Model(config, **kw)


class SegmentedCache:
    """One session's splice table (SegmentedCache, cache.hpp:30-61): ordered
    segments cloud -> edge -> generated with gapless positions, over pages of
    the model's pools (the same page ids in every layer)."""

    def __init__(self, model: Model):
        self.model = model
        self.segments: list[SegmentRef] = []

    @property
    def n_layers(self) -> int:
        return self.model.config.n_layers

    def empty(self) -> bool:
        return not self.segments

    def end_position(self) -> int:
        return self.segments[-1].end_position if self.segments else 0

    def append(self, segments) -> None:
        """SegmentedCache::append (cache.cpp:25-53): validated first, atomic."""
        if isinstance(segments, SegmentRef):
            segments = [segments]
        pos, last = self.end_position(), (self.segments[-1].origin if self.segments else -1)
        for s in segments:
            if s.pos_offset != pos:
                raise InvalidArgument(f"SegmentedCache::append: segment starts at "
                                      f"{s.pos_offset}, cache ends at {pos}")
            if s.length <= 0:
                raise InvalidArgument("SegmentedCache::append: empty segment")
            if s.origin < last:
                raise InvalidArgument("SegmentedCache::append: origin order must be "
                                      "(cloud, edge, generated)")
            pos, last = s.pos_offset + s.length, s.origin
        self.segments.extend(segments)

    def check_consistent(self) -> str:
        pos, last = None, -1
        for s in self.segments:
            if pos is not None and s.pos_offset != pos:
                return "gap in position coverage"
            if s.origin < last:
                return "origin order violated"
            pos, last = s.end_position, s.origin
        return ""

    def _grow_generated(self, n: int) -> None:
        """append_generated_token (cache.cpp:55-80) without the copy: the new
        rows take the last page's free slots or fresh pages."""
        P = self.model.page_tokens
        segs = self.segments
        pos = self.end_position()
        if not segs or segs[-1].origin != ORIGIN_GENERATED:
            segs.append(SegmentRef(ORIGIN_GENERATED, pos, n, self.model.pages.alloc(-(-n // P))))
            return
        g = segs[-1]
        free = g.pages.size * P - g.length
        if n > free:
            g.pages = np.concatenate([g.pages, self.model.pages.alloc(-(-(n - free) // P))])
        g.length += n

    def _shrink_generated(self, n: int) -> None:
        g = self.segments[-1]
        P = self.model.page_tokens
        g.length -= n
        keep = -(-g.length // P)
        if keep < g.pages.size:
            self.model.pages.release(g.pages[keep:])
            g.pages = g.pages[:keep]
        if g.length == 0:
            self.segments.pop()

    def release(self) -> None:
        for s in self.segments:
            self.model.pages.release(s.pages)
        self.segments = []


def _batch_arrays(tables):
    """(seg_indptr, segs, page_table) of several segment lists (one per request)."""
    indptr = np.zeros(len(tables) + 1, dtype=np.int64)
    recs, pages, off = [], [], 0
    for b, segs in enumerate(tables):
        for s in segs:
            recs.append((s.origin, s.length, s.pos_offset, off))
            pages.append(np.asarray(s.pages, dtype=np.int32))
            off += s.pages.size
        indptr[b + 1] = len(recs)
    segs_arr = np.array(recs, dtype=SEGMENT_DTYPE) if recs else np.zeros(0, SEGMENT_DTYPE)
    pt = np.concatenate(pages).astype(np.int32) if pages else np.zeros(1, np.int32)
    return indptr, segs_arr, np.ascontiguousarray(pt)


@dataclass
class PrefillResult:
    """prefill's result (model.hpp:87-90): the new segment (one page list for
    all layers, NOT yet appended), the final hidden rows, and the greedy
    token / logits of the last row (what decode_greedy reads from
    prefill_hidden)."""
    segment: SegmentRef
    hidden: object
    logits: object
    next_token: int
    model: Model = field(repr=False, default=None)

    @property
    def segments(self):
        return [self.segment]

    def release(self) -> None:
        """Frees the segment's pages when it is never appended."""
        self.model.pages.release(self.segment.pages)


@dataclass
class DecodeResult:
    next_token: int
    logits: np.ndarray


def _check_tokens(model: Model, tokens) -> None:
    V = model.config.vocab_size
    for t in tokens:
        if not 0 <= int(t) < V:
            raise InvalidArgument(f"embed: unknown token id {int(t)}")


def prefill(model: Model, tokens, origin: int, pos_offset: int, cache: SegmentedCache,
            *, want_hidden: bool = True) -> PrefillResult:
    """prefill (model.cpp:211-236): the new tokens attend to the cache's
    segments and causally to each other; their K/V go to fresh pages."""
    tokens = [int(t) for t in tokens]
    if not tokens:
        raise InvalidArgument("prefill: empty token list")
    if cache.end_position() != pos_offset:
        raise InvalidArgument(f"prefill: pos_offset {pos_offset} does not match cache end "
                              f"{cache.end_position()}")
    if pos_offset + len(tokens) > model.config.max_positions:
        raise InvalidArgument("embed: positions overflow max_positions")
    _check_tokens(model, tokens)
    P = model.page_tokens
    seg = SegmentRef(origin, pos_offset, len(tokens), model.pages.alloc(-(-len(tokens) // P)))
    try:
        nxt, logits, hidden = model.forward([cache.segments + [seg]], [len(tokens)], tokens,
                                            want_hidden=want_hidden)
    except Exception:
        model.pages.release(seg.pages)
        raise
    return PrefillResult(seg, hidden, logits[0], int(nxt[0].item()), model)


def decode_step(model: Model, cache: SegmentedCache, last_token: int) -> DecodeResult:
    """decode_step (model.cpp:257-283): embeds last_token at the cache end,
    runs all layers, appends its K/V to the generated segment, returns the
    greedy next token and its logits."""
    nxt, logits = decode_batch(model, [cache], [last_token], want_logits=True)
    return DecodeResult(int(nxt[0]), logits[0])


def decode_batch(model: Model, caches, last_tokens, *, want_logits: bool = False):
    """One decode step for B sessions in ONE forward pass (batched serving of
    decode_step). Returns (next ids numpy [B], logits numpy [B][V] or None)."""
    for c in caches:
        if c.empty():
            raise InvalidArgument("decode_step: empty cache")
        issue = c.check_consistent()
        if issue:
            raise InvalidArgument(f"decode_step: inconsistent cache: {issue}")
        if c.end_position() + 1 > model.config.max_positions:
            raise InvalidArgument("embed: positions overflow max_positions")
    _check_tokens(model, last_tokens)
    for c in caches:
        c._grow_generated(1)
    out, buf = None, None
    if want_logits and model.tdtype == _torch().float32:
        # logits and next ids in one device buffer: one device->host copy
        torch = _torch()
        B, V = len(caches), model.config.vocab_size
        buf = torch.empty(B * V + B, dtype=torch.float32, device=f"cuda:{model.device}")
        out = (buf[B * V:].view(torch.int32), buf[:B * V].view(B, V))
    try:
        nxt, logits, _ = model.forward([c.segments for c in caches], [1] * len(caches),
                                       list(last_tokens), want_logits=want_logits, out=out)
    except Exception:
        for c in caches:
            c._shrink_generated(1)
        raise
    if buf is not None:
        host = _to_host(model, buf)
        return host[B * V:].view(np.int32).copy(), host[:B * V].reshape(B, V).copy()
    if logits is None:
        return _to_host(model, nxt).copy(), None
    return nxt.cpu().numpy(), logits.cpu().numpy()


@dataclass
class VerifyResult:
    """Greedy speculative verify of one session: the accepted drafts
    d1..dn, the bonus token g_n (the next ``last`` token), every row's target
    g_0..g_k and, if asked, the rows' logits."""
    accepted: list
    next_token: int
    targets: np.ndarray
    logits: object = None


def verify_greedy(model: Model, cache: SegmentedCache, last_token: int, drafts, *,
                  want_logits: bool = False) -> VerifyResult:
    """Speculative verify as SURVEY §8a a16 builds it from the reference:
    prefill(model, [last, d1..dk], generated, end_position, cache)
    (model.cpp:211-236), then unembed_logits + argmax_token per row
    (model.cpp:238-255); n = the longest draft prefix the targets reproduce.
    The cache keeps the K/V of last, d1..dn — as n + 1 decode_step calls
    would — and the bonus token g_n is returned as the next token."""
    drafts = [int(d) for d in drafts]
    toks = [int(last_token)] + drafts
    if cache.empty():
        raise InvalidArgument("verify: empty cache")
    issue = cache.check_consistent()
    if issue:
        raise InvalidArgument(f"verify: inconsistent cache: {issue}")
    if cache.end_position() + len(toks) > model.config.max_positions:
        raise InvalidArgument("embed: positions overflow max_positions")
    _check_tokens(model, toks)
    cache._grow_generated(len(toks))
    try:
        tgt, nacc, logits = model.verify([cache.segments], [len(toks)], toks, want_logits=want_logits)
        tgt = tgt.cpu().numpy()
        n = int(nacc.cpu().numpy()[0])
    except Exception:
        cache._shrink_generated(len(toks))
        raise
    cache._shrink_generated(len(drafts) - n)   # keep last, d1..dn
    return VerifyResult(drafts[:n], int(tgt[n]), tgt,
                        logits.cpu().numpy() if logits is not None else None)


def _to_host(model: Model, t):
    """Device tensor -> numpy view of a per-model pinned landing buffer that
    is reused across steps (a direct DMA instead of a staged pageable copy);
    callers copy out what they keep."""
    torch = _torch()
    nbytes = t.numel() * t.element_size()
    pin = getattr(model, "_pinned_out", None)
    if pin is None or pin.numel() < nbytes:
        pin = torch.empty(max(nbytes, 4096), dtype=torch.uint8, pin_memory=True)
        model._pinned_out = pin
    dst = pin[:nbytes].view(t.dtype)
    dst.copy_(t.reshape(-1), non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return dst.numpy()


def generate_batch(model: Model, caches, first_tokens, n_steps: int):
    """n_steps greedy decode steps for every session, resident on the device
    (ep_model_generate): the generated segments grow by n_steps and the
    tokens come back once at the end. Returns [B][n_steps]."""
    if n_steps <= 0:
        return [[] for _ in caches]
    for c in caches:
        if c.empty():
            raise InvalidArgument("decode_step: empty cache")
        if c.end_position() + n_steps > model.config.max_positions:
            raise InvalidArgument("embed: positions overflow max_positions")
    _check_tokens(model, first_tokens)
    for c in caches:
        c._grow_generated(n_steps)
    try:
        return model.generate([c.segments for c in caches], n_steps, list(first_tokens))
    except Exception:
        for c in caches:
            c._shrink_generated(n_steps)
        raise


def decode_greedy(model: Model, cache: SegmentedCache, prefill_result: PrefillResult,
                  n_steps: int, *, device_loop: bool = True):
    """decode_greedy (model.cpp:285-297), starting from the greedy token of
    the last prefilled row. device_loop: the n_steps - 1 decode steps run as
    one device-resident rollout (generate_batch); otherwise one decode_step
    (host round trip) per token."""
    out = []
    if n_steps == 0:
        return out
    out.append(prefill_result.next_token)
    if device_loop:
        return out + generate_batch(model, [cache], [out[0]], n_steps - 1)[0]
    while len(out) < n_steps:
        nxt, _ = decode_batch(model, [cache], [out[-1]])
        out.append(int(nxt[0]))
    return out


def generate_monolithic(model: Model, prompt, n_steps: int, *, device_loop: bool = True):
    """model.cpp:299-305."""
    cache = SegmentedCache(model)
    try:
        pf = prefill(model, prompt, ORIGIN_EDGE, 0, cache, want_hidden=False)
        cache.append(pf.segments)
        return decode_greedy(model, cache, pf, n_steps, device_loop=device_loop)
    finally:
        cache.release()


def generate_split(model: Model, cloud_prompt, edge_prompt, n_steps: int, *,
                   device_loop: bool = True):
    """model.cpp:307-316: cloud prefill, edge prefill against the cloud KV,
    decode on the edge-side cache."""
    cache = SegmentedCache(model)
    try:
        cloud = prefill(model, cloud_prompt, ORIGIN_CLOUD, 0, cache, want_hidden=False)
        cache.append(cloud.segments)
        edge = prefill(model, edge_prompt, ORIGIN_EDGE, len(cloud_prompt), cache,
                       want_hidden=False)
        cache.append(edge.segments)
        return decode_greedy(model, cache, edge, n_steps, device_loop=device_loop)
    finally:
        cache.release()
