"""Host mirror of the reference attention API over the B200 C-ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/core/include/edgeprompt/attention.hpp:13-52:

* ``CausalSpan(query_offset, key_offset)``                  (attention.hpp:13-16)
* ``PartialAttention(out, lse, n_keys)`` + ``identity``       (attention.hpp:24-30)
* ``full_attention(q, k, v, span)``                           (attention.hpp:35)
* ``partial_attention(q, seg_k, seg_v, span)``                (attention.hpp:39-40)
* ``fuse_partials(parts)`` / ``merge_partials(parts)``        (attention.hpp:47, :52)

Host numpy fp64 inputs go through the synchronous drop-in entry points
(``ep_*_f64``: staged to HBM, computed by the CUDA kernels, copied back), like
the reference's value-semantics functions. CUDA torch tensors (fp64/fp32) go
through the stream-ordered ``ep_*_dev`` entry points and stay on the device.
Errors raise ``InvalidArgument`` (a ``ValueError``) where the reference throws
``std::invalid_argument`` and ``DomainError`` (an ``ArithmeticError``) where it
throws ``std::domain_error``.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import DomainError, InvalidArgument, check, lib

_dp = C.POINTER(C.c_double)


class Handle:
    """Owns one ``ep_handle`` (device binding + workspace)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().ep_create(device, C.byref(h)), "ep_create")
        self._h = h
        self.device = device

    @property
    def ptr(self) -> C.c_void_p:
        return self._h

    def launch_count(self) -> int:
        return int(lib().ep_launch_count(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().ep_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_handle(device: int = 0) -> Handle:
    """Per-thread handle (an ep_handle is single-thread, ep_attn.h)."""
    hs = getattr(_tls, "handles", None)
    if hs is None:
        hs = _tls.handles = {}
    if device not in hs:
        hs[device] = Handle(device)
    return hs[device]


@dataclass(frozen=True)
class CausalSpan:
    query_offset: int = 0
    key_offset: int = 0


@dataclass
class PartialAttention:
    out: np.ndarray
    lse: np.ndarray
    n_keys: int = 0

    @staticmethod
    def identity(n_query: int, d_head: int) -> "PartialAttention":
        return PartialAttention(np.zeros((n_query, d_head)), np.full(n_query, -np.inf), 0)


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _check_shapes(q, k, v, where: str) -> None:
    # attention.cpp:14-25
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise InvalidArgument(f"{where}: expected 2-D q/k/v")
    if q.shape[1] == 0:
        raise InvalidArgument(f"{where}: zero head width")
    if k.shape[1] != q.shape[1]:
        raise InvalidArgument(f"{where}: q is {q.shape[0]}x{q.shape[1]} but k is "
                              f"{k.shape[0]}x{k.shape[1]}")
    if k.shape[0] != v.shape[0]:
        raise InvalidArgument(f"{where}: k has {k.shape[0]} rows but v has {v.shape[0]}")
    if v.shape[1] != q.shape[1]:
        raise InvalidArgument(f"{where}: v width {v.shape[1]} differs from head width "
                              f"{q.shape[1]}")


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def partial_attention(q, seg_k, seg_v, span: CausalSpan = CausalSpan(), *, handle=None,
                      stream=None):
    """attention.cpp:80-114. Fully masked rows are the identity (lse = -inf)."""
    _check_shapes(q, seg_k, seg_v, "partial_attention")
    if _is_torch_cuda(q):
        return _partial_dev(q, seg_k, seg_v, span, handle, stream)
    q, k, v = _f64(q), _f64(seg_k), _f64(seg_v)
    n_q, d = q.shape
    out = np.zeros((n_q, d))
    lse = np.zeros(n_q)
    h = handle or default_handle()
    check(lib().ep_partial_attention_f64(h.ptr, q.ctypes.data_as(_dp), n_q,
                                         k.ctypes.data_as(_dp), v.ctypes.data_as(_dp), k.shape[0],
                                         d, span.query_offset, span.key_offset,
                                         out.ctypes.data_as(_dp), lse.ctypes.data_as(_dp)),
          "partial_attention")
    return PartialAttention(out, lse, k.shape[0])


def _partial_dev(q, k, v, span, handle, stream):
    import torch
    dt = {torch.float64: _capi.EP_F64, torch.float32: _capi.EP_F32}.get(q.dtype)
    if dt is None or k.dtype != q.dtype or v.dtype != q.dtype:
        raise _capi.Unsupported("partial_attention: device path takes fp64 or fp32 q/k/v")
    for t in (q, k, v):
        if t.stride(1) != 1:
            raise InvalidArgument("partial_attention: rows must be contiguous")
    n_q, d = q.shape
    out = torch.empty((n_q, d), dtype=q.dtype, device=q.device)
    lse = torch.empty((n_q,), dtype=q.dtype, device=q.device)
    h = handle or default_handle(q.device.index or 0)
    check(lib().ep_partial_attention_dev(h.ptr, dt, q.data_ptr(), q.stride(0), n_q, k.data_ptr(),
                                         k.stride(0), v.data_ptr(), v.stride(0), k.shape[0], d,
                                         span.query_offset, span.key_offset, out.data_ptr(),
                                         d, lse.data_ptr(), _stream_ptr(stream)),
          "partial_attention")
    return PartialAttention(out, lse, k.shape[0])


def full_attention(q, k, v, span: CausalSpan = CausalSpan(), *, handle=None):
    """attention.cpp:45-78; DomainError if a row has no visible key."""
    _check_shapes(q, k, v, "full_attention")
    if _is_torch_cuda(q):
        for i in range(q.shape[0]):
            if span.query_offset + i < span.key_offset or k.shape[0] == 0:
                raise DomainError(f"full_attention: query at position {span.query_offset + i} "
                                  "has no visible key")
        return _partial_dev(q, k, v, span, handle, None).out
    q, k, v = _f64(q), _f64(k), _f64(v)
    out = np.zeros(q.shape)
    h = handle or default_handle()
    check(lib().ep_full_attention_f64(h.ptr, q.ctypes.data_as(_dp), q.shape[0],
                                      k.ctypes.data_as(_dp), v.ctypes.data_as(_dp), k.shape[0],
                                      q.shape[1], span.query_offset, span.key_offset,
                                      out.ctypes.data_as(_dp)), "full_attention")
    return out


def _host_parts(parts):
    outs = [_f64(p.out) for p in parts]
    lses = [_f64(p.lse) for p in parts]
    n_q, d = outs[0].shape
    for o, l in zip(outs, lses):
        if o.shape != (n_q, d) or l.shape != (n_q,):
            raise InvalidArgument("merge_partials: partials disagree on shape")
    po = (_dp * len(parts))(*[o.ctypes.data_as(_dp) for o in outs])
    pl = (_dp * len(parts))(*[l.ctypes.data_as(_dp) for l in lses])
    return outs, lses, po, pl, n_q, d


def merge_partials(parts, *, handle=None, stream=None) -> PartialAttention:
    """attention.cpp:116-145: fold lse in order, convex LSE-weighted sum."""
    parts = list(parts)
    if not parts:
        raise InvalidArgument("merge_partials: no partials")
    n_keys = sum(int(p.n_keys) for p in parts)
    if _is_torch_cuda(parts[0].out):
        import torch
        outs = torch.stack([p.out for p in parts]).contiguous()
        lses = torch.stack([p.lse for p in parts]).contiguous()
        P, n_q, d = outs.shape
        dt = {torch.float64: _capi.EP_F64, torch.float32: _capi.EP_F32}[outs.dtype]
        out = torch.empty((n_q, d), dtype=outs.dtype, device=outs.device)
        lse = torch.empty((n_q,), dtype=outs.dtype, device=outs.device)
        h = handle or default_handle(outs.device.index or 0)
        check(lib().ep_merge_partials_dev(h.ptr, dt, P, outs.data_ptr(), lses.data_ptr(), n_q, d,
                                          out.data_ptr(), lse.data_ptr(), _stream_ptr(stream)),
              "merge_partials")
        return PartialAttention(out, lse, n_keys)
    outs, lses, po, pl, n_q, d = _host_parts(parts)
    out = np.zeros((n_q, d))
    lse = np.zeros(n_q)
    h = handle or default_handle()
    check(lib().ep_merge_partials_f64(h.ptr, len(parts), po, pl, n_q, d,
                                      out.ctypes.data_as(_dp), lse.ctypes.data_as(_dp)),
          "merge_partials")
    return PartialAttention(out, lse, n_keys)


def fuse_partials(parts, *, handle=None):
    """attention.cpp:147-156: merged output; DomainError if a row is masked everywhere."""
    parts = list(parts)
    if not parts:
        raise InvalidArgument("fuse_partials: no partials")
    if _is_torch_cuda(parts[0].out):
        m = merge_partials(parts, handle=handle)
        import torch
        if bool(torch.isneginf(m.lse).any()):
            row = int(torch.nonzero(torch.isneginf(m.lse))[0])
            raise DomainError(f"fuse_partials: query row {row} is masked in every partial")
        return m.out
    outs, lses, po, pl, n_q, d = _host_parts(parts)
    out = np.zeros((n_q, d))
    h = handle or default_handle()
    check(lib().ep_fuse_partials_f64(h.ptr, len(parts), po, pl, n_q, d, out.ctypes.data_as(_dp)),
          "fuse_partials")
    return out
