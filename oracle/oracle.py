"""ctypes front-end for the CHECKERS — test infrastructure, never the product.

Two implementations sit behind the same Python functions:

* ``impl="port"`` — ``oracle/_build/libep_oracle.so``, the plain-C restatement
  (``ep_oracle.c``) of the reference path;
* ``impl="ref"``  — ``oracle/_ref/libep_ref.so``, the unmodified reference
  sources (``/root/reference/proj/core/src/{matrix,attention,cache,model}.cpp``)
  behind ``ref_capi.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libep_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libep_ref.so")
DROPIN_SO = os.path.join(HERE, "_ref", "libep_ref_dropin.so")
REF_SRC = "/root/reference/proj/core"

DT_F32, DT_BF16, DT_F64 = 0, 1, 2
EPO_OK, EPO_EINVAL, EPO_EMASKED = 0, 1, 2

_dp = C.POINTER(C.c_double)


def build(with_ref: bool | None = None) -> None:
    """Compile the C port, and the reference wrapper when the reference tree is here."""
    targets = ["port"]
    if with_ref is None:
        with_ref = os.path.isdir(REF_SRC)
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError):
    """std::invalid_argument in the reference."""


class DomainError(OracleError):
    """std::domain_error in the reference."""


_EXC = {1: InvalidArgument, 2: DomainError, 3: IndexError, 4: OracleError}


def _raise(rc: int, where: str, lib=None) -> None:
    if rc == 0:
        return
    msg = where
    if lib is not None and hasattr(lib, "epref_last_error"):
        msg += ": " + lib.epref_last_error().decode()
    raise _EXC.get(rc, OracleError)(msg)


_libs: dict[str, C.CDLL] = {}


def _load(impl: str) -> C.CDLL:
    if impl in _libs:
        return _libs[impl]
    path = {"port": PORT_SO, "ref": REF_SO, "dropin": DROPIN_SO}[impl]
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (make -C oracle {impl})")
    lib = C.CDLL(path)
    if impl == "port":
        lib.epo_log_add_exp.restype = C.c_double
        lib.epo_log_add_exp.argtypes = [C.c_double, C.c_double]
        lib.epo_argmax.restype = C.c_uint32
        lib.epo_argmax.argtypes = [_dp, C.c_size_t]
        lib.epo_partial_attention.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp,
                                              C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                              C.c_size_t, _dp, _dp]
        lib.epo_full_attention.argtypes = [_dp, C.c_size_t, _dp, _dp, C.c_size_t, C.c_size_t,
                                           C.c_size_t, C.c_size_t, _dp]
        lib.epo_merge_partials.argtypes = [C.c_size_t, C.POINTER(_dp), C.POINTER(_dp),
                                           C.c_size_t, C.c_size_t, _dp, _dp]
        lib.epo_fuse_partials.argtypes = [C.c_size_t, C.POINTER(_dp), C.POINTER(_dp),
                                          C.c_size_t, C.c_size_t, _dp]
        lib.epo_spliced_attention.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                              _dp, _dp]
        lib.epo_verify_greedy.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_void_p, _dp]
        lib.epo_fill_uniform.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_uint64,
                                         C.c_double, C.c_double]
        lib.epo_kv_frame_decode.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                            C.c_void_p]
        lib.epo_f64_to_bf16.restype = C.c_uint16
        lib.epo_f64_to_bf16.argtypes = [C.c_double]
        lib.epo_kv_ingest.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]
    else:
        lib.epref_last_error.restype = C.c_char_p
        lib.epref_log_add_exp.restype = C.c_double
        lib.epref_log_add_exp.argtypes = [C.c_double, C.c_double]
        lib.epref_argmax.restype = C.c_uint32
        lib.epref_argmax.argtypes = [_dp, C.c_size_t]
        lib.epref_partial_attention.argtypes = [_dp, C.c_size_t, _dp, _dp, C.c_size_t,
                                                C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp]
        lib.epref_full_attention.argtypes = [_dp, C.c_size_t, _dp, _dp, C.c_size_t, C.c_size_t,
                                             C.c_size_t, C.c_size_t, _dp]
        lib.epref_merge_partials.argtypes = [C.c_size_t, C.POINTER(_dp), C.POINTER(_dp),
                                             C.c_size_t, C.c_size_t, _dp, _dp]
        lib.epref_fuse_partials.argtypes = [C.c_size_t, C.POINTER(_dp), C.POINTER(_dp),
                                            C.c_size_t, C.c_size_t, _dp]
        lib.epref_spliced_attention.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                                _dp, _dp]
        lib.epref_cache_create.restype = C.c_void_p
        lib.epref_cache_create.argtypes = [C.c_void_p]
        lib.epref_cache_destroy.argtypes = [C.c_void_p]
        lib.epref_cache_attention.argtypes = [C.c_void_p, _dp, C.c_int, C.c_void_p, C.c_int64,
                                              _dp, _dp]
        lib.epref_model_create.restype = C.c_void_p
        lib.epref_model_create.argtypes = [C.c_size_t] * 5 + [C.c_uint64]
        lib.epref_model_destroy.argtypes = [C.c_void_p]
        lib.epref_model_weight_sum.restype = C.c_double
        lib.epref_model_weight_sum.argtypes = [C.c_void_p]
        lib.epref_generate_split.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                             C.c_size_t, C.c_size_t, C.c_void_p]
        lib.epref_generate_monolithic.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t,
                                                  C.c_size_t, C.c_void_p]
        lib.epref_session_create.restype = C.c_void_p
        lib.epref_session_create.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                             C.c_size_t]
        lib.epref_session_destroy.argtypes = [C.c_void_p]
        lib.epref_session_n_segments.restype = C.c_size_t
        lib.epref_session_n_segments.argtypes = [C.c_void_p]
        lib.epref_session_end_position.restype = C.c_size_t
        lib.epref_session_end_position.argtypes = [C.c_void_p]
        lib.epref_session_segment.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p,
                                              C.c_void_p, C.POINTER(C.c_size_t),
                                              C.POINTER(C.c_size_t), C.POINTER(C.c_int)]
        lib.epref_session_first_token.argtypes = [C.c_void_p, C.POINTER(C.c_uint32)]
        lib.epref_session_decode_step.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p,
                                                  C.POINTER(C.c_uint32)]
        lib.epref_session_verify.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                             C.c_void_p]
        if hasattr(lib, "epref_kv_frame_encode"):
            lib.epref_kv_frame_encode.restype = C.c_size_t
            lib.epref_kv_frame_encode.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_size_t]
            lib.epref_end_of_prefill_frame.restype = C.c_size_t
            lib.epref_end_of_prefill_frame.argtypes = [C.c_void_p, C.c_size_t]
            lib.epref_kv_frame_decode.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                                  C.c_void_p]
    _libs[impl] = lib
    return lib


def available(impl: str) -> bool:
    return os.path.exists({"port": PORT_SO, "ref": REF_SO, "dropin": DROPIN_SO}[impl])


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# --------------------------------------------------------------- SplitMix64 --

class SplitMix64:
    """rng.hpp:10-29, bit-exact (Python ints masked to 64 bits)."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.state = seed & self.M

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & self.M
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()

    def matrix(self, rows: int, cols: int, lo: float, hi: float) -> np.ndarray:
        return np.array([[self.uniform(lo, hi) for _ in range(cols)] for _ in range(rows)],
                        dtype=np.float64).reshape(rows, cols)


def fill_uniform(dtype: int, n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Draws 0..n-1 of SplitMix64(seed) as uniform(lo, hi), rounded to dtype
    (bf16 returned as raw uint16)."""
    np_dt = {DT_F32: np.float32, DT_BF16: np.uint16, DT_F64: np.float64}[dtype]
    out = np.empty(n, dtype=np_dt)
    _load("port").epo_fill_uniform(dtype, out.ctypes.data, n, seed & SplitMix64.M, lo, hi)
    return out


def bf16_to_f64(raw: np.ndarray) -> np.ndarray:
    return (raw.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


# ----------------------------------------------------------------- kernels --

def log_add_exp(a: float, b: float, impl: str = "port") -> float:
    lib = _load(impl)
    return (lib.epo_log_add_exp if impl == "port" else lib.epref_log_add_exp)(a, b)


def argmax(logits, impl: str = "port") -> int:
    lg = _f64(logits)
    lib = _load(impl)
    f = lib.epo_argmax if impl == "port" else lib.epref_argmax
    return int(f(_p(lg), lg.size))


def partial_attention(q, k, v, q_off: int, k_off: int, impl: str = "port"):
    """(out [n_q x d], lse [n_q]) — attention.cpp:80-114."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    n_q, d = q.shape
    n_keys = k.shape[0]
    out = np.zeros((n_q, d))
    lse = np.zeros(n_q)
    lib = _load(impl)
    if impl == "port":
        if k.shape[1] != d or v.shape != k.shape:
            raise InvalidArgument("partial_attention: shape mismatch")
        rc = lib.epo_partial_attention(_p(q), d, n_q, _p(k), d, _p(v), d, n_keys, d, q_off,
                                       k_off, _p(out), _p(lse))
        _raise(rc, "partial_attention")
    else:
        if k.shape[1] != d or v.shape[0] != n_keys or v.shape[1] != d:
            # the wrapper passes one d for q/k/v; reproduce the reference's check
            raise InvalidArgument("partial_attention: shape mismatch")
        rc = lib.epref_partial_attention(_p(q), n_q, _p(k), _p(v), n_keys, d, q_off, k_off,
                                         _p(out), _p(lse))
        _raise(rc, "partial_attention", lib)
    return out, lse


def full_attention(q, k, v, q_off: int, k_off: int, impl: str = "port"):
    q, k, v = _f64(q), _f64(k), _f64(v)
    n_q, d = q.shape
    out = np.zeros((n_q, d))
    lib = _load(impl)
    f = lib.epo_full_attention if impl == "port" else lib.epref_full_attention
    rc = f(_p(q), n_q, _p(k), _p(v), k.shape[0], d, q_off, k_off, _p(out))
    _raise(rc, "full_attention", lib if impl != "port" else None)
    return out


def _parts_arrays(parts):
    outs = [_f64(o) for o, _ in parts]
    lses = [_f64(l) for _, l in parts]
    po = (_dp * len(parts))(*[_p(o) for o in outs])
    pl = (_dp * len(parts))(*[_p(l) for l in lses])
    return outs, lses, po, pl


def merge_partials(parts, impl: str = "port"):
    """parts: list of (out [n_q x d], lse [n_q]) — attention.cpp:116-145."""
    if not parts:
        raise InvalidArgument("merge_partials: no partials")
    outs, lses, po, pl = _parts_arrays(parts)
    n_q, d = outs[0].shape
    out = np.zeros((n_q, d))
    lse = np.zeros(n_q)
    lib = _load(impl)
    f = lib.epo_merge_partials if impl == "port" else lib.epref_merge_partials
    rc = f(len(parts), po, pl, n_q, d, _p(out), _p(lse))
    _raise(rc, "merge_partials", lib if impl != "port" else None)
    return out, lse


def fuse_partials(parts, impl: str = "port"):
    if not parts:
        raise InvalidArgument("fuse_partials: no partials")
    outs, lses, po, pl = _parts_arrays(parts)
    n_q, d = outs[0].shape
    out = np.zeros((n_q, d))
    lib = _load(impl)
    f = lib.epo_fuse_partials if impl == "port" else lib.epref_fuse_partials
    rc = f(len(parts), po, pl, n_q, d, _p(out))
    _raise(rc, "fuse_partials", lib if impl != "port" else None)
    return out


# ------------------------------------------------------- batched splice ----

class _Segment(C.Structure):
    _fields_ = [("origin", C.c_int32), ("len", C.c_int32), ("pos_offset", C.c_int64),
                ("page_off", C.c_int64)]


class _SpliceBatch(C.Structure):
    _fields_ = [("kv_dtype", C.c_int), ("n_kv_heads", C.c_int), ("n_q_heads", C.c_int),
                ("d_head", C.c_int), ("page_tokens", C.c_int), ("k_pages", C.c_void_p),
                ("v_pages", C.c_void_p), ("batch", C.c_int), ("n_q", C.c_int),
                ("seg_indptr", C.c_void_p), ("segs", C.c_void_p), ("page_table", C.c_void_p),
                ("q_pos", C.c_void_p), ("q_dtype", C.c_int), ("q", C.c_void_p)]


SEGMENT_DTYPE = np.dtype([("origin", "<i4"), ("len", "<i4"), ("pos_offset", "<i8"),
                          ("page_off", "<i8")])


@dataclass
class HostSpliceBatch:
    """Host (numpy) view of a paged splice batch, in the CUDA path's layout.

    k_pages / v_pages: [num_pages][Hkv][page_tokens][d] float32 or raw-bf16 uint16.
    segs: SEGMENT_DTYPE records, seg_indptr [B+1], page_table int32,
    q_pos int64 [B], q [B][n_q][Hq][d] float32 or raw-bf16 uint16.
    """
    kv_dtype: int
    n_kv_heads: int
    n_q_heads: int
    d_head: int
    page_tokens: int
    k_pages: np.ndarray
    v_pages: np.ndarray
    seg_indptr: np.ndarray
    segs: np.ndarray
    page_table: np.ndarray
    q_pos: np.ndarray
    q_dtype: int
    q: np.ndarray
    n_q: int

    @property
    def batch(self) -> int:
        return len(self.seg_indptr) - 1

    def _struct(self) -> _SpliceBatch:
        return _SpliceBatch(self.kv_dtype, self.n_kv_heads, self.n_q_heads, self.d_head,
                            self.page_tokens, self.k_pages.ctypes.data, self.v_pages.ctypes.data,
                            self.batch, self.n_q, self.seg_indptr.ctypes.data,
                            self.segs.ctypes.data, self.page_table.ctypes.data,
                            self.q_pos.ctypes.data, self.q_dtype, self.q.ctypes.data)


def spliced_attention(sb: HostSpliceBatch, n_threads: int = 1, units=None,
                      impl: str = "port"):
    """Returns (out [B][n_q][Hq][d], lse [B][n_q][Hq]) in fp64. Rows of units
    not in ``units`` are left NaN."""
    for name in ("k_pages", "v_pages", "seg_indptr", "segs", "page_table", "q_pos", "q"):
        assert getattr(sb, name).flags.c_contiguous, name
    assert sb.seg_indptr.dtype == np.int64 and sb.page_table.dtype == np.int32
    assert sb.q_pos.dtype == np.int64 and sb.segs.dtype == SEGMENT_DTYPE
    out = np.full((sb.batch, sb.n_q, sb.n_q_heads, sb.d_head), np.nan)
    lse = np.full((sb.batch, sb.n_q, sb.n_q_heads), np.nan)
    st = sb._struct()
    ul = None
    n_units = 0
    if units is not None:
        ul = np.ascontiguousarray(units, dtype=np.int64)
        n_units = ul.size
    lib = _load(impl)
    f = lib.epo_spliced_attention if impl == "port" else lib.epref_spliced_attention
    rc = f(C.addressof(st), n_threads, ul.ctypes.data if ul is not None else None, n_units,
           _p(out), _p(lse))
    _raise(rc, "spliced_attention", lib if impl != "port" else None)
    return out, lse


class RefBatchCache:
    """The reference's own layout for a batch (fp64 KVSegments, heads
    concatenated), built once outside any timed region; ``attention`` then runs
    transformer_layer's attention block (model.cpp:167-181) per (request,
    q-head) unit on n_threads host threads."""

    def __init__(self, sb: HostSpliceBatch):
        self.lib = _load("ref")
        self.sb = sb
        self._st = sb._struct()
        self.h = self.lib.epref_cache_create(C.addressof(self._st))
        if not self.h:
            raise OracleError(self.lib.epref_last_error().decode())
        q = sb.q
        self.q = bf16_to_f64(q) if sb.q_dtype == DT_BF16 else _f64(q)
        self.q = np.ascontiguousarray(self.q)

    def attention(self, n_threads: int = 1, units=None, out=None, lse=None):
        sb = self.sb
        if out is None:
            out = np.full((sb.batch, sb.n_q, sb.n_q_heads, sb.d_head), np.nan)
        if lse is None:
            lse = np.full((sb.batch, sb.n_q, sb.n_q_heads), np.nan)
        ul = None if units is None else np.ascontiguousarray(units, dtype=np.int64)
        rc = self.lib.epref_cache_attention(self.h, _p(self.q), n_threads,
                                            None if ul is None else ul.ctypes.data,
                                            0 if ul is None else ul.size, _p(out), _p(lse))
        _raise(rc, "cache_attention", self.lib)
        return out, lse

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.epref_cache_destroy(self.h)
            self.h = None


def verify_greedy(attn_out, w_score, drafts):
    """attn_out [B][n_q][W] fp64, w_score [W][V], drafts [B][k] ->
    (target_ids [B][n_q], n_accepted [B], top2_gap [B][n_q])."""
    a = _f64(attn_out)
    w = _f64(w_score)
    dr = np.ascontiguousarray(drafts, dtype=np.int32)
    B, n_q, W = a.shape
    V = w.shape[1]
    tgt = np.zeros((B, n_q), dtype=np.int32)
    nacc = np.zeros(B, dtype=np.int32)
    gap = np.zeros((B, n_q))
    rc = _load("port").epo_verify_greedy(_p(a), B, n_q, W, _p(w), V, dr.ctypes.data,
                                         tgt.ctypes.data, nacc.ctypes.data, _p(gap))
    _raise(rc, "verify_greedy")
    return tgt, nacc, gap


# -------------------------------------------------- reference model (ref) --

class RefModel:
    """init_model / generate_* / decode_step of the reference (model.cpp)."""

    def __init__(self, n_layers, n_heads, d_model, vocab, max_positions=512, seed=1,
                 impl: str = "ref"):
        self.lib = _load(impl)
        self.cfg = dict(n_layers=n_layers, n_heads=n_heads, d_model=d_model, vocab=vocab,
                        max_positions=max_positions, seed=seed)
        self.h = self.lib.epref_model_create(n_layers, n_heads, d_model, vocab, max_positions,
                                             seed & SplitMix64.M)
        if not self.h:
            raise InvalidArgument(self.lib.epref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.epref_model_destroy(self.h)
            self.h = None

    def weight_sum(self) -> float:
        return self.lib.epref_model_weight_sum(self.h)

    def generate_split(self, cloud, edge, n_steps):
        c = np.ascontiguousarray(cloud, dtype=np.uint32)
        e = np.ascontiguousarray(edge, dtype=np.uint32)
        out = np.zeros(n_steps, dtype=np.uint32)
        rc = self.lib.epref_generate_split(self.h, c.ctypes.data, c.size, e.ctypes.data, e.size,
                                           n_steps, out.ctypes.data)
        _raise(rc, "generate_split", self.lib)
        return out.tolist()

    def generate_monolithic(self, prompt, n_steps):
        p = np.ascontiguousarray(prompt, dtype=np.uint32)
        out = np.zeros(n_steps, dtype=np.uint32)
        rc = self.lib.epref_generate_monolithic(self.h, p.ctypes.data, p.size, n_steps,
                                                out.ctypes.data)
        _raise(rc, "generate_monolithic", self.lib)
        return out.tolist()

    def session(self, cloud, edge) -> "RefSession":
        return RefSession(self, cloud, edge)


class RefSession:
    def __init__(self, model: RefModel, cloud, edge):
        self.m = model
        self.lib = model.lib
        c = np.ascontiguousarray(cloud, dtype=np.uint32)
        e = np.ascontiguousarray(edge, dtype=np.uint32)
        self.h = self.lib.epref_session_create(model.h, c.ctypes.data, c.size, e.ctypes.data,
                                               e.size)
        if not self.h:
            raise InvalidArgument(self.lib.epref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.epref_session_destroy(self.h)
            self.h = None

    @property
    def n_segments(self) -> int:
        return self.lib.epref_session_n_segments(self.h)

    @property
    def end_position(self) -> int:
        return self.lib.epref_session_end_position(self.h)

    def segment(self, layer: int, seg: int):
        """(k [len x D], v [len x D], pos_offset, origin) of one cached segment."""
        n = C.c_size_t()
        pos = C.c_size_t()
        org = C.c_int()
        rc = self.lib.epref_session_segment(self.h, layer, seg, None, None, C.byref(n),
                                            C.byref(pos), C.byref(org))
        _raise(rc, "segment", self.lib)
        D = self.m.cfg["d_model"]
        k = np.zeros((n.value, D))
        v = np.zeros((n.value, D))
        rc = self.lib.epref_session_segment(self.h, layer, seg, k.ctypes.data, v.ctypes.data,
                                            C.byref(n), C.byref(pos), C.byref(org))
        _raise(rc, "segment", self.lib)
        return k, v, pos.value, org.value

    def first_token(self) -> int:
        t = C.c_uint32()
        _raise(self.lib.epref_session_first_token(self.h, C.byref(t)), "first_token", self.lib)
        return t.value

    def verify(self, tokens):
        """(targets [n], logits [n][V]): the reference's prefill of ``tokens``
        ([last, d1..dk]) as a generated segment at the cache end, then
        unembed_logits + argmax_token per row. The session's
        cache is unchanged."""
        t = np.ascontiguousarray(tokens, dtype=np.uint32)
        V = self.m.cfg["vocab"]
        logits = np.zeros((t.size, V))
        tg = np.zeros(t.size, dtype=np.uint32)
        rc = self.lib.epref_session_verify(self.h, t.ctypes.data, t.size, logits.ctypes.data,
                                           tg.ctypes.data)
        _raise(rc, "verify", self.lib)
        return tg.astype(np.int64), logits

    def decode_step(self, last: int):
        logits = np.zeros(self.m.cfg["vocab"])
        nxt = C.c_uint32()
        rc = self.lib.epref_session_decode_step(self.h, last, logits.ctypes.data, C.byref(nxt))
        _raise(rc, "decode_step", self.lib)
        return nxt.value, logits


# -------------------------------------------------------------- KV ingest --
# EPKV kv frames (wire.hpp:59-75; wire.cpp:70-221) and their decode into
# device-layout pages.

WIRE_OK, WIRE_BAD_MAGIC, WIRE_BAD_VERSION, WIRE_TRUNCATED, WIRE_LENGTH_OVERFLOW, \
    WIRE_MALFORMED, WIRE_NOT_KV = range(7)


class KVFrameInfo(C.Structure):
    """epo_kv_frame_info."""
    _fields_ = [("session_id", C.c_uint32), ("seq_len", C.c_uint32), ("layer", C.c_uint16),
                ("n_heads", C.c_uint16), ("d_head", C.c_uint16), ("pad", C.c_uint16)]


def kv_frame_encode(session_id, layer, k, v):
    """The reference's own encode_frame of a KVFrame (oracle/_ref). k, v:
    [seq_len][n_heads][d_head] float64 -> frame bytes."""
    k = _f64(k)
    v = _f64(v)
    seq, H, d = k.shape
    info = KVFrameInfo(session_id, seq, layer, H, d, 0)
    lib = _load("ref")
    n = lib.epref_kv_frame_encode(C.byref(info), k.ctypes.data, v.ctypes.data, None, 0)
    out = np.empty(n, dtype=np.uint8)
    lib.epref_kv_frame_encode(C.byref(info), k.ctypes.data, v.ctypes.data, out.ctypes.data, n)
    return out


def end_of_prefill_frame():
    lib = _load("ref")
    out = np.empty(16, dtype=np.uint8)
    n = lib.epref_end_of_prefill_frame(out.ctypes.data, 16)
    return out[:n].copy()


def kv_frame_decode(frame, impl: str = "port"):
    """(code, info, k, v): code is WIRE_*; k, v [seq][H][d] float64 when OK."""
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    lib = _load(impl)
    f = lib.epo_kv_frame_decode if impl == "port" else lib.epref_kv_frame_decode
    info = KVFrameInfo()
    rc = f(frame.ctypes.data, frame.size, C.byref(info), None, None)
    if rc != WIRE_OK:
        return rc, None, None, None
    n = info.seq_len * info.n_heads * info.d_head
    k = np.empty(n)
    v = np.empty(n)
    rc = f(frame.ctypes.data, frame.size, C.byref(info), k.ctypes.data, v.ctypes.data)
    shape = (info.seq_len, info.n_heads, info.d_head)
    return rc, info, k.reshape(shape), v.reshape(shape)


def f64_to_bf16(x) -> np.ndarray:
    lib = _load("port")
    x = _f64(x)
    return np.array([lib.epo_f64_to_bf16(float(a)) for a in x.reshape(-1)], dtype=np.uint16)


def kv_ingest(frame, kv_dtype: int, page_tokens: int, page_table, num_pages: int):
    """Port of the device ingest: (code, info, k_pages, v_pages) with pages
    [num_pages][n_heads][page_tokens][d] (bf16 raw uint16 or float32)."""
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    code, info, _, _ = kv_frame_decode(frame)
    if code != WIRE_OK:
        return code, None, None, None
    dt = np.uint16 if kv_dtype == DT_BF16 else np.float32
    shape = (num_pages, info.n_heads, page_tokens, info.d_head)
    kp = np.zeros(shape, dtype=dt)
    vp = np.zeros(shape, dtype=dt)
    pt = np.ascontiguousarray(page_table, dtype=np.int32)
    lib = _load("port")
    rc = lib.epo_kv_ingest(frame.ctypes.data, frame.size, kv_dtype, page_tokens, pt.ctypes.data,
                           kp.ctypes.data, vp.ctypes.data, C.byref(info))
    return rc, info, kp, vp
