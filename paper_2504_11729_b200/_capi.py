"""ctypes binding of include/ep/ep_attn.h (libep_b200.so).

Loading fails loudly when the library is missing — there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
# EP_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("EP_LIB") or os.path.join(PKG, "_lib", "libep_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "ep", "ep_attn.h")
HEADERS = [HEADER, os.path.join(os.path.dirname(PKG), "include", "ep", "ep_model.h")]

EP_OK, EP_EINVAL, EP_EMASKED, EP_ECUDA, EP_ENCCL, EP_ENOMEM, EP_EUNSUPPORTED, EP_EWIRE = range(8)
EP_F32, EP_BF16, EP_F64 = 0, 1, 2


class EPError(RuntimeError):
    status = -1


class InvalidArgument(EPError, ValueError):
    """std::invalid_argument in the reference (attention.cpp:14-25, :117)."""
    status = EP_EINVAL


class DomainError(EPError, ArithmeticError):
    """std::domain_error in the reference (attention.cpp:52-56, :150-153)."""
    status = EP_EMASKED


class CudaError(EPError):
    status = EP_ECUDA


class NcclError(EPError):
    status = EP_ENCCL


class OutOfMemory(EPError, MemoryError):
    status = EP_ENOMEM


class Unsupported(EPError, NotImplementedError):
    status = EP_EUNSUPPORTED


class WireError(EPError, ValueError):
    """edgeprompt::wire::WireError (wire.hpp:94-104): a malformed EPKV frame;
    ``kind`` = WireError::Kind + 1 (see KV_FRAME_KINDS), 6 = not a kv frame."""
    status = EP_EWIRE
    kind = 0


KV_FRAME_KINDS = ("ok", "bad_magic", "bad_version", "truncated", "length_overflow", "malformed",
                  "not_kv_frame")

_ERRORS = {cls.status: cls for cls in (InvalidArgument, DomainError, CudaError, NcclError,
                                       OutOfMemory, Unsupported, WireError)}


class Segment(C.Structure):
    """ep_segment (KVSegment, cache.hpp:18-28)."""
    _fields_ = [("origin", C.c_int32), ("len", C.c_int32), ("pos_offset", C.c_int64),
                ("page_off", C.c_int64)]


class KVFrameInfo(C.Structure):
    """ep_kv_frame_info."""
    _fields_ = [("session_id", C.c_uint32), ("seq_len", C.c_uint32), ("layer", C.c_uint16),
                ("n_heads", C.c_uint16), ("d_head", C.c_uint16), ("pad", C.c_uint16),
                ("wire_error", C.c_int32)]


class KVPoolDesc(C.Structure):
    """ep_kv_pool."""
    _fields_ = [("dtype", C.c_int32), ("n_kv_heads", C.c_int32), ("d_head", C.c_int32),
                ("page_tokens", C.c_int32), ("num_pages", C.c_int64), ("k_pages", C.c_void_p),
                ("v_pages", C.c_void_p)]


class ModelConfigDesc(C.Structure):
    """ep_model_config (ModelConfig, model.hpp:15-25, + storage dtype)."""
    _fields_ = [("n_layers", C.c_int32), ("n_heads", C.c_int32), ("d_model", C.c_int32),
                ("vocab_size", C.c_int32), ("max_positions", C.c_int32), ("dtype", C.c_int32),
                ("init_seed", C.c_uint64)]


_lib: C.CDLL | None = None

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_sz = C.c_size_t

_SIGS = {
    "ep_abi_version": (C.c_int, []),
    "ep_last_error": (C.c_char_p, []),
    "ep_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "ep_destroy": (C.c_int, [_vp]),
    "ep_partial_attention_f64": (C.c_int, [_vp, _dp, _sz, _dp, _dp, _sz, _sz, _sz, _sz, _dp, _dp]),
    "ep_full_attention_f64": (C.c_int, [_vp, _dp, _sz, _dp, _dp, _sz, _sz, _sz, _sz, _dp]),
    "ep_merge_partials_f64": (C.c_int, [_vp, _sz, C.POINTER(_dp), C.POINTER(_dp), _sz, _sz, _dp,
                                        _dp]),
    "ep_fuse_partials_f64": (C.c_int, [_vp, _sz, C.POINTER(_dp), C.POINTER(_dp), _sz, _sz, _dp]),
    "ep_partial_attention_dev": (C.c_int, [_vp, C.c_int, _vp, _sz, _sz, _vp, _sz, _vp, _sz, _sz,
                                           _sz, _sz, _sz, _vp, _sz, _vp, _vp]),
    "ep_merge_partials_dev": (C.c_int, [_vp, C.c_int, _sz, _vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "ep_merge_partials_packed_dev": (C.c_int, [_vp, C.c_int32, _vp, C.c_int32, C.c_int32,
                                               C.c_int32, _vp, _vp, _vp]),
    "ep_peer_group_create": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(_vp)]),
    "ep_peer_group_export": (C.c_int, [_vp, _vp]),
    "ep_peer_group_base": (C.c_int, [_vp, C.POINTER(_vp)]),
    "ep_peer_group_connect_ipc": (C.c_int, [_vp, _vp]),
    "ep_peer_group_connect_ptrs": (C.c_int, [_vp, C.POINTER(_vp)]),
    "ep_splitkv_combine_dev": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp, C.c_int32, _vp, _vp, _vp]),
    "ep_peer_group_destroy": (C.c_int, [_vp]),
    "ep_spliced_attention_splitkv": (C.c_int, [_vp, _vp, C.POINTER(KVPoolDesc), C.c_int32, _vp, _vp,
                                               C.c_int32, _vp, _vp, _vp]),
    "ep_plan_create_prefill": (C.c_int, [_vp, C.POINTER(KVPoolDesc), C.c_int32, C.c_int32, _vp,
                                         _vp, _vp, _vp, C.POINTER(_vp)]),
    "ep_plan_create": (C.c_int, [_vp, C.POINTER(KVPoolDesc), C.c_int32, C.c_int32, C.c_int32, _vp,
                                 _vp, _vp, _vp, C.c_int32, C.POINTER(_vp)]),
    "ep_plan_update": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "ep_plan_destroy": (C.c_int, [_vp]),
    "ep_plan_info": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64)]),
    "ep_spliced_attention": (C.c_int, [_vp, _vp, C.POINTER(KVPoolDesc), C.c_int32, _vp, C.c_int32,
                                       _vp, _vp, _vp]),
    "ep_fill_uniform": (C.c_int, [_vp, C.c_int, _vp, _sz, C.c_uint64, C.c_double, C.c_double,
                                  _vp]),
    "ep_launch_count": (C.c_int64, [_vp]),
    "ep_kv_append": (C.c_int, [_vp, C.POINTER(KVPoolDesc), C.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "ep_kv_ingest_frame": (C.c_int, [_vp, C.POINTER(KVPoolDesc), _vp, _sz, _vp, C.c_int32,
                                     C.POINTER(KVFrameInfo), _vp]),
    "ep_cache_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "ep_cache_destroy": (C.c_int, [_vp]),
    "ep_cache_end_position": (C.c_int64, [_vp, C.c_int32]),
    "ep_cache_append": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, _vp, C.c_int32]),
    "ep_cache_append_generated": (C.c_int, [_vp, _vp, _vp, C.c_int32, _vp, _vp, _vp]),
    "ep_cache_truncate": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.POINTER(C.c_int32)]),
    "ep_cache_check_consistent": (C.c_int, [_vp]),
    "ep_cache_layer_arrays": (C.c_int, [_vp, C.c_int32, _vp, _vp, C.c_int64, _vp, C.c_int64,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ep_plan_create_cache": (C.c_int, [_vp, C.POINTER(KVPoolDesc), _vp, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(_vp)]),
    "ep_plan_update_cache": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, _vp]),
    "ep_kv_ingest_frame_async": (C.c_int, [_vp, C.POINTER(KVPoolDesc), _vp, _sz, _vp, C.c_int32,
                                           _vp]),
    "ep_kv_ingest_poll": (C.c_int, [_vp, _vp, C.POINTER(KVFrameInfo)]),
}

_SIGS.update({
    "ep_verifier_create": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.POINTER(_vp)]),
    "ep_verifier_destroy": (C.c_int, [_vp]),
    "ep_verify_greedy": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp, _vp,
                                   _vp, _vp, _vp]),
})

_SIGS.update({
    "ep_model_create": (C.c_int, [_vp, C.POINTER(ModelConfigDesc), C.c_int32, C.c_int32,
                                  C.c_int64, C.POINTER(_vp)]),
    "ep_model_destroy": (C.c_int, [_vp]),
    "ep_model_weight_sum": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "ep_model_kv_pool": (C.c_int, [_vp, C.c_int32, C.POINTER(KVPoolDesc)]),
    "ep_model_weight": (C.c_int, [_vp, C.c_char_p, C.c_int32, C.POINTER(_vp),
                                  C.POINTER(C.c_size_t)]),
    "ep_model_forward": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                   _vp]),
    "ep_model_generate": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp, C.c_int32, _vp, _vp, _vp]),
    "ep_model_verify": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ep_model_last_attention_path": (C.c_int, [_vp]),
})

# Optional entry points (present when the corresponding kernels are built).
_OPTIONAL_SIGS: dict = {}


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2504_11729_b200.build` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        for name, (res, args) in _OPTIONAL_SIGS.items():
            if hasattr(L, name):
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
        _lib = L
    return _lib


def check(rc: int, where: str = "") -> None:
    if rc == EP_OK:
        return
    msg = lib().ep_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, EPError)(f"{where}: {msg}" if where else msg)


def header_symbols() -> list[str]:
    """Function names declared in include/ep/*.h."""
    text = "\n".join(open(h).read() for h in HEADERS)
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ep_[a-z0-9_]+)\s*\(", text)))
