"""Speculative draft verification: fused score + greedy accept (K4) behind the
tcgen05 verify attention (K3).

The reference has no speculative decoding; SURVEY §8a a16 constructs it from
prefill over [last, d1..dk] (model.cpp:211-236) + unembed_logits + argmax_token
(model.cpp:238-255): g_j = argmax(LN(row_j) @ W_score), accepted n = longest
prefix with d_i == g_{i-1}, emit d1..dn then g_n.
"""
from __future__ import annotations

import ctypes as C

from ._capi import InvalidArgument, check, lib
from .attention import Handle, default_handle


class VerifyGreedy:
    """Owns an ep_verifier for one W_score (device bf16, given as W^T
    [vocab][width])."""

    def __init__(self, w_score_t, handle: Handle | None = None):
        import torch
        if w_score_t.dtype != torch.bfloat16 or w_score_t.dim() != 2 or not w_score_t.is_contiguous():
            raise InvalidArgument("VerifyGreedy: w_score_t must be contiguous bf16 [vocab][width]")
        self.w = w_score_t
        self.vocab, self.width = int(w_score_t.shape[0]), int(w_score_t.shape[1])
        self.handle = handle or default_handle(w_score_t.device.index or 0)
        v = C.c_void_p()
        check(lib().ep_verifier_create(self.handle.ptr, self.width, self.vocab, w_score_t.data_ptr(),
                                       C.byref(v)), "ep_verifier_create")
        self._v = v

    def __call__(self, attn_out, drafts, logits: bool = False, stream=None):
        """attn_out: fp32 (preferred) or bf16 [B][n_q][Hq][d] (Hq*d == width);
        drafts int32 [B][n_q-1]. Returns (target_ids [B][n_q], n_accepted [B],
        logits or None)."""
        import torch
        B, n_q = int(attn_out.shape[0]), int(attn_out.shape[1])
        dt = {torch.float32: 0, torch.bfloat16: 1}.get(attn_out.dtype)
        if dt is None or not attn_out.is_contiguous() or attn_out[0, 0].numel() != self.width:
            raise InvalidArgument("VerifyGreedy: attn_out must be contiguous fp32/bf16 "
                                  "[B][n_q][width]")
        dr = drafts.to(torch.int32).contiguous()
        if tuple(dr.shape) != (B, n_q - 1):
            raise InvalidArgument("VerifyGreedy: drafts must be [B][n_q-1]")
        tgt = torch.empty((B, n_q), dtype=torch.int32, device=attn_out.device)
        nacc = torch.empty((B,), dtype=torch.int32, device=attn_out.device)
        lg = torch.empty((B * n_q, self.vocab), dtype=torch.float32,
                         device=attn_out.device) if logits else None
        s = torch.cuda.current_stream().cuda_stream if stream is None else getattr(
            stream, "cuda_stream", stream)
        check(lib().ep_verify_greedy(self.handle.ptr, self._v, B, n_q, dt, attn_out.data_ptr(),
                                     dr.data_ptr(), tgt.data_ptr(), nacc.data_ptr(),
                                     lg.data_ptr() if lg is not None else None, s),
              "ep_verify_greedy")
        return tgt, nacc, (lg.view(B, n_q, self.vocab) if lg is not None else None)

    def close(self):
        if getattr(self, "_v", None):
            lib().ep_verifier_destroy(self._v)
            self._v = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
