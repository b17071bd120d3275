"""Helpers for the GPU parity tests: move an oracle HostSpliceBatch onto the
device through the product's own KVPool / SpliceTable / SplicedAttention."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def torch_from_raw(arr: np.ndarray, kv_dtype: int, device="cuda"):
    import torch
    if kv_dtype == O.DT_BF16:
        return torch.from_numpy(arr.view(np.int16)).to(device).view(torch.bfloat16)
    return torch.from_numpy(arr).to(device)


def to_device(sb: O.HostSpliceBatch, handle=None):
    """Returns (pool, table, attn, q) for the product path."""
    from paper_2504_11729_b200.splice import KVPool, SpliceTable, SplicedAttention
    k = torch_from_raw(sb.k_pages, sb.kv_dtype)
    v = torch_from_raw(sb.v_pages, sb.kv_dtype)
    pool = KVPool(sb.k_pages.shape[0], sb.n_kv_heads, sb.d_head, sb.page_tokens,
                  dtype="bf16" if sb.kv_dtype == O.DT_BF16 else "f32", k=k, v=v)
    table = SpliceTable(sb.batch, sb.page_tokens)
    for b in range(sb.batch):
        for s in sb.segs[sb.seg_indptr[b]:sb.seg_indptr[b + 1]]:
            npg = -(-int(s["len"]) // sb.page_tokens)
            pages = sb.page_table[int(s["page_off"]):int(s["page_off"]) + npg]
            table.append(b, int(s["origin"]), int(s["pos_offset"]), int(s["len"]), pages)
    table.q_pos[:] = sb.q_pos
    attn = SplicedAttention(pool, table, sb.n_q_heads, sb.n_q, handle=handle)
    q = torch_from_raw(sb.q, sb.q_dtype)
    return pool, table, attn, q


def tol_for(kv_dtype: int) -> float:
    """north_star: 1e-3 relative for fp32, 2e-2 for bf16 (|got-want|/max(1,|want|))."""
    return 2e-2 if kv_dtype == O.DT_BF16 else 1e-3
