"""Paged splice-table cases shared by the golden generator, the CPU oracle
tests and the GPU parity tests. Pool contents and queries are SplitMix64
U(-1, 1) draws rounded to the kernel dtype (SURVEY §8d "Inputs"), so the
device and the oracle see identical values."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def make_case(kv_dtype: int, n_q_heads: int, n_kv_heads: int, d: int, requests, n_q: int = 1,
              page_tokens: int = 64, seed: int = 1, spare_pages: int = 1) -> O.HostSpliceBatch:
    """requests: list of per-request segment lists [(origin, length, share_key)].
    Segments with the same non-None share_key reuse the same pages (a cloud
    prompt referenced by several requests). Query rows sit at the end of each
    request's cache: q_pos = end - n_q (decode: the self token is the last key;
    verify: the last n_q keys are the accepted token + drafts, causal)."""
    P = page_tokens
    shared: dict = {}
    next_page = 0
    seg_recs, page_table, indptr, q_pos = [], [], [0], []
    for segs in requests:
        pos = 0
        for origin, length, key in segs:
            npg = -(-length // P)
            if key is not None and key in shared:
                pages, slen = shared[key]
                assert slen == length
            else:
                pages = list(range(next_page, next_page + npg))
                next_page += npg
                if key is not None:
                    shared[key] = (pages, length)
            seg_recs.append((origin, length, pos, len(page_table)))
            page_table.extend(pages)
            pos += length
        indptr.append(len(seg_recs))
        q_pos.append(pos - n_q)
    num_pages = next_page + spare_pages
    per_pool = num_pages * n_kv_heads * P * d
    k = O.fill_uniform(kv_dtype, per_pool, seed * 1000 + 1).reshape(num_pages, n_kv_heads, P, d)
    v = O.fill_uniform(kv_dtype, per_pool, seed * 1000 + 2).reshape(num_pages, n_kv_heads, P, d)
    B = len(requests)
    q = O.fill_uniform(kv_dtype, B * n_q * n_q_heads * d, seed * 1000 + 3).reshape(
        B, n_q, n_q_heads, d)
    return O.HostSpliceBatch(
        kv_dtype=kv_dtype, n_kv_heads=n_kv_heads, n_q_heads=n_q_heads, d_head=d,
        page_tokens=P, k_pages=np.ascontiguousarray(k), v_pages=np.ascontiguousarray(v),
        seg_indptr=np.array(indptr, dtype=np.int64),
        segs=np.array(seg_recs, dtype=O.SEGMENT_DTYPE),
        page_table=np.array(page_table if page_table else [0], dtype=np.int32),
        q_pos=np.array(q_pos, dtype=np.int64), q_dtype=kv_dtype, q=np.ascontiguousarray(q),
        n_q=n_q)


CLOUD, EDGE, GEN = 0, 1, 2

# Small cases with every structural feature: ragged page tails, shared cloud
# pages, GQA, MHA, multi-row causal queries, a single-page request.
SMALL_CASES = {
    "gqa4_bf16_decode": dict(kv_dtype=O.DT_BF16, n_q_heads=8, n_kv_heads=2, d=128, n_q=1,
                             requests=[[(CLOUD, 300, "c"), (EDGE, 37, None), (GEN, 5, None)],
                                       [(CLOUD, 300, "c"), (EDGE, 130, None), (GEN, 1, None)],
                                       [(EDGE, 64, None)],
                                       [(CLOUD, 300, "c"), (EDGE, 1, None), (GEN, 64, None)]]),
    "mha_f32_d64_decode": dict(kv_dtype=O.DT_F32, n_q_heads=4, n_kv_heads=4, d=64, n_q=1,
                               requests=[[(CLOUD, 512, None), (EDGE, 64, None), (GEN, 3, None)]]),
    "gqa2_f32_d128_nq2": dict(kv_dtype=O.DT_F32, n_q_heads=4, n_kv_heads=2, d=128, n_q=2,
                              requests=[[(CLOUD, 200, None), (EDGE, 70, None), (GEN, 2, None)],
                                        [(EDGE, 3, None)]]),
    # speculative verify (n_q = k+1 causal rows over the last n_q keys):
    # the tcgen05 path (rows = 4*5 = 20 and 4*9 = 36)
    "gqa4_bf16_verify_k4": dict(kv_dtype=O.DT_BF16, n_q_heads=8, n_kv_heads=2, d=128, n_q=5,
                                requests=[[(CLOUD, 300, "c"), (EDGE, 37, None), (GEN, 12, None)],
                                          [(CLOUD, 300, "c"), (EDGE, 130, None), (GEN, 5, None)],
                                          [(EDGE, 5, None)],
                                          [(CLOUD, 64, None), (EDGE, 64, None), (GEN, 64, None)]]),
    "gqa4_bf16_verify_k8": dict(kv_dtype=O.DT_BF16, n_q_heads=8, n_kv_heads=2, d=128, n_q=9,
                                requests=[[(CLOUD, 700, None), (EDGE, 90, None), (GEN, 20, None)],
                                          [(EDGE, 9, None)]]),
    "gqa4_bf16_d64_nq2": dict(kv_dtype=O.DT_BF16, n_q_heads=8, n_kv_heads=2, d=64, n_q=2,
                              requests=[[(CLOUD, 129, "c"), (EDGE, 65, None), (GEN, 9, None)],
                                        [(CLOUD, 129, "c"), (EDGE, 2, None)]]),
}


def small_case(name: str, seed: int = 7) -> O.HostSpliceBatch:
    return make_case(seed=seed, **SMALL_CASES[name])
