"""BASELINE config 5: 256 requests share ONE 8192-token cloud-prompt segment
(the same pages in every request's splice table) plus a private ragged edge
segment of U{32..2048} tokens drawn from SplitMix64(5); decode, n_q = 1,
7B shape (Hq 32, Hkv 8, d 128, bf16), page size 64.

    python tools/multitenant_bench.py [--steps 50]

Reports tokens/s, the unique-byte rate (each shared byte counted once, SURVEY
§8d) and the L2-fed request-byte rate (every request's view counted).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

B, HQ, HKV, D, P = 256, 32, 8, 128, 64
CLOUD = 8192


def edge_lengths():
    from oracle.oracle import SplitMix64
    r = SplitMix64(5)
    return [32 + r.next_u64() % 2017 for _ in range(B)]


def setup(h):
    import numpy as np
    import torch
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.splice import KVPool, SpliceTable, SplicedAttention
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    edges = edge_lengths()
    cloud_pages = CLOUD // P
    edge_pages = [-(-e // P) for e in edges]
    n_pages = cloud_pages + sum(edge_pages) + B  # + one generated page per request
    pool = KVPool(n_pages, HKV, D, P, dtype="bf16")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.k.data_ptr(), pool.k.numel(), 52,
                                    -1.0, 1.0, s))
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.v.data_ptr(), pool.v.numel(), 53,
                                    -1.0, 1.0, s))
    table = SpliceTable(B, P)
    shared = np.arange(cloud_pages, dtype=np.int32)
    nxt = cloud_pages
    for b, e in enumerate(edges):
        table.append(b, 0, 0, CLOUD, shared)
        table.append(b, 1, CLOUD, e, np.arange(nxt, nxt + edge_pages[b], dtype=np.int32))
        nxt += edge_pages[b]
        table.append(b, 2, CLOUD + e, 1, np.array([nxt], dtype=np.int32))
        nxt += 1
        table.q_pos[b] = CLOUD + e
    attn = SplicedAttention(pool, table, HQ, 1, handle=h)
    q = torch.empty((B, 1, HQ, D), dtype=torch.bfloat16, device="cuda")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, q.data_ptr(), q.numel(), 51, -1.0, 1.0, s))
    unique = (CLOUD + sum(edges) + B) * 2 * HKV * D * 2
    viewed = sum(CLOUD + e + 1 for e in edges) * 2 * HKV * D * 2
    return pool, table, attn, q, unique, viewed, edges


def run(steps=50, warmup=5, h=None):
    import torch
    from paper_2504_11729_b200.attention import Handle
    h = h or Handle(torch.cuda.current_device())
    pool, table, attn, q, unique, viewed, edges = setup(h)
    o = torch.empty_like(q)
    lse = torch.empty((B, 1, HQ), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        attn(q, o=o, lse=lse, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        attn(q, o=o, lse=lse, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {
        "workload": "cfg5 multi-tenant: 256 requests share one 8192-token cloud segment + "
                    "ragged U{32..2048} edge (SplitMix64(5)), Hq=32 Hkv=8 d=128 bf16, decode",
        "ms_per_step": ms, "tokens_per_s": B / (ms / 1e3),
        "unique_bytes": unique, "unique_gbs": unique / (ms / 1e3) / 1e9,
        "viewed_bytes": viewed, "viewed_gbs": viewed / (ms / 1e3) / 1e9,
        "mean_edge": sum(edges) / len(edges),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    print(json.dumps(run(args.steps, args.warmup)))


if __name__ == "__main__":
    main()
