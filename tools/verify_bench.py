"""BASELINE config 3: speculative verify, k = 4 and 8 draft tokens per request
against 16K spliced KV (cloud 14336 + edge 1536 + generated 512), batch 64,
7B shape (Hq 32, Hkv 8, d 128, bf16), W_score 4096 x 4096 bf16, greedy accept.

    python tools/verify_bench.py [--steps 50] [--warmup 5] [--k 4 8]

One verify step = K3 attention (tcgen05) + K4 score/argmax/accept. Reports
p50/p99 step latency (CUDA events per step), the attention-only time, HBM
GB/s of the attention (unique K/V bytes) and the tensor work rate.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

B, HQ, HKV, D, P = 64, 32, 8, 128, 64
CLOUD, EDGE, GEN = 14336, 1536, 512
S = CLOUD + EDGE + GEN
V = 4096
KV_BYTES = B * S * 2 * HKV * D * 2


def setup(k: int, h):
    import numpy as np
    import torch
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.splice import KVPool, SpliceTable, SplicedAttention
    from paper_2504_11729_b200.verify import VerifyGreedy
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    n_q = k + 1
    ppr = S // P
    pool = KVPool(B * ppr, HKV, D, P, dtype="bf16")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.k.data_ptr(), pool.k.numel(), 32,
                                    -1.0, 1.0, s))
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.v.data_ptr(), pool.v.numel(), 132,
                                    -1.0, 1.0, s))
    table = SpliceTable(B, P)
    for b in range(B):
        pages = np.arange(b * ppr, (b + 1) * ppr, dtype=np.int32)
        table.append(b, 0, 0, CLOUD, pages[:CLOUD // P])
        table.append(b, 1, CLOUD, EDGE, pages[CLOUD // P:(CLOUD + EDGE) // P])
        table.append(b, 2, CLOUD + EDGE, GEN, pages[(CLOUD + EDGE) // P:])
        table.q_pos[b] = S - n_q
    attn = SplicedAttention(pool, table, HQ, n_q, handle=h)
    q = torch.empty((B, n_q, HQ, D), dtype=torch.bfloat16, device="cuda")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, q.data_ptr(), q.numel(), 31, -1.0, 1.0, s))
    w_t = torch.empty((V, HQ * D), dtype=torch.bfloat16, device="cuda")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, w_t.data_ptr(), w_t.numel(), 33, -1.0,
                                    1.0, s))
    ver = VerifyGreedy(w_t, handle=h)
    drafts = torch.randint(0, V, (B, k), dtype=torch.int32, device="cuda")
    o = torch.empty((B, n_q, HQ, D), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, n_q, HQ), dtype=torch.float32, device="cuda")
    return dict(pool=pool, table=table, attn=attn, q=q, ver=ver, drafts=drafts, o=o, lse=lse)


def run(k: int, steps: int, warmup: int, h=None):
    import torch
    from paper_2504_11729_b200.attention import Handle
    h = h or Handle(0)
    st = setup(k, h)
    attn, q, ver, drafts, o, lse = (st[x] for x in ("attn", "q", "ver", "drafts", "o", "lse"))
    stream = torch.cuda.current_stream()

    def step():
        attn(q, o=o, lse=lse, stream=stream)
        return ver(o, drafts, stream=stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    l0 = h.launch_count()
    for e0, e1, e2 in evs:
        e0.record(stream)
        attn(q, o=o, lse=lse, stream=stream)
        e1.record(stream)
        ver(o, drafts, stream=stream)
        e2.record(stream)
    torch.cuda.synchronize()
    launches = h.launch_count() - l0
    tot = sorted(a.elapsed_time(c) for a, _, c in evs)
    att = sorted(a.elapsed_time(b) for a, b, _ in evs)
    p50, p99 = tot[len(tot) // 2], tot[min(len(tot) - 1, int(len(tot) * 0.99))]
    a50 = att[len(att) // 2]
    n_q = k + 1
    rows = 4 * n_q
    flops_attn = 4.0 * rows * S * D * B * HKV
    flops_score = 2.0 * B * n_q * HQ * D * V
    n_ctas, n_items, _ = st["attn"].info()
    return {
        "k": k, "batch": B, "keys": S, "n_q": n_q,
        "step_p50_ms": p50, "step_p99_ms": p99, "attention_p50_ms": a50,
        "score_accept_p50_ms": p50 - a50,
        "attention_hbm_gbs": KV_BYTES / (a50 / 1e3) / 1e9,
        "attention_tflops": flops_attn / (a50 / 1e3) / 1e12,
        "score_tflops_useful": flops_score / ((p50 - a50) / 1e3) / 1e12 if p50 > a50 else None,
        "query_tokens_per_s": B * n_q / (p50 / 1e3),
        "kv_bytes": KV_BYTES, "gpu_launches_per_step": launches / steps,
        "plan": {"ctas": n_ctas, "items": n_items},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--k", type=int, nargs="+", default=[4, 8])
    args = ap.parse_args()
    from paper_2504_11729_b200.attention import Handle
    h = Handle(0)
    for k in args.k:
        print(json.dumps(run(k, args.steps, args.warmup, h)), flush=True)


if __name__ == "__main__":
    main()
