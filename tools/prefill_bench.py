"""Prefill tiles on the tensor cores (north_star: "tcgen05
for the multi-token verify and cloud-prompt prefill tiles"), 7B shape
(Hq 32, Hkv 8, d 128, bf16):

  * cloud: a 4096-token cloud prompt per request, all 4096 tokens are queries
    (CloudServer::serve_stream -> transformer_layer, cloud.cpp:160-172);
  * edge: 512 edge tokens per request against one shared 4096-token cloud
    prompt (edge.cpp:148-164), batch 32.

    python tools/prefill_bench.py [--steps 20] [--warmup 3]

FLOPs = 4 * d * Hq per (query, visible key) pair (QK and PV, causal);
reported against the measured dense bf16 peak (MEASURED_PEAKS.json).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HQ, HKV, D, P = 32, 8, 128, 64
def _bf16_peak():
    """Dense bf16 burst TFLOP/s from the driver-written MEASURED_PEAKS.json
    (this pool's B200s); the B200_PROFILING.md fallback when absent."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured"
    except Exception:
        return 2250.0, "fallback (nominal dense bf16)"


BF16_PEAK_TFLOPS, BF16_PEAK_KIND = _bf16_peak()


def setup(kind: str, batch: int, h):
    import numpy as np
    import torch
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.splice import KVPool, SplicedPrefill, SpliceTable
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    cloud, edge = 4096, (0 if kind == "cloud" else 512)
    if kind == "cloud":
        n_pages = batch * cloud // P
    else:
        n_pages = cloud // P + batch * edge // P
    pool = KVPool(n_pages, HKV, D, P, dtype="bf16")
    for t, seed in ((pool.k, 41), (pool.v, 42)):
        _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, t.data_ptr(), t.numel(), seed, -1.0,
                                        1.0, s))
    table = SpliceTable(batch, P)
    n_new = []
    pairs = 0
    for b in range(batch):
        if kind == "cloud":
            table.append(b, 0, 0, cloud, np.arange(b * cloud // P, (b + 1) * cloud // P,
                                                   dtype=np.int32))
            n_new.append(cloud)
            pairs += cloud * (cloud + 1) // 2
        else:
            table.append(b, 0, 0, cloud, np.arange(0, cloud // P, dtype=np.int32))
            base = cloud // P + b * edge // P
            table.append(b, 1, cloud, edge, np.arange(base, base + edge // P, dtype=np.int32))
            n_new.append(edge)
            pairs += edge * cloud + edge * (edge + 1) // 2
    pre = SplicedPrefill(pool, table, HQ, n_new, handle=h)
    q = torch.empty((sum(n_new), HQ, D), dtype=torch.bfloat16, device="cuda")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, q.data_ptr(), q.numel(), 43, -1.0, 1.0, s))
    o = torch.empty_like(q)
    lse = torch.empty((sum(n_new), HQ), dtype=torch.float32, device="cuda")
    return pre, q, o, lse, pairs


def run(kind: str, batch: int, steps: int, warmup: int, h=None):
    import torch
    from paper_2504_11729_b200.attention import Handle
    h = h or Handle(0)
    pre, q, o, lse, pairs = setup(kind, batch, h)
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        pre(q, o=o, lse=lse, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        pre(q, o=o, lse=lse, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    flops = 4.0 * D * HQ * pairs
    tf = flops / (ms / 1e3) / 1e12
    return {
        "workload": (f"{kind} prefill: " + ("4096-token cloud prompt per request, all tokens queries"
                                            if kind == "cloud" else
                                            "512 edge tokens per request vs one shared 4096-token "
                                            "cloud prompt") + f", batch {batch}, Hq=32 Hkv=8 d=128 bf16"),
        "batch": batch, "query_tokens": int(q.shape[0]), "ms": ms,
        "query_tokens_per_s": q.shape[0] / (ms / 1e3),
        "causal_flops": flops, "tflops": tf, "frac_of_bf16_peak": tf / BF16_PEAK_TFLOPS,
        "bf16_peak_tflops": BF16_PEAK_TFLOPS, "bf16_peak_kind": BF16_PEAK_KIND,
        "plan": dict(zip(("ctas", "items", "pages"), pre.info())),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--kind", nargs="+", default=["cloud", "edge"])
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    for kind in args.kind:
        batch = 4 if kind == "cloud" else 32
        print(json.dumps(run(kind, batch, args.steps, args.warmup)), flush=True)


if __name__ == "__main__":
    main()
