"""Minimal driver for profiling: BASELINE config 2 spliced decode, N launches.

    python tools/decode_only.py [--steps 10] [--workload cfg2|cfg5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.attention import Handle
    from paper_2504_11729_b200.splice import KVPool, SpliceTable, SplicedAttention
    h = Handle(0)
    pool = KVPool(bench.B * bench.PAGES_PER_REQ, bench.HKV, bench.D, bench.P, dtype="bf16")
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.k.data_ptr(), pool.k.numel(), 22, -1.0, 1.0, s)
    lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.v.data_ptr(), pool.v.numel(), 23, -1.0, 1.0, s)
    q = torch.empty((bench.B, 1, bench.HQ, bench.D), dtype=torch.bfloat16, device="cuda")
    lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, q.data_ptr(), q.numel(), 21, -1.0, 1.0, s)
    table = bench.build_requests_table(SpliceTable, pool, bench.B)
    attn = SplicedAttention(pool, table, bench.HQ, 1, handle=h)
    o = torch.empty_like(q)
    for _ in range(args.steps):
        attn(q, o=o)
    torch.cuda.synchronize()
    print("ok", attn.info(), float(o.float().abs().sum()))


if __name__ == "__main__":
    main()
