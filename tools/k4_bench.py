"""K4 alone (score GEMM + refine + accept), repeated back to back on the same
config-3 rows (W_score stays L2-resident between calls) vs interleaved with
the attention (the verify step), to separate DRAM first-touch from the
mainloop's own limits.

    python tools/k4_bench.py [--k 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    import torch
    import verify_bench as VB
    from paper_2504_11729_b200.attention import Handle
    h = Handle(0)
    st = VB.setup(args.k, h)
    attn, q, ver, drafts, o, lse = (st[x] for x in ("attn", "q", "ver", "drafts", "o", "lse"))
    s = torch.cuda.current_stream()
    attn(q, o=o, lse=lse, stream=s)
    for _ in range(5):
        ver(o, drafts, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.steps):
        ver(o, drafts, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    hot = e0.elapsed_time(e1) / args.steps
    print(json.dumps({"k": args.k, "score_accept_back_to_back_ms": hot}))


if __name__ == "__main__":
    main()
