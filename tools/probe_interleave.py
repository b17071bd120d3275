"""Probe: does the spliced-decode kernel run slower when another kernel sits
between consecutive launches? (config-4 shard shape, 1 GPU)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch
import splitkv_bench as SB
from paper_2504_11729_b200.attention import Handle

def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    h = Handle(0)
    pool, table, attn, q, n_loc = SB.build_local(batch, 2, 0, h)
    rows = batch * SB.HQ
    o = torch.empty((batch, 1, SB.HQ, SB.D), dtype=torch.float32, device="cuda")
    l = torch.empty((batch, 1, SB.HQ), dtype=torch.float32, device="cuda")
    small = torch.empty(1024, device="cuda")
    st = torch.cuda.current_stream()
    def a(): attn(q, o=o, lse=l, stream=st)
    def b(): a(); small.add_(1.0)
    def c(): a(); torch.cuda._sleep(20000)
    res = {}
    for name, f in (("attn", a), ("attn+tiny", b), ("attn+sleep", c), ("attn2", a)):
        for _ in range(5): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(30): f()
        e1.record(st); torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 30
    # per-launch events
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(61)]
    ev[0].record(st)
    for i in range(30):
        a(); ev[2*i+1].record(st); small.add_(1.0); ev[2*i+2].record(st)
    torch.cuda.synchronize()
    res["attn_in_loop"] = sum(ev[2*i].elapsed_time(ev[2*i+1]) for i in range(30)) / 30
    res["tiny_in_loop"] = sum(ev[2*i+1].elapsed_time(ev[2*i+2]) for i in range(30)) / 30
    print(json.dumps(res))

main()
