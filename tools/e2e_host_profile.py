"""Host cost per call of the config-2 e2e decode step (growing cache):
ep_cache_append_generated, ep_plan_update_cache, ep_kv_append,
ep_spliced_attention (Python wrappers included), the torch copies.

    python tools/e2e_host_profile.py
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.attention import Handle
    from paper_2504_11729_b200.splice import KVPool, SpliceCache, SpliceTable, SplicedAttention
    h = Handle(0)
    B, P = bench.B, bench.P
    pool = KVPool(B * bench.PAGES_PER_REQ, bench.HKV, bench.D, P, dtype="bf16")
    table = bench.build_requests_table(SpliceTable, pool, B)
    cache = SpliceCache(1, B, P)
    for b in range(B):
        for sg in table.requests[b]:
            cache.append(b, sg.origin, sg.pos_offset, sg.length, sg.pages)
    attn = SplicedAttention.from_cache(pool, cache, bench.HQ, 1, handle=h)
    q = torch.zeros((B, 1, bench.HQ, bench.D), dtype=torch.bfloat16, device="cuda")
    o = torch.empty_like(q)
    lib = _capi.lib()
    pd = pool.desc()
    ones = np.ones(B, np.int32)
    sl = np.zeros((2, B), np.int32)
    kv = torch.zeros((2, B, bench.HKV, bench.D), dtype=torch.bfloat16, device="cuda")
    sd = torch.zeros((2, B), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    n = 60
    res = {}

    def t(name, fn):
        # host time of each call with the GPU idle (synchronised before each)
        tot = 0.0
        for i in range(n):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(i)
            tot += time.perf_counter() - t0
        res[name] = round(tot / n * 1e6, 1)
        torch.cuda.synchronize()

    def grow(i):
        if i % 60 == 59:
            for b in range(B):
                cache.truncate(b, 59)
        cache.append_generated(ones, out=(sl[0], sl[1]))

    t("append_generated", grow)
    t("update_from_cache", lambda i: attn.update_from_cache(s))
    t("kv_append", lambda i: lib.ep_kv_append(h.ptr, C.byref(pd), B, sd[0].data_ptr(), sd[1].data_ptr(),
                                               kv[0].data_ptr(), kv[1].data_ptr(), s.cuda_stream))
    t("attention_call", lambda i: attn(q, o=o, stream=s))
    qh = q.cpu().pin_memory()
    t("torch_copy_h2d", lambda i: q.copy_(qh, non_blocking=True))
    ev = torch.cuda.Event()
    t("event_record_wait", lambda i: (ev.record(s), s.wait_event(ev)))
    t("plain_ctypes_abi_version", lambda i: lib.ep_abi_version())
    t("ep_spliced_attention_direct", lambda i: lib.ep_spliced_attention(h.ptr, attn.plan, C.byref(pd), 1, q.data_ptr(), 1,
                                                                       o.data_ptr(), None, s.cuda_stream))
    print(res)
    import cProfile
    import pstats
    pr = cProfile.Profile()
    torch.cuda.synchronize()
    pr.enable()
    for i in range(n):
        attn(q, o=o, stream=s)
        attn.update_from_cache(s)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def phases():
    """Per-phase host time of the bench's e2e loop body (GPU kept busy)."""
    import torch
    import bench
    from cuda.bindings import runtime as rt
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.attention import Handle
    from paper_2504_11729_b200.splice import KVPool, SpliceCache, SpliceTable, SplicedAttention
    h = Handle(0)
    B, P = bench.B, bench.P
    pool = KVPool(B * bench.PAGES_PER_REQ, bench.HKV, bench.D, P, dtype="bf16")
    table = bench.build_requests_table(SpliceTable, pool, B)
    cache = SpliceCache(1, B, P)
    for b in range(B):
        for sg in table.requests[b]:
            cache.append(b, sg.origin, sg.pos_offset, sg.length, sg.pages)
    attn = SplicedAttention.from_cache(pool, cache, bench.HQ, 1, handle=h)
    lib = _capi.lib()
    pd = pool.desc()
    pdr = C.byref(pd)
    q = torch.zeros((B, 1, bench.HQ, bench.D), dtype=torch.bfloat16, device="cuda")
    o = torch.empty_like(q)
    lse = torch.empty((B, 1, bench.HQ), dtype=torch.float32, device="cuda")
    sl = np.zeros((2, B), np.int32)
    sd = torch.zeros((2, B), dtype=torch.int32, device="cuda")
    kv = torch.zeros((2, B, bench.HKV, bench.D), dtype=torch.bfloat16, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    ones = np.ones(B, np.int32)
    ptrs = (sd[0].data_ptr(), sd[1].data_ptr(), kv[0].data_ptr(), kv[1].data_ptr())
    acc = {k: 0.0 for k in ("grow", "update", "append", "attn")}
    n = 300
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n)]
    st = torch.cuda.current_stream()
    for i in range(n):
        evs[i][0].record(st)
        t0 = time.perf_counter()
        if i % 60 == 59:
            for b in range(B):
                cache.truncate(b, 59)
        cache.append_generated(ones, out=(sl[0], sl[1]))
        t1 = time.perf_counter()
        lib.ep_plan_update_cache(attn.plan, cache.ptr, 0, 1, sp)
        evs[i][1].record(st)
        t2 = time.perf_counter()
        lib.ep_kv_append(h.ptr, pdr, B, *ptrs, sp)
        evs[i][2].record(st)
        t3 = time.perf_counter()
        lib.ep_spliced_attention(h.ptr, attn.plan, pdr, 1, q.data_ptr(), 1, o.data_ptr(), lse.data_ptr(), sp)
        evs[i][3].record(st)
        t4 = time.perf_counter()
        for k, a, b_ in (("grow", t0, t1), ("update", t1, t2), ("append", t2, t3), ("attn", t3, t4)):
            acc[k] += (b_ - a)
    torch.cuda.synchronize()
    print("host us", {k: round(v / n * 1e6, 1) for k, v in acc.items()})
    g = {"upload": 0.0, "append": 0.0, "attn": 0.0, "gap_to_next": 0.0}
    for i in range(50, n - 1):
        g["upload"] += evs[i][0].elapsed_time(evs[i][1])
        g["append"] += evs[i][1].elapsed_time(evs[i][2])
        g["attn"] += evs[i][2].elapsed_time(evs[i][3])
        g["gap_to_next"] += evs[i][3].elapsed_time(evs[i + 1][0])
    print("gpu us", {k: round(v / (n - 51) * 1e3, 2) for k, v in g.items()})


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "phases":
    phases()
