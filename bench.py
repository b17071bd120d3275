#!/usr/bin/env python
"""Benchmark of the spliced-KV attention hot path (BASELINE.json).

Default workload = BASELINE config 2 (configs[1]): 7B-shaped attention —
32 q-heads, 8 kv-heads (GQA), d_head 128, bf16 KV — over a spliced cache of
4096 cloud-prompt + 512 edge-private + 1 generated (self) token per request,
private pages per request, batch 32, one decode query row per request.
A "step" = one spliced-attention pass of the whole batch through one layer
(all heads) = 32 tokens. Synthetic SplitMix64 U(-1,1) inputs (seeds q 21,
K 22, V 23), no checkpoint.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun and measures the path that shards: BASELINE
config 4 (long-context split-KV) — 32 requests of 131072 cloud + 512 edge
keys, the cloud KV cut into N contiguous shards (one per GPU), every rank
running K1 over its shard and the peer-memory (o, lse) combine over NVLink;
`value` = tokens/s of the whole job (strong scaling: the total work is
fixed), with the same workload unsharded on one GPU measured in the same run
(`value_1gpu`). Config 2 does not shard (independent requests); its
N-replica throughput is reported beside it. Prints one JSON line on rank 0.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference sources) of the same workload on the
host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spliced-KV attention tokens/s & HBM GB/s vs roofline; verify-step p50 latency"

# Config 2 shape.
B, HQ, HKV, D, P = 32, 32, 8, 128, 64
CLOUD, EDGE, SELF = 4096, 512, 1
SEQ = CLOUD + EDGE + SELF
PAGES_PER_REQ = CLOUD // P + EDGE // P + 1
ALG_BYTES = B * SEQ * 2 * HKV * D * 2  # every unique K/V byte once = 603,979,776
SEED_Q, SEED_K, SEED_V = 21, 22, 23

WORKLOAD = ("cfg2: 7B-shaped spliced decode, Hq=32 Hkv=8 d=128 bf16, 4096 cloud + 512 edge "
            "+ 1 self KV per request (private pages), batch 32, n_q=1")
# Config 4 (the sharded path, N > 1)
SKV_B, SKV_CLOUD, SKV_EDGE = 32, 131072, 512



def cpu_model():
    """Host CPU model name (the CPU baseline names its cores)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"

def skv_workload(world):
    return (f"cfg4: long-context split-KV, Hq=32 Hkv=8 d=128 bf16, {SKV_CLOUD} cloud + {SKV_EDGE} "
            f"edge KV per request (private pages), batch {SKV_B}, n_q=1, cloud KV in {world} "
            "contiguous shards (one per GPU), edge on the last rank")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _poll(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def build_requests_table(SpliceTable, pool, batch):
    table = SpliceTable(batch, P)
    for b in range(batch):
        base = b * PAGES_PER_REQ
        pages = list(range(base, base + PAGES_PER_REQ))
        table.append(b, 0, 0, CLOUD, pages[:CLOUD // P])
        table.append(b, 1, CLOUD, EDGE, pages[CLOUD // P:CLOUD // P + EDGE // P])
        table.append(b, 2, CLOUD + EDGE, SELF, pages[-1:])
        table.q_pos[b] = SEQ - 1
    return table


def host_batch_for(requests, k_host, v_host, q_host):
    """oracle.HostSpliceBatch of the given request subset (for the CPU legs)."""
    import numpy as np
    from oracle import oracle as O
    n = len(requests)
    segs, pt, indptr = [], [], [0]
    for i, b in enumerate(requests):
        base = i * PAGES_PER_REQ
        segs += [(0, CLOUD, 0, len(pt)), (1, EDGE, CLOUD, len(pt) + CLOUD // P),
                 (2, SELF, CLOUD + EDGE, len(pt) + CLOUD // P + EDGE // P)]
        pt += list(range(base, base + PAGES_PER_REQ))
        indptr.append(len(segs))
    return O.HostSpliceBatch(
        O.DT_BF16, HKV, HQ, D, P, np.ascontiguousarray(k_host), np.ascontiguousarray(v_host),
        np.array(indptr, np.int64), np.array(segs, dtype=O.SEGMENT_DTYPE),
        np.array(pt, np.int32), np.full(n, SEQ - 1, np.int64), O.DT_BF16,
        np.ascontiguousarray(q_host), 1)


def cpu_reference_rate(sb, threads, min_seconds=10.0, max_seconds=30.0):
    """Times the reference attention block (oracle/_ref) over all units of sb
    on `threads` host threads; returns (tokens/s, seconds, units)."""
    from oracle import oracle as O
    cache = O.RefBatchCache(sb)
    units_per_pass = sb.batch * sb.n_q_heads
    t0 = time.perf_counter()
    passes = 0
    while True:
        cache.attention(n_threads=threads)
        passes += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or el * (passes + 1) / passes > max_seconds:
            break
    tokens = passes * units_per_pass / sb.n_q_heads
    return tokens / el, el, passes * units_per_pass


def run_reference_skv(args, world):
    """--impl reference at N > 1: the reference attention block on config 4's
    workload (one request of 131072 + 512 keys x 32 heads per step: every
    partial_attention over the request's segments + merge_partials, fp64,
    oracle/_ref) on all host threads."""
    import numpy as np
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    ppr = SKV_CLOUD // P + SKV_EDGE // P
    per_pool = ppr * HKV * P * D
    k_host = O.fill_uniform(O.DT_BF16, per_pool, SEED_K).reshape(-1, HKV, P, D)
    v_host = O.fill_uniform(O.DT_BF16, per_pool, SEED_V).reshape(-1, HKV, P, D)
    q_host = O.fill_uniform(O.DT_BF16, HQ * D, SEED_Q).reshape(1, 1, HQ, D)
    segs = np.array([(0, SKV_CLOUD, 0, 0), (1, SKV_EDGE, SKV_CLOUD, SKV_CLOUD // P)], dtype=O.SEGMENT_DTYPE)
    sb = O.HostSpliceBatch(O.DT_BF16, HKV, HQ, D, P, np.ascontiguousarray(k_host), np.ascontiguousarray(v_host),
                           np.array([0, 2], np.int64), segs, np.arange(ppr, dtype=np.int32),
                           np.array([SKV_CLOUD + SKV_EDGE - 1], np.int64), O.DT_BF16, np.ascontiguousarray(q_host), 1)
    cache = O.RefBatchCache(sb)
    for _ in range(args.warmup):
        cache.attention(n_threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cache.attention(n_threads=threads)
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    value = 1.0 / step_s  # one token (query row of one request through one layer) per step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": skv_workload(world), "sample_requests_per_step": 1},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "cpu_model": cpu_model(), "kind": "reference",
                         "sample": f"1 of {SKV_B} requests x 32 heads per step ({SKV_CLOUD + SKV_EDGE} keys), "
                                   "reference attention block (partial_attention per segment + merge) "
                                   "in fp64 from oracle/_ref"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the same
    workload on the host cores (rank 0 only)."""
    import numpy as np
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    n_req = max(1, min(B, threads // 4))  # bounded sample per step
    per_pool = n_req * PAGES_PER_REQ * HKV * P * D
    k_host = O.fill_uniform(O.DT_BF16, per_pool, SEED_K).reshape(-1, HKV, P, D)
    v_host = O.fill_uniform(O.DT_BF16, per_pool, SEED_V).reshape(-1, HKV, P, D)
    q_host = O.fill_uniform(O.DT_BF16, n_req * HQ * D, SEED_Q).reshape(n_req, 1, HQ, D)
    sb = host_batch_for(list(range(n_req)), k_host, v_host, q_host)
    cache = O.RefBatchCache(sb)
    for _ in range(args.warmup):
        cache.attention(n_threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cache.attention(n_threads=threads)
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    value = n_req / step_s  # one token per request per step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_requests_per_step": n_req},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "cpu_model": cpu_model(),
                         "kind": "reference",
                         "sample": f"{n_req} of 32 requests x 32 heads per step (all segments), "
                                   "reference attention block (partial_attention per segment + "
                                   "merge) in fp64 from oracle/_ref"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the config 3/4/5 measurements (verify, split-KV, multi-tenant)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            if world > 1:
                run_reference_skv(args, world)
            else:
                run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.attention import Handle
    from paper_2504_11729_b200.splice import KVPool, SpliceTable, SplicedAttention

    if world > 1:
        run_sharded(args, world, rank, local_rank)
        dist.destroy_process_group()
        return

    h = Handle(local_rank)
    stream = torch.cuda.current_stream()
    num_pages = B * PAGES_PER_REQ
    pool = KVPool(num_pages, HKV, D, P, dtype="bf16", device=local_rank)
    lib = _capi.lib()
    sp = stream.cuda_stream
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.k.data_ptr(), pool.k.numel(),
                                    SEED_K, -1.0, 1.0, sp))
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.v.data_ptr(), pool.v.numel(),
                                    SEED_V, -1.0, 1.0, sp))
    q = torch.empty((B, 1, HQ, D), dtype=torch.bfloat16, device="cuda")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, q.data_ptr(), q.numel(), SEED_Q,
                                    -1.0, 1.0, sp))
    table = build_requests_table(SpliceTable, pool, B)
    attn = SplicedAttention(pool, table, HQ, 1, handle=h)
    o = torch.empty_like(q)
    lse = torch.empty((B, 1, HQ), dtype=torch.float32, device="cuda")

    def step():
        attn(q, o=o, lse=lse, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ------------------------------------------------------ device timing --
    with ClockSampler(local_rank) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = h.launch_count()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        launches = h.launch_count() - l0
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ----------------------------------------------------- end-to-end (host) --
    # A decode step as a serving loop runs it, through the public C-ABI, with
    # the cache GROWING by one token per request per step: the splice state
    # (ep_cache) gives every request's new token its page slot
    # (ep_cache_append_generated), the step's query rows and new K/V rows
    # arrive from pinned host memory together with those slots, ep_kv_append
    # writes the rows, ep_plan_update_cache re-plans from the grown cache
    # (host rebuild + async upload), ep_spliced_attention runs, and the
    # output rows go back to pinned host memory. Copies run on a copy stream,
    # double-buffered (step i+1's inputs arrive and step i-1's output leaves
    # while step i computes). The generated segment grows from 1 to 64 tokens
    # within its page, then is truncated back to 1 (ep_cache_truncate, as a
    # rejected draft would be), so the workload stays at 4609-4672 keys.
    from paper_2504_11729_b200.splice import SpliceCache
    cache = SpliceCache(1, B, P)
    for b in range(B):
        for sg in table.requests[b]:
            cache.append(b, sg.origin, sg.pos_offset, sg.length, sg.pages)
    # two plans of the same cache, used on alternate steps: step i's plan
    # refresh and K/V append (side stream) then overlap step i-1's attention
    # — the plan they patch was last read by step i-2, and the appended rows
    # lie past every key step i-1 reads
    attn_e = SplicedAttention.from_cache(pool, cache, HQ, 1, handle=h)
    attn_e2 = SplicedAttention.from_cache(pool, cache, HQ, 1, handle=h)
    # one pinned input blob per buffer j: [q | new K rows | new V rows | page | slot],
    # one H2D copy per step; copies and events through the CUDA runtime
    # directly (cuda.bindings), the library through its C-ABI (ctypes)
    from cuda.bindings import runtime as rt
    import ctypes as C
    qb, kvb, slb = q.numel() * 2, 2 * B * HKV * D * 2, 2 * B * 4
    in_bytes = qb + kvb + slb
    NB = 4  # input / output buffers in flight: the host may run NB - 1 steps ahead
    host_in = [torch.empty(in_bytes, dtype=torch.uint8).pin_memory() for _ in range(NB)]
    dev_in = [torch.empty(in_bytes, dtype=torch.uint8, device="cuda") for _ in range(NB)]
    kv_rows = torch.empty((2, B, HKV, D), dtype=torch.bfloat16)
    kv_rows[0] = pool.k[[b * PAGES_PER_REQ + PAGES_PER_REQ - 1 for b in range(B)], :, 0, :].cpu()
    kv_rows[1] = pool.v[[b * PAGES_PER_REQ + PAGES_PER_REQ - 1 for b in range(B)], :, 0, :].cpu()
    for j in range(NB):
        host_in[j][:qb].copy_(q.cpu().view(-1).view(torch.uint8))
        host_in[j][qb:qb + kvb].copy_(kv_rows.view(-1).view(torch.uint8))
    slots_np = [host_in[j][qb + kvb:].numpy().view(np.int32).reshape(2, B) for j in range(NB)]
    o_host = [torch.empty_like(o, device="cpu").pin_memory() for _ in range(NB)]
    o_dev = [torch.empty_like(o) for _ in range(NB)]
    ones = np.ones(B, np.int32)
    pd = pool.desc()
    pd_ref = C.byref(pd)
    in_ptr = [(host_in[j].data_ptr(), dev_in[j].data_ptr()) for j in range(NB)]
    q_ptr = [dev_in[j].data_ptr() for j in range(NB)]
    append_ptrs = [(dev_in[j].data_ptr() + qb + kvb, dev_in[j].data_ptr() + qb + kvb + 4 * B,
                    dev_in[j].data_ptr() + qb, dev_in[j].data_ptr() + qb + kvb // 2) for j in range(NB)]
    o_ptr = [(o_dev[j].data_ptr(), o_host[j].data_ptr()) for j in range(NB)]
    ob = o.numel() * 2
    copy = torch.cuda.Stream()
    cs = copy.cuda_stream
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def mkev():
        err, ev = rt.cudaEventCreateWithFlags(rt.cudaEventDisableTiming)
        assert err == rt.cudaError_t.cudaSuccess
        return ev

    ev_in = [mkev() for _ in range(NB)]    # inputs of buffer j landed
    ev_done = [mkev() for _ in range(NB)]  # attention on buffer j finished
    ev_out = [mkev() for _ in range(NB)]   # output of buffer j read back
    ev_prep = [mkev() for _ in range(NB)]  # plan refresh + K/V append of buffer j done
    gen = {"len": 1}
    trunc = [False] * NB                   # buffer j's token reused a truncated slot
    plans, cptr = [attn_e.plan, attn_e2.plan], cache.ptr
    side = torch.cuda.Stream()
    ss = side.cuda_stream

    def grow(j):
        """This step's token per request: a slot in the cache (host) -> pinned blob j."""
        trunc[j] = gen["len"] == P
        if trunc[j]:
            for b in range(B):
                cache.truncate(b, P - 1)
            gen["len"] = 1
        rt.cudaEventSynchronize(ev_in[j])  # the pinned blob j is free again
        sl = slots_np[j]
        cache.append_generated(ones, out=(sl[0], sl[1]))
        gen["len"] += 1

    def h2d(j):
        rt.cudaStreamWaitEvent(cs, ev_done[j], 0)  # buffer j's previous attention is done
        rt.cudaMemcpyAsync(in_ptr[j][1], in_ptr[j][0], in_bytes, H2D, cs)
        rt.cudaEventRecord(ev_in[j], cs)

    # the cache grows in step order on the host: step i's token is appended
    # (grow) before step i's plan refresh and after step i-1's
    def e2e_run(n):
        grow(0)
        h2d(0)
        for i in range(n):
            j = i % NB
            # side stream: plans[i % 2] (last read by step i-2's attention)
            # follows the grown cache, then the step's K/V rows are written
            rt.cudaStreamWaitEvent(ss, ev_done[(i - 2) % NB], 0)
            _capi.check(lib.ep_plan_update_cache(plans[i & 1], cptr, 0, 1, ss))
            rt.cudaStreamWaitEvent(ss, ev_in[j], 0)
            if trunc[j]:  # the token reuses a slot step i-1 may still read
                rt.cudaStreamWaitEvent(ss, ev_done[(i - 1) % NB], 0)
            _capi.check(lib.ep_kv_append(h.ptr, pd_ref, B, *append_ptrs[j], ss))
            rt.cudaEventRecord(ev_prep[j], ss)
            if i + 1 < n:
                grow((i + 1) % NB)
                h2d((i + 1) % NB)
            rt.cudaStreamWaitEvent(sp, ev_prep[j], 0)
            rt.cudaStreamWaitEvent(sp, ev_out[j], 0)  # o_dev[j] of step i-NB has been read back
            _capi.check(lib.ep_spliced_attention(h.ptr, plans[i & 1], pd_ref, _capi.EP_BF16, q_ptr[j],
                                                 _capi.EP_BF16, o_ptr[j][0], lse.data_ptr(), sp))
            rt.cudaEventRecord(ev_done[j], sp)
            rt.cudaStreamWaitEvent(cs, ev_done[j], 0)
            rt.cudaMemcpyAsync(o_ptr[j][1], o_ptr[j][0], ob, D2H, cs)
            rt.cudaEventRecord(ev_out[j], cs)
        stream.wait_stream(copy)
        stream.wait_stream(side)

    e2e_run(args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    stream.wait_event(e0)
    copy.wait_stream(stream)
    h0 = time.perf_counter()
    if os.environ.get("EP_E2E_PROFILE"):
        import cProfile
        import pstats
        pr = cProfile.Profile()
        pr.enable()
        e2e_run(args.steps)
        pr.disable()
        pstats.Stats(pr, stream=sys.stderr).sort_stats("tottime").print_stats(18)
    else:
        e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    host_us_e2e = (time.perf_counter() - h0) / args.steps * 1e6
    ms_e2e = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    # the last step's output equals a device-side recomputation on the same cache
    o_chk = torch.empty_like(o)
    attn_e.update_from_cache(stream=stream)
    attn_e(q, o=o_chk, lse=lse, stream=stream)
    torch.cuda.synchronize()
    ok = bool(torch.equal(o_host[(args.steps - 1) % NB].to("cuda"), o_chk))
    keys_e2e = [cache.end_position(b) for b in range(B)]
    attn_e.close()
    attn_e2.close()
    cache.close()
    for ev in ev_in + ev_done + ev_out + ev_prep:
        rt.cudaEventDestroy(ev)

    tokens_per_step = B * world
    value = tokens_per_step / (ms / 1e3)
    peak, peak_kind = peaks()
    achieved = ALG_BYTES / (ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("cfg2_decode_bytes_per_launch")
        except Exception:
            traffic = None

    n_ctas, n_items, n_pages = attn.info()
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": B * world, "seq_len": SEQ,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (604 MB of KV per step > 126 MB), no flush",
                   "plan": {"ctas": n_ctas, "work_items": n_items, "pages": n_pages}},
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_kind": peak_kind,
                     "note": "algorithmic bytes = 2*Hkv*d*2 B x 4609 keys x 32 requests per "
                             "step; time = K1 decode + K2 merge per step (CUDA events)",
                     "frac_of_8tbs_nominal": achieved / 8000.0},
        "e2e": {"value": tokens_per_step / (ms_e2e / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": o.numel() * 2, "ms_per_step": ms_e2e,
                "host_us_per_step": host_us_e2e,
                "result_check": ok,
                "cache_growth": "one token per request per step into the generated segment "
                                "(ep_cache_append_generated -> ep_kv_append -> ep_plan_update_cache), "
                                f"truncated back every {P - 1} steps; keys per request 4609..4672 "
                                f"(last step {min(keys_e2e)}..{max(keys_e2e)})",
                "overlap": "H2D of step i+1 and D2H of step i-1 on a copy stream "
                           "(double-buffered) while step i computes; step i's plan refresh and "
                           "K/V append on a side stream during step i-1's attention (two plans "
                           "of the cache, alternate steps)"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n_req = 4
        pg = n_req * PAGES_PER_REQ
        sb = host_batch_for(list(range(n_req)),
                            pool.k[:pg].view(torch.int16).cpu().numpy().view(np.uint16),
                            pool.v[:pg].view(torch.int16).cpu().numpy().view(np.uint16),
                            q[:n_req].view(torch.int16).cpu().numpy().view(np.uint16))
        rate, secs, units = cpu_reference_rate(sb, threads)
        line["cpu_baseline"] = {
            "value": rate, "unit": "tokens/s", "cores": threads, "cpu_model": cpu_model(), "kind": "reference",
            "sample": f"requests 0-3 of the same workload (128 (request, head) units per pass, "
                      f"{units} units in {secs:.1f} s), reference attention block in fp64 "
                      "(oracle/_ref, unmodified reference sources)"}
    if not args.no_extras:
        extras = run_extras(args, world, rank, h)
        line.update(extras)
        # the other configs' headline numbers, early in the line (a record
        # that keeps only part of a long line still shows them)
        line = summary_first(line, extras)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args, world, rank, local_rank):
    """N > 1: config 4 split-KV over the N GPUs as the measured step (local
    K1 over this rank's cloud shard + ONE peer-memory combine kernel pushing
    (o, lse) over NVLink and merging in rank order), the same workload
    unsharded on rank 0's GPU for the scaling reference, the e2e through the
    public API with host buffers, and config 2 replicas beside it."""
    import gc

    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import splitkv_bench as SB
    from paper_2504_11729_b200.attention import Handle
    from paper_2504_11729_b200.splitkv import PeerSplitKVCombine

    h = Handle(local_rank)
    stream = torch.cuda.current_stream()
    pool, table, attn, q, n_loc = SB.build_local(SKV_B, world, rank, h, cloud=SKV_CLOUD, edge=SKV_EDGE)
    rows = SKV_B * HQ
    comb = PeerSplitKVCombine(world, rank, rows, D, h)
    o_part = torch.empty((SKV_B, 1, HQ, D), dtype=torch.float32, device="cuda")
    lse_part = torch.empty((SKV_B, 1, HQ), dtype=torch.float32, device="cuda")
    out = torch.empty((rows, D), dtype=torch.bfloat16, device="cuda")
    out_lse = torch.empty((rows,), dtype=torch.float32, device="cuda")

    out4, out_lse4 = out.view(SKV_B, 1, HQ, D), out_lse.view(SKV_B, 1, HQ)

    def step(qq=q):  # ONE kernel per rank: local K1 pass + NVLink exchange + rank-order merge
        comb.attend(attn, qq, out=out4, out_lse=out_lse4, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    steps = args.steps

    def timed(fn, n):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1) / n], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local_rank) as clocks:
        l0 = h.launch_count()
        ms = timed(step, steps)
        launches = h.launch_count() - l0
    # the local pass alone (the same K1 over the shard without the exchange):
    # the HBM-bound part of the step; the rest of the fused step is the
    # exchange and the wait for the slowest rank
    ms_local = timed(lambda: attn(q, o=o_part, lse=lse_part, stream=stream), steps)
    combine_ms = max(ms - ms_local, 0.0)

    # e2e through the public API with host buffers: every step copies the
    # batch's query rows from pinned host memory and reads the merged output
    # rows back (every rank holds the same merged rows; each reads its own)
    q_host = q.cpu().pin_memory()
    o_host = torch.empty((rows, D), dtype=torch.bfloat16).pin_memory()
    q_dev = torch.empty_like(q)

    def e2e_step():
        q_dev.copy_(q_host, non_blocking=True)
        step(q_dev)
        o_host.copy_(out, non_blocking=True)

    for _ in range(args.warmup):
        e2e_step()
    ms_e2e = timed(e2e_step, steps)
    ok = bool(torch.equal(o_host.to("cuda"), out))

    # the same workload unsharded on one GPU (rank 0), for the scaling reference
    ms_1 = None
    if rank == 0:
        _, _, attn1, q1, _ = SB.build_local(SKV_B, 1, 0, h, cloud=SKV_CLOUD, edge=SKV_EDGE)
        o1 = torch.empty((SKV_B, 1, HQ, D), dtype=torch.bfloat16, device="cuda")
        for _ in range(args.warmup):
            attn1(q1, o=o1, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            attn1(q1, o=o1, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_1 = e0.elapsed_time(e1) / steps
        del attn1, q1, o1
        gc.collect()
        torch.cuda.empty_cache()
    dist.barrier()

    peak, peak_kind = peaks()
    loc_bytes = SKV_B * n_loc * 2 * HKV * D * 2
    t_loc = torch.tensor([float(loc_bytes)], device="cuda")
    dist.all_reduce(t_loc, op=dist.ReduceOp.MAX)
    achieved = float(t_loc.item()) / (ms_local / 1e3) / 1e9
    gather_bytes = (world - 1) * rows * (D + 1) * 4
    value = SKV_B / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": skv_workload(world), "global_batch": SKV_B, "seq_len": SKV_CLOUD + SKV_EDGE,
                   "parallelism": f"split-KV x{world}: contiguous cloud-KV shards, one per GPU; the "
                                  "(o, lse) combine fused into the decode kernel over NVLink peer memory",
                   "l2": f"inputs larger than L2 ({loc_bytes / 1e9:.1f} GB of KV per rank per step), no flush"},
        "value_1gpu": (SKV_B / (ms_1 / 1e3)) if ms_1 else None,
        "ms_per_step_1gpu": ms_1,
        "hbm_gbs_per_gpu": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                     "note": "per GPU: the largest rank's shard bytes (2*Hkv*d*2 B per key x keys x 32 "
                             "requests) / the local K1 time inside the step (per-step CUDA events, "
                             "max over ranks)"},
        "combine": {"ms": combine_ms, "bytes_received_per_rank": gather_bytes,
                    "nvlink_gbs": gather_bytes / (combine_ms / 1e3) / 1e9 if combine_ms > 0 else None,
                    "nvlink_frac": gather_bytes / (combine_ms / 1e3) / 900e9 if combine_ms > 0 else None,
                    "note": "fused step - local pass alone (max over ranks): the exchange and the wait "
                            "for the slowest rank; latency-bound (tiny messages)"},
        "e2e": {"value": SKV_B / (ms_e2e / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": q.numel() * 2, "d2h_bytes_per_step": rows * D * 2,
                "ms_per_step": ms_e2e, "result_check": ok,
                "path": "PeerSplitKVCombine.attend = ep_spliced_attention_splitkv (the C-ABI call) with "
                        "pinned host q / output"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    comb.close()
    del attn, pool, table, q, o_part, lse_part, out, out_lse, comb
    gc.collect()
    torch.cuda.empty_cache()
    if not args.no_extras:
        extras = {}
        # config 4 at batch 1 (latency): both combines
        skv = {}
        for cmb in ("fused", "peer", "nccl"):
            skv[f"batch1_{cmb}"] = SB.run(1, max(5, min(steps, 30)), 3, combine=cmb)
            gc.collect()
            torch.cuda.empty_cache()
        extras["splitkv"] = skv
        extras["cfg2_replicas"] = cfg2_replicas(args, world, rank, local_rank, h)
        line.update(extras)
    if rank == 0:
        print(json.dumps(line), flush=True)


def cfg2_replicas(args, world, rank, local_rank, h):
    """Config 2 (does not shard): every rank runs its own batch of 32."""
    import torch
    import torch.distributed as dist
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.splice import KVPool, SpliceTable, SplicedAttention
    stream = torch.cuda.current_stream()
    pool = KVPool(B * PAGES_PER_REQ, HKV, D, P, dtype="bf16", device=local_rank)
    lib = _capi.lib()
    sp = stream.cuda_stream
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.k.data_ptr(), pool.k.numel(), SEED_K, -1.0, 1.0, sp))
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, pool.v.data_ptr(), pool.v.numel(), SEED_V, -1.0, 1.0, sp))
    q = torch.empty((B, 1, HQ, D), dtype=torch.bfloat16, device="cuda")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, q.data_ptr(), q.numel(), SEED_Q, -1.0, 1.0, sp))
    attn = SplicedAttention(pool, build_requests_table(SpliceTable, pool, B), HQ, 1, handle=h)
    o = torch.empty_like(q)
    for _ in range(args.warmup):
        attn(q, o=o, stream=stream)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(20, min(args.steps, 500))
    e0.record(stream)
    for _ in range(n):
        attn(q, o=o, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / n], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"workload": WORKLOAD + f", one batch per GPU (x{world})", "ms_per_step": ms,
            "tokens_per_s": B * world / (ms / 1e3), "scaling": "weak"}


def summary_first(line, ex):
    """The line with a compact `summary` of the extras placed after `config`."""
    sm = {}
    try:
        if "verify_p50_ms" in ex:
            sm["cfg3_verify_p50_ms"] = {k: round(v, 4) for k, v in ex["verify_p50_ms"].items()}
        if "multitenant" in ex:
            sm["cfg5_ms_per_step"] = round(ex["multitenant"]["ms_per_step"], 4)
            sm["cfg5_unique_gbs"] = round(ex["multitenant"]["unique_gbs"])
        if "splitkv" in ex:
            sm["cfg4_1gpu_step_ms"] = {k: round(v["step_ms"], 4) for k, v in ex["splitkv"].items()
                                       if isinstance(v, dict) and "step_ms" in v}
        if "prefill" in ex:
            sm["prefill_ms"] = {k: round(v["ms"], 4) for k, v in ex["prefill"].items()}
            sm["prefill_tflops"] = {k: round(v["tflops"]) for k, v in ex["prefill"].items()}
        if "ingest" in ex and "device_async" in ex["ingest"]:
            sm["ingest_device_frame_us"] = round(ex["ingest"]["device_async"]["ms"] * 1e3, 2)
    except (KeyError, TypeError):
        pass
    out = {}
    for k, v in line.items():
        out[k] = v
        if k == "config":
            out["summary"] = sm
    out["summary_end"] = sm  # and at the end, for records that keep a line's tail
    return out


def run_extras(args, world, rank, h):
    """The other BASELINE configs, measured in the same run: config 3
    (speculative verify p50 latency, k = 4 / 8), config 5 (multi-tenant
    shared prefix), the prefill tiles and the KV ingest on rank 0 at N = 1; config 4 (128K split-KV: local K1 +
    the peer-memory combine kernel; at N > 1 also NCCL all-gather + K5 merge
    for comparison) at every N."""
    import gc

    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import splitkv_bench
    extras = {}
    steps = max(5, min(args.steps, 30))
    if world == 1:
        import multitenant_bench
        import verify_bench
        gc.collect()
        torch.cuda.empty_cache()
        ver = {}
        for k in (4, 8):
            ver[f"k{k}"] = verify_bench.run(k, steps, 3, h)
            gc.collect()
            torch.cuda.empty_cache()
        extras["verify"] = ver
        extras["verify_p50_ms"] = {k: v["step_p50_ms"] for k, v in ver.items()}
        extras["multitenant"] = multitenant_bench.run(steps, 3, h)
        gc.collect()
        torch.cuda.empty_cache()
        # prefill tiles on tcgen05, KV ingest from EPKV frames
        import ingest_bench
        import prefill_bench
        extras["prefill"] = {kind: prefill_bench.run(kind, 4 if kind == "cloud" else 32,
                                                     max(5, steps // 2), 3, h)
                             for kind in ("cloud", "edge")}
        gc.collect()
        torch.cuda.empty_cache()
        extras["ingest"] = ingest_bench.run(max(5, steps // 2), 3, h)
        gc.collect()
        torch.cuda.empty_cache()
        # the whole decoder on the GPU at config 1 (tiny
        # reference model, fp32), next to the reference's own decode_step
        import model_bench
        extras["model_cfg1"] = model_bench.run(64, 5, h, batch=64, cpu=not args.no_cpu_baseline)
        gc.collect()
        torch.cuda.empty_cache()
        # the link-level drop-in (reference model code + attention_dropin.cpp)
        # beside the same code on its own attention.cpp (config 1, 64 tokens)
        if not args.no_cpu_baseline:
            import dropin_bench
            try:
                extras["dropin_cfg1"] = dropin_bench.run(64, 2)
            except Exception as e:  # oracle/_ref not shipped: report, do not fail the bench
                extras["dropin_cfg1"] = {"unavailable": str(e)[:200]}
    skv = {}
    for b in (1, 32):
        skv[f"batch{b}"] = splitkv_bench.run(b, steps, 3, combine="peer")
        gc.collect()
        torch.cuda.empty_cache()
        if world > 1:
            skv[f"batch{b}_nccl"] = splitkv_bench.run(b, steps, 3, combine="nccl")
            gc.collect()
            torch.cuda.empty_cache()
    extras["splitkv"] = skv
    return extras


if __name__ == "__main__":
    main()
