"""BASELINE config 4: long-context split-KV. A 131072-token cloud prompt per
request is sharded contiguously across the P GPUs of one box (edge 512 on the
last rank); every rank runs the spliced decode kernel over its shard (fp32
o + lse), then the combine in rank order — either ONE peer-memory combine kernel over NVLink
(ep_splitkv_combine_dev, default) or NCCL all-gather + the K5 merge.

    torchrun --nproc-per-node P tools/splitkv_bench.py [--batch 32] [--check]

Times (CUDA events, max over ranks): the local attention, and the whole step
(local attention + combine). --check compares rank 0's merged
output with an unsharded single-GPU run of the same batch.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HQ, HKV, D, P = 32, 8, 128, 64


def _hbm_peak():
    """Measured HBM copy GB/s from the driver-written MEASURED_PEAKS.json."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback
CLOUD, EDGE = 131072, 512


def build_local(batch, world, rank, h, cloud=CLOUD, edge=EDGE, seed=41):
    """This rank's pool/table/plan for `batch` requests; KV of global token t of
    request b is row t of a seeded token-major tensor (identical on all ranks)."""
    import numpy as np
    import torch
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.splice import KVPool, SpliceTable, SplicedAttention
    from paper_2504_11729_b200.splitkv import shard_segments
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    segments = [(0, cloud), (1, edge)]
    shards = shard_segments(segments, world, rank)
    n_loc = sum(x.length for x in shards)
    pages_per_req = sum(-(-x.length // P) for x in shards)
    pool = KVPool(max(1, batch * pages_per_req), HKV, D, P, dtype="bf16")
    table = SpliceTable(batch, P)
    n_total = cloud + edge
    tok = torch.empty((n_total, HKV, D), dtype=torch.bfloat16, device="cuda")
    for b in range(batch):
        pg = b * pages_per_req
        page_lists = []
        for x in shards:
            npg = -(-x.length // P)
            page_lists.append(np.arange(pg, pg + npg, dtype=np.int32))
            pg += npg
        for kv, off in (("k", 0), ("v", 1)):
            # the request's whole token-major K (or V), identical on every rank;
            # this rank keeps its shards' rows
            _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, tok.data_ptr(), tok.numel(),
                                            seed * 1000003 + b * 7919 + off * 104729, -1.0, 1.0, s))
            target = pool.k if kv == "k" else pool.v
            for x, pages in zip(shards, page_lists):
                t = torch.arange(x.length, device="cuda")
                pidx = torch.as_tensor(pages.astype(np.int64), device="cuda")[t // P]
                target[pidx, :, t % P, :] = tok[x.pos_offset:x.pos_offset + x.length]
        for x, pages in zip(shards, page_lists):
            table.append(b, x.origin, x.pos_offset, x.length, pages)
        table.q_pos[b] = cloud + edge - 1
    attn = SplicedAttention(pool, table, HQ, 1, handle=h)
    q = torch.empty((batch, 1, HQ, D), dtype=torch.bfloat16, device="cuda")
    _capi.check(lib.ep_fill_uniform(h.ptr, _capi.EP_BF16, q.data_ptr(), q.numel(), seed + 5, -1.0,
                                    1.0, s))
    return pool, table, attn, q, n_loc


def oracle_check(pool1, q1, b, heads, out, out_lse, cloud=CLOUD, edge=EDGE):
    """fp64 oracle (oracle/ep_oracle.c) on units (b, h) of the unsharded
    layout of build_local(batch, 1, ...), against the merged rows out /
    out_lse [rows]; returns (max rel err of o, of lse) with the reference's
    metric |got - want| / max(1, |want|)."""
    import numpy as np
    import torch
    from oracle import oracle as O
    ppr = -(-cloud // P) + -(-edge // P)
    pages = torch.arange(b * ppr, (b + 1) * ppr, device=pool1.k.device)
    kp = pool1.k[pages].view(torch.int16).cpu().numpy().view(np.uint16)
    vp = pool1.v[pages].view(torch.int16).cpu().numpy().view(np.uint16)
    segs = np.array([(0, cloud, 0, 0), (1, edge, cloud, -(-cloud // P))], dtype=O.SEGMENT_DTYPE)
    qb = q1[b:b + 1].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    sb = O.HostSpliceBatch(kv_dtype=O.DT_BF16, n_kv_heads=HKV, n_q_heads=HQ, d_head=D, page_tokens=P,
                           k_pages=np.ascontiguousarray(kp), v_pages=np.ascontiguousarray(vp),
                           seg_indptr=np.array([0, 2], np.int64), segs=segs,
                           page_table=np.arange(ppr, dtype=np.int32),
                           q_pos=np.array([cloud + edge - 1], np.int64), q_dtype=O.DT_BF16,
                           q=np.ascontiguousarray(qb), n_q=1)
    want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4, units=heads)
    got_o = out.float().cpu().numpy().reshape(-1, HQ, D)[b]
    got_l = out_lse.cpu().numpy().reshape(-1, HQ)[b]
    e_o = max(float(np.max(np.abs(got_o[h] - want_o[0, 0, h]) / np.maximum(1.0, np.abs(want_o[0, 0, h]))))
              for h in heads)
    e_l = max(float(abs(got_l[h] - want_l[0, 0, h]) / max(1.0, abs(want_l[0, 0, h]))) for h in heads)
    return e_o, e_l


def run(batch, steps, warmup, check=False, combine="peer", graph=False, cloud=CLOUD, edge=EDGE):
    """combine: "peer" = one ep_splitkv_combine_dev kernel over NVLink peer
    memory; "nccl" = NCCL all-gather + K5 merge; "fused" = the combine inside
    the decode kernel (ep_spliced_attention_splitkv). graph: replay the step
    (attention + combine) as one CUDA graph (removes host launch overhead)."""
    import torch
    import torch.distributed as dist
    from paper_2504_11729_b200.attention import Handle
    from paper_2504_11729_b200.splitkv import PeerSplitKVCombine, SplitKVCombine
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    h = Handle(torch.cuda.current_device())
    pool, table, attn, q, n_loc = build_local(batch, world, rank, h, cloud=cloud, edge=edge)
    rows = batch * HQ
    comb = None
    if world > 1:
        comb = (PeerSplitKVCombine(world, rank, rows, D, h) if combine in ("peer", "fused") else
                SplitKVCombine(world, rows, D, handle=h, device="cuda"))
    fused = world > 1 and combine == "fused"
    o_part = torch.empty((batch, 1, HQ, D), dtype=torch.float32, device="cuda")
    lse_part = torch.empty((batch, 1, HQ), dtype=torch.float32, device="cuda")
    out = torch.empty((rows, D), dtype=torch.bfloat16, device="cuda")
    out_lse = torch.empty((rows,), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step(st=stream):
        if fused:  # one kernel: local pass + NVLink exchange + rank-order merge
            comb.attend(attn, q, out=out.view(batch, 1, HQ, D), out_lse=out_lse.view(batch, 1, HQ), stream=st)
            return
        attn(q, o=o_part, lse=lse_part, stream=st)
        if comb is not None:
            comb(o_part.view(rows, D), lse_part.view(rows), out=out, out_lse=out_lse, stream=st)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(stream)
    for _ in range(steps):
        attn(q, o=o_part, lse=lse_part, stream=stream)
    e[1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    run_step = step
    if graph:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step(side)  # warm the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            step(torch.cuda.current_stream())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        run_step = g.replay
    import time
    e[2].record(stream)
    h0 = time.perf_counter()
    for _ in range(steps):
        run_step()
    host_us = (time.perf_counter() - h0) / steps * 1e6
    e[3].record(stream)
    torch.cuda.synchronize()
    t_attn = e[0].elapsed_time(e[1]) / steps
    t_step = e[2].elapsed_time(e[3]) / steps
    t = torch.tensor([t_attn, t_step], device="cuda")
    per_rank_times = None
    if world > 1:
        allt = torch.empty((world, 2), device="cuda")
        dist.all_gather_into_tensor(allt, t)
        per_rank_times = [[round(float(x), 4) for x in r] for r in allt.cpu()]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_attn, t_step = float(t[0]), float(t[1])
    per_rank = None
    if world > 1 and not fused:
        # where the step goes on each rank: attention vs combine (incl. waiting for peers)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps + 1)]
        torch.cuda.synchronize()
        dist.barrier()
        ev[0].record(stream)
        for i in range(steps):
            attn(q, o=o_part, lse=lse_part, stream=stream)
            ev[2 * i + 1].record(stream)
            comb(o_part.view(rows, D), lse_part.view(rows), out=out, out_lse=out_lse, stream=stream)
            ev[2 * i + 2].record(stream)
        torch.cuda.synchronize()
        a_ms = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps)) / steps
        c_ms = sum(ev[2 * i + 1].elapsed_time(ev[2 * i + 2]) for i in range(steps)) / steps
        mine = torch.tensor([a_ms, c_ms], device="cuda")
        allr = torch.empty((world, 2), device="cuda")
        dist.all_gather_into_tensor(allr, mine)
        per_rank = [[round(float(x), 4) for x in r] for r in allr.cpu()]
    t_attn_b2b = t_attn
    if per_rank:
        # inside the step the attention and the combine are serialised (the
        # combine waits for every rank): report those parts, max over ranks
        t_attn = max(r[0] for r in per_rank)
    loc_bytes = batch * n_loc * 2 * HKV * D * 2
    gather_bytes = (world - 1) * rows * (D + 1) * 4  # received per rank
    res = {
        "workload": f"cfg4 split-KV: {cloud} cloud + {edge} edge keys, Hq=32 Hkv=8 d=128 bf16, "
                    f"batch {batch}, {world} GPU(s)",
        "batch": batch, "gpus": world, "combine": combine if world > 1 else None, "step_ms": t_step, "local_attention_ms": t_attn,
        "combine_ms": (max(r[1] for r in per_rank) if per_rank else 0.0),
        "local_attention_back_to_back_ms": t_attn_b2b,
        "tokens_per_s": batch / (t_step / 1e3),
        "local_hbm_gbs": loc_bytes / (t_attn / 1e3) / 1e9,
        "allgather_bytes_per_rank": gather_bytes,
        # NVLink roofline of the exchange: bytes each rank receives over the
        # combine time vs 900 GB/s per direction (NVLink 5) — tiny messages,
        # so the combine is latency-bound and this fraction is small
        "combine_nvlink_gbs": (gather_bytes / (max(r[1] for r in per_rank) / 1e3) / 1e9
                               if per_rank else None),
        "combine_nvlink_frac": (gather_bytes / (max(r[1] for r in per_rank) / 1e3) / 900e9
                                if per_rank else None),
        "local_hbm_frac": loc_bytes / (t_attn / 1e3) / (_hbm_peak() * 1e9),
        "graph": graph, "host_launch_us_per_step": host_us,
    }
    if per_rank is not None:
        res["per_rank_attention_combine_ms"] = per_rank
    if per_rank_times is not None:
        res["per_rank_attention_b2b_step_ms"] = per_rank_times
    if check:
        ok = True
        if world > 1:
            # rank 0 recomputes the unsharded batch on its own GPU, and the
            # fp64 oracle recomputes sampled units of the last request from
            # the same pages (merge in rank = segment order, attention.cpp:116-145)
            if rank == 0:
                pool1, table1, attn1, q1, _ = build_local(batch, 1, 0, h, cloud=cloud, edge=edge)
                o1, l1 = attn1(q1, o_dtype=torch.float32)
                torch.cuda.synchronize()
                err = (out.float() - o1.reshape(rows, D)).abs().max().item()
                lerr = (out_lse - l1.reshape(rows)).abs().max().item()
                res["check_max_abs_err"] = err
                res["check_lse_max_abs_err"] = lerr
                ok = err < 2e-2 and lerr < 1e-3
                e_o, e_l = oracle_check(pool1, q1, batch - 1, [0, 13, 31], out, out_lse, cloud, edge)
                res["check_oracle_rel_err"] = e_o
                res["check_oracle_lse_rel_err"] = e_l
                ok = ok and e_o <= 2e-2 and e_l <= 1e-4
        res["check_ok"] = ok
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()  # no peer still writes into our buffers
        if hasattr(comb, "close"):
            comb.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 32])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--combine", choices=["peer", "nccl", "fused"], nargs="+", default=["peer"])
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--edge", type=int, default=EDGE)
    ap.add_argument("--cloud", type=int, default=CLOUD,
                    help="cloud tokens (e.g. 131072 / P on one GPU = one rank's local pass)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("EP_TRACE_FILE") and world > 1:  # debug traces: one file per rank
        os.environ["EP_TRACE_FILE"] = os.environ["EP_TRACE_FILE"] + f".r{local}"
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    for cmb in args.combine:
        for b in args.batch:
            r = run(b, args.steps, args.warmup, check=args.check, combine=cmb, graph=args.graph,
                    cloud=args.cloud, edge=args.edge)
            if int(os.environ.get("RANK", "0")) == 0:
                print(json.dumps(r), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
