"""Host logic of the cross-GPU split-KV path (config 4) on CPU: world_size 2
with the gloo backend. Each rank takes its contiguous cloud shard
(splitkv.shard_segments), computes its partial (o, lse) with the CPU oracle
(test stand-in for the CUDA kernel), and SplitKVCombine all-gathers the packed
partials and merges them in rank order — which must equal unsharded attention
over the whole spliced cache (attention.cpp:116-156)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2504_11729_b200.splitkv import Shard, SplitKVCombine, shard_segments

HQ, HKV, D, P = 4, 2, 16, 64


def _batch(shards, k_tok, v_tok, q, q_pos):
    """HostSpliceBatch of one request made of `shards` (global positions)."""
    pages_k, pages_v, recs, pt = [], [], [], []
    for s in shards:
        n_pg = -(-s.length // P)
        recs.append((s.origin, s.length, s.pos_offset, len(pt)))
        for i in range(n_pg):
            kp = np.zeros((HKV, P, D))
            vp = np.zeros((HKV, P, D))
            a = s.pos_offset + i * P
            b = min(s.pos_offset + s.length, a + P)
            kp[:, :b - a] = k_tok[a:b].transpose(1, 0, 2)
            vp[:, :b - a] = v_tok[a:b].transpose(1, 0, 2)
            pt.append(len(pages_k))
            pages_k.append(kp)
            pages_v.append(vp)
    kk = np.ascontiguousarray(np.stack(pages_k).astype(np.float32)) if pages_k else np.zeros((1, HKV, P, D), np.float32)
    vv = np.ascontiguousarray(np.stack(pages_v).astype(np.float32)) if pages_v else np.zeros((1, HKV, P, D), np.float32)
    return O.HostSpliceBatch(O.DT_F32, HKV, HQ, D, P, kk, vv,
                             np.array([0, len(recs)], np.int64),
                             np.array(recs, dtype=O.SEGMENT_DTYPE),
                             np.array(pt if pt else [0], np.int32),
                             np.array([q_pos], np.int64), O.DT_F32, q, 1)


def _case():
    segments = [(0, 1000), (1, 77), (2, 3)]  # cloud, edge, generated (incl. self)
    n = sum(l for _, l in segments)
    k_tok = O.fill_uniform(O.DT_F32, n * HKV * D, 41).reshape(n, HKV, D).astype(np.float64)
    v_tok = O.fill_uniform(O.DT_F32, n * HKV * D, 42).reshape(n, HKV, D).astype(np.float64)
    q = O.fill_uniform(O.DT_F32, HQ * D, 43).reshape(1, 1, HQ, D)
    return segments, k_tok, v_tok, q, n - 1


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        segments, k_tok, v_tok, q, q_pos = _case()
        shards = shard_segments(segments, world, rank)
        if shards:
            o, lse = O.spliced_attention(_batch(shards, k_tok, v_tok, q, q_pos))
        else:  # identity partial (attention.cpp:37-43)
            o, lse = np.zeros((1, 1, HQ, D)), np.full((1, 1, HQ), -np.inf)

        def gather(out, inp):
            parts = [torch.empty_like(inp) for _ in range(world)]
            dist.all_gather(parts, inp)
            out.copy_(torch.cat(parts))

        def merge(packed, w, rows, d):
            pk = packed.numpy().astype(np.float64).reshape(w, rows * (d + 1))
            parts = [(pk[p, :rows * d].reshape(rows, d), pk[p, rows * d:]) for p in range(w)]
            return O.merge_partials(parts)

        comb = SplitKVCombine(world, HQ, D, gather=gather, merge=merge)
        mo, ml = comb(torch.from_numpy(o.astype(np.float32)), torch.from_numpy(lse.astype(np.float32)))
        result_q.put((rank, [(s.origin, s.pos_offset, s.length) for s in shards], mo, ml))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_segments_partition():
    segs = [(0, 131072), (1, 512)]
    for world in (1, 2, 4, 8):
        got = [shard_segments(segs, world, r) for r in range(world)]
        flat = [s for g in got for s in g]
        assert [s.pos_offset for s in flat] == sorted(s.pos_offset for s in flat)
        assert sum(s.length for s in flat) == 131072 + 512
        pos = 0
        for s in flat:  # gapless, ordered = segment order across ranks
            assert s.pos_offset == pos
            pos += s.length
        assert all(s.origin == 0 for g in got[:-1] for s in g)
        assert got[-1][-1] == Shard(1, 131072, 512)


@pytest.mark.parametrize("world", [2])
def test_splitkv_gloo_matches_unsharded(world):
    segments, k_tok, v_tok, q, q_pos = _case()
    full = [Shard(o, p, l) for (o, l), p in zip(segments, np.cumsum([0] + [l for _, l in segments])[:-1])]
    want_o, want_l = O.spliced_attention(_batch(full, k_tok, v_tok, q, q_pos))
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, result_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [result_q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, shards, mo, ml in res:
        assert shards  # every rank owns part of the cloud prompt
        np.testing.assert_allclose(mo, want_o.reshape(HQ, D), rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(ml, want_l.reshape(HQ), rtol=1e-6)
