"""GPU: prompt-id-keyed shared cloud KV end to end — per-layer kv frames
(the reference's encode_frame) ingested once into shared pages, two sessions
splice them in front of private edge segments, and the spliced decode over
each layer equals the fp64 oracle on the same pages."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")]


def test_cached_prompt_shared_by_sessions(cuda_handle):
    import torch
    from paper_2504_11729_b200.prompt_cache import PromptKVCache
    from paper_2504_11729_b200.splice import KVPool, PageAllocator, SpliceTable, SplicedAttention
    from tests.cases import rel_err
    from tests.gpu_util import torch_from_raw
    L, Hkv, Hq, d, P, cloud, n_pages = 2, 2, 8, 128, 64, 150, 16
    alloc = PageAllocator(n_pages)
    pools = [KVPool(n_pages, Hkv, d, P, dtype="bf16", allocator=alloc) for _ in range(L)]
    cache = PromptKVCache(pools)
    rng = np.random.default_rng(1)
    frames = [O.kv_frame_encode(1, l, rng.uniform(-1, 1, (cloud, Hkv, d)),
                                rng.uniform(-1, 1, (cloud, Hkv, d))) for l in range(L)]
    entry = cache.ingest(42, frames, handle=cuda_handle)
    assert entry.seq_len == cloud and alloc.free_pages == n_pages - 3
    assert cache.ingest(42, [b"junk"] * L) is entry          # served from cache, no decode
    sessions = [cache.lookup(42) for _ in range(2)]
    edges = [70, 5]
    table = SpliceTable(2, P)
    for b, (e, n) in enumerate(zip(sessions, edges)):
        pages = alloc.alloc(-(-n // P))
        for pool in pools:
            kv = torch.from_numpy(rng.uniform(-1, 1, (2, n, Hkv, d))).to("cuda", torch.bfloat16)
            pool.write(pages, kv[0], kv[1])
        table.append(b, 0, 0, e.seq_len, e.pages)
        table.append(b, 1, e.seq_len, n, pages)
        table.q_pos[b] = e.seq_len + n - 1
    q_raw = O.fill_uniform(O.DT_BF16, 2 * Hq * d, 5).reshape(2, 1, Hq, d)
    q = torch_from_raw(np.ascontiguousarray(q_raw), O.DT_BF16)
    indptr, segs, pt = table.arrays()
    for pool in pools:
        attn = SplicedAttention(pool, table, Hq, 1, handle=cuda_handle)
        o, _ = attn(q, o_dtype=torch.float32)
        kp, vp = pool.host_raw()
        sb = O.HostSpliceBatch(kv_dtype=O.DT_BF16, n_kv_heads=Hkv, n_q_heads=Hq, d_head=d,
                               page_tokens=P, k_pages=kp, v_pages=vp, seg_indptr=indptr,
                               segs=segs, page_table=pt,
                               q_pos=np.ascontiguousarray(table.q_pos, dtype=np.int64),
                               q_dtype=O.DT_BF16, q=np.ascontiguousarray(q_raw), n_q=1)
        want, _ = O.spliced_attention(sb)
        assert rel_err(o.cpu().numpy(), want) < 1e-4
    # cloud pages are shared: the cache + two sessions hold each
    assert all(alloc.refcount(int(p)) == 3 for p in entry.pages)
    for s in sessions:
        cache.release(s)
    assert cache.evict(42) and all(alloc.refcount(int(p)) == 0 for p in entry.pages)
