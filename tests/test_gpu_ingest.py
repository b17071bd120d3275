"""GPU parity of the KV ingest (ep_kv_ingest_frame):
frames written by the reference's own encode_frame (oracle/_ref) are decoded
into the page pool from pinned host, pageable host and device memory, and
the pages must equal the C oracle's decode + round + scatter BIT-EXACTLY;
malformed frames fail with the reference's WireError kind."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")]


def _frame(seq, H, d, seed, specials=False):
    rng = np.random.default_rng(seed)
    k = rng.uniform(-2, 2, (seq, H, d))
    v = rng.standard_normal((seq, H, d)) * 3
    if specials:
        k[0, 0, :8] = [np.inf, -np.inf, np.nan, 1e300, -1e-300, 2 ** -140 * 1.5, 1 + 2 ** -8, 0.0]
    return O.kv_frame_encode(17, 2, k, v)


def _pool(H, d, dtype, num_pages):
    from paper_2504_11729_b200.splice import KVPool
    return KVPool(num_pages, H, d, 64, dtype=dtype)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("where", ["pinned", "pageable", "device"])
def test_ingest_bit_exact(cuda_handle, dtype, where):
    import torch
    seq, H, d = 200, 8, 128
    fr = _frame(seq, H, d, seed=3, specials=True)
    num_pages = 7
    pages = np.array([6, 2, 0, 4], dtype=np.int32)  # scattered, last page partial (200 = 3*64 + 8)
    pool = _pool(H, d, dtype, num_pages)
    if where == "pinned":
        src = torch.from_numpy(fr).pin_memory()
    elif where == "device":
        src = torch.from_numpy(fr).cuda()
    else:
        src = fr
    info = pool.ingest_frame(src, pages, handle=cuda_handle)
    torch.cuda.synchronize()
    assert (info.seq_len, info.n_heads, info.d_head, info.layer, info.session_id) == (seq, H, d, 2, 17)
    kv_dt = O.DT_BF16 if dtype == "bf16" else O.DT_F32
    code, _, want_k, want_v = O.kv_ingest(fr, kv_dt, 64, pages, num_pages)
    assert code == O.WIRE_OK
    if dtype == "bf16":
        got_k = pool.k.view(torch.int16).cpu().numpy().view(np.uint16)
        got_v = pool.v.view(torch.int16).cpu().numpy().view(np.uint16)
    else:
        got_k, got_v = pool.k.cpu().numpy(), pool.v.cpu().numpy()
    for p in pages:
        assert np.array_equal(got_k[p].view(np.uint8), want_k[p].view(np.uint8)), p
        assert np.array_equal(got_v[p].view(np.uint8), want_v[p].view(np.uint8)), p


def test_ingest_unaligned_device_frame(cuda_handle):
    """A device frame at an odd 8-byte offset (payload 16-byte aligned)."""
    import torch
    fr = _frame(64, 4, 64, seed=4)
    buf = torch.zeros(fr.size + 8, dtype=torch.uint8, device="cuda")
    buf[8:].copy_(torch.from_numpy(fr))
    pool = _pool(4, 64, "bf16", 2)
    pool.ingest_frame(buf[8:], [1], handle=cuda_handle)
    _, _, want_k, _ = O.kv_ingest(fr, O.DT_BF16, 64, [1], 2)
    got = pool.k.view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got[1], want_k[1])


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("shape", [(3, 20), (8, 128), (5, 36), (2, 6)])
@pytest.mark.parametrize("offset", [0, 8])
def test_ingest_row_shapes_and_offsets(cuda_handle, dtype, shape, offset):
    """Rows whose quad count is not a multiple of 32 (the last lane of a row
    reads its own fourth value), rows wider than one CTA (8 x 128), d_head % 4
    != 0 (2 x 6, the pair kernel), with the payload 16-byte aligned (offset 8:
    frame+24 lands on a 16-byte boundary) or at +8 (offset 0)."""
    import torch
    H, d = shape
    seq = 131
    fr = _frame(seq, H, d, seed=11 + H, specials=d >= 8)
    buf = torch.zeros(fr.size + 16, dtype=torch.uint8, device="cuda")
    buf[offset:offset + fr.size].copy_(torch.from_numpy(fr))
    pages = np.array([2, 0, 3], dtype=np.int32)
    pool = _pool(H, d, dtype, 4)
    pool.ingest_frame(buf[offset:offset + fr.size], pages, handle=cuda_handle)
    torch.cuda.synchronize()
    kv_dt = O.DT_BF16 if dtype == "bf16" else O.DT_F32
    code, _, want_k, want_v = O.kv_ingest(fr, kv_dt, 64, pages, 4)
    assert code == O.WIRE_OK
    if dtype == "bf16":
        got_k = pool.k.view(torch.int16).cpu().numpy().view(np.uint16)
        got_v = pool.v.view(torch.int16).cpu().numpy().view(np.uint16)
    else:
        got_k, got_v = pool.k.cpu().numpy(), pool.v.cpu().numpy()
    for p in pages:
        assert np.array_equal(got_k[p].view(np.uint8), want_k[p].view(np.uint8)), p
        assert np.array_equal(got_v[p].view(np.uint8), want_v[p].view(np.uint8)), p


def test_ingest_errors_match_reference(cuda_handle):
    import torch
    from paper_2504_11729_b200._capi import InvalidArgument, WireError
    fr = _frame(70, 4, 64, seed=5)
    pool = _pool(4, 64, "bf16", 2)
    cases = {}
    b = fr.copy(); b[0] = ord("Q"); cases["bad_magic"] = b
    b = fr.copy(); b[4] = 7; cases["bad_version"] = b
    cases["truncated"] = fr[:-1].copy()
    b = fr.copy(); b[6:10] = np.frombuffer(np.uint32(0xFFFFFFF0).tobytes(), np.uint8); cases["overflow"] = b
    b = fr.copy(); b[16] ^= 2; cases["shape"] = b
    cases["end_of_prefill"] = O.end_of_prefill_frame()
    for name, b in cases.items():
        want = O.kv_frame_decode(b, "ref")[0]
        for src in (b, torch.from_numpy(b).cuda()):
            with pytest.raises(WireError) as ei:
                pool.ingest_frame(src, [0, 1], handle=cuda_handle)
            assert ei.value.kind == want, (name, ei.value.kind, want)
    with pytest.raises(InvalidArgument):   # head shape does not match the pool (edge.cpp:53-55)
        _pool(8, 64, "bf16", 2).ingest_frame(fr, [0, 1], handle=cuda_handle)
    with pytest.raises(InvalidArgument):   # not enough pages
        pool.ingest_frame(fr, [0], handle=cuda_handle)


def test_ingested_kv_attends_like_oracle(cuda_handle):
    """Cloud KV arriving as a frame, then spliced decode over it (the edge's
    per-layer flow, edge.cpp:148-164) equals the oracle on the same pages."""
    import torch
    from paper_2504_11729_b200.splice import SpliceTable, SplicedAttention
    from tests.cases import rel_err
    from tests.gpu_util import torch_from_raw
    seq, H, Hq, d = 300, 2, 8, 128
    fr = _frame(seq, H, d, seed=6)
    pages = np.array([3, 1, 4, 0, 2], dtype=np.int32)
    pool = _pool(H, d, "bf16", 5)
    pool.ingest_frame(fr, pages, handle=cuda_handle)
    table = SpliceTable(1, 64)
    table.append(0, 0, 0, seq, pages)
    table.q_pos[0] = seq - 1
    attn = SplicedAttention(pool, table, Hq, 1, handle=cuda_handle)
    q_raw = O.fill_uniform(O.DT_BF16, Hq * d, 99).reshape(1, 1, Hq, d)
    o, lse = attn(torch_from_raw(np.ascontiguousarray(q_raw), O.DT_BF16), o_dtype=torch.float32)
    _, _, kp, vp = O.kv_ingest(fr, O.DT_BF16, 64, pages, 5)
    sb = O.HostSpliceBatch(kv_dtype=O.DT_BF16, n_kv_heads=H, n_q_heads=Hq, d_head=d, page_tokens=64,
                           k_pages=kp, v_pages=vp, seg_indptr=np.array([0, 1], np.int64),
                           segs=np.array([(0, seq, 0, 0)], dtype=O.SEGMENT_DTYPE), page_table=pages,
                           q_pos=np.array([seq - 1], np.int64), q_dtype=O.DT_BF16,
                           q=np.ascontiguousarray(q_raw), n_q=1)
    want_o, _ = O.spliced_attention(sb)
    assert rel_err(o.cpu().numpy(), want_o) < 1e-4


def _read_pool(pool, dtype):
    import torch
    if dtype == "bf16":
        return (pool.k.view(torch.int16).cpu().numpy().view(np.uint16),
                pool.v.view(torch.int16).cpu().numpy().view(np.uint16))
    return pool.k.cpu().numpy(), pool.v.cpu().numpy()


@pytest.mark.parametrize("where", ["device", "pinned"])
@pytest.mark.parametrize("offset", [1, 2, 4, 6, 30])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_ingest_misaligned_payload(cuda_handle, where, offset, dtype):
    """A kv frame at any byte offset of a receive buffer (e.g. right after a
    30-byte session_init frame): payloads that are not 8-byte aligned are
    staged into an aligned buffer instead of faulting (the reference's
    decode_frame reads bytes and accepts any alignment)."""
    import torch
    seq, H, d = 131, 4, 64
    fr = _frame(seq, H, d, seed=40 + offset, specials=True)
    buf = torch.zeros(fr.size + 64, dtype=torch.uint8)
    buf[offset:offset + fr.size].copy_(torch.from_numpy(fr))
    buf = buf.cuda() if where == "device" else buf.pin_memory()
    pages = np.array([2, 0, 3], dtype=np.int32)
    pool = _pool(H, d, dtype, 4)
    pool.ingest_frame(buf[offset:offset + fr.size], pages, handle=cuda_handle)
    torch.cuda.synchronize()
    kv_dt = O.DT_BF16 if dtype == "bf16" else O.DT_F32
    _, _, want_k, want_v = O.kv_ingest(fr, kv_dt, 64, pages, 4)
    got_k, got_v = _read_pool(pool, dtype)
    for p in pages:
        assert np.array_equal(got_k[p].view(np.uint8), want_k[p].view(np.uint8)), p
        assert np.array_equal(got_v[p].view(np.uint8), want_v[p].view(np.uint8)), p


def test_ingest_staging_ordered_across_streams(cuda_handle):
    """Pageable frames share one staging buffer per handle: a second frame
    staged on another stream must not overwrite the first frame's bytes before
    the first ingest kernel has read them."""
    import torch
    seq, H, d = 4096, 8, 128
    frs = [_frame(seq, H, d, seed=60 + i) for i in range(2)]
    pools = [_pool(H, d, "bf16", 64) for _ in range(2)]
    pages = np.arange(64, dtype=np.int32)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    # a long kernel ahead of the first ingest on s0 keeps its read pending
    with torch.cuda.stream(s0):
        torch.cuda._sleep(20_000_000)
    pools[0].ingest_frame(frs[0], pages, handle=cuda_handle, stream=s0)
    pools[1].ingest_frame(frs[1], pages, handle=cuda_handle, stream=s1)
    torch.cuda.synchronize()
    for fr, pool in zip(frs, pools):
        _, _, want_k, want_v = O.kv_ingest(fr, O.DT_BF16, 64, pages, 64)
        got_k, got_v = _read_pool(pool, "bf16")
        assert np.array_equal(got_k, want_k) and np.array_equal(got_v, want_v)


@pytest.mark.parametrize("offset", [0, 8, 3])
def test_ingest_async_device_frames(cuda_handle, offset):
    """ep_kv_ingest_frame_async: a valid device frame is ingested with no host
    sync and the pages equal the synchronous path's; a corrupted header is
    caught by the kernel (nothing written) and reported at the next poll with
    the reference's WireError kind; the status clears after the poll."""
    import torch
    from paper_2504_11729_b200._capi import InvalidArgument, WireError
    from paper_2504_11729_b200.splice import KVPool
    seq, H, d = 200, 8, 128
    fr = _frame(seq, H, d, seed=70, specials=True)
    pages = np.array([6, 2, 0, 4], dtype=np.int32)

    def dev(b):
        buf = torch.zeros(b.size + 16, dtype=torch.uint8, device="cuda")
        buf[offset:offset + b.size].copy_(torch.from_numpy(b))
        return buf[offset:offset + b.size]

    pool = _pool(H, d, "bf16", 7)
    pool.ingest_frame_async(dev(fr), pages, handle=cuda_handle)
    KVPool.ingest_poll(cuda_handle)
    _, _, want_k, want_v = O.kv_ingest(fr, O.DT_BF16, 64, pages, 7)
    got_k, got_v = _read_pool(pool, "bf16")
    for p in pages:
        assert np.array_equal(got_k[p], want_k[p]) and np.array_equal(got_v[p], want_v[p])

    bad = {}
    b = fr.copy(); b[0] = ord("Q"); bad["bad_magic"] = b
    b = fr.copy(); b[4] = 7; bad["bad_version"] = b
    b = fr.copy(); b[5] = 3; bad["end_of_prefill_type"] = b
    b = fr.copy(); b[16:20] = np.frombuffer(np.uint32(seq - 1).tobytes(), np.uint8); bad["seq"] = b
    for name, b in bad.items():
        want = O.kv_frame_decode(b, "ref")[0]
        p2 = _pool(H, d, "bf16", 7)
        p2.ingest_frame_async(dev(b), pages, handle=cuda_handle)
        with pytest.raises(WireError) as ei:
            KVPool.ingest_poll(cuda_handle)
        assert ei.value.kind == want, (name, ei.value.kind, want)
        assert not p2.k.view(torch.int16).any().item(), name   # nothing written
        KVPool.ingest_poll(cuda_handle)                        # cleared
    # frame whose head shape differs from the pool's (same byte length: 4 x 256)
    fr2 = _frame(seq, 4, 256, seed=71)
    p3 = _pool(H, d, "bf16", 7)
    p3.ingest_frame_async(dev(fr2), pages, handle=cuda_handle)
    with pytest.raises(InvalidArgument):
        KVPool.ingest_poll(cuda_handle)
    # a length that does not fit the pool shape fails immediately
    with pytest.raises(WireError):
        pool.ingest_frame_async(dev(fr[:-1].copy()), pages, handle=cuda_handle)


@pytest.mark.parametrize("P", [64, 128, 192])
@pytest.mark.parametrize("shape", [(8, 128), (4, 64)])
@pytest.mark.parametrize("offset", [0, 8])
def test_ingest_page_sizes(cuda_handle, P, shape, offset):
    """The row kernel's compile-time quad splits (d_head 128 -> 32 quads,
    64 -> 16) and its page index by shift (64, 128) or division (192 tokens
    per page), bf16 pages: bit-exact vs the C oracle's decode + round + scatter."""
    import torch
    from paper_2504_11729_b200.splice import KVPool
    H, d = shape
    seq = 2 * P + 37  # a partial last page
    fr = _frame(seq, H, d, seed=P + d, specials=True)
    buf = torch.zeros(fr.size + 16, dtype=torch.uint8, device="cuda")
    buf[offset:offset + fr.size].copy_(torch.from_numpy(fr))
    pages = np.array([3, 0, 2], dtype=np.int32)
    pool = KVPool(4, H, d, P, dtype="bf16")
    pool.ingest_frame(buf[offset:offset + fr.size], pages, handle=cuda_handle)
    torch.cuda.synchronize()
    code, _, want_k, want_v = O.kv_ingest(fr, O.DT_BF16, P, pages, 4)
    assert code == O.WIRE_OK
    got_k = pool.k.view(torch.int16).cpu().numpy().view(np.uint16)
    got_v = pool.v.view(torch.int16).cpu().numpy().view(np.uint16)
    for p in pages:
        assert np.array_equal(got_k[p].view(np.uint8), want_k[p].view(np.uint8)), p
        assert np.array_equal(got_v[p].view(np.uint8), want_v[p].view(np.uint8)), p
