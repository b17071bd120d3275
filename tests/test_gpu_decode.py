"""GPU parity of K1/K2 (spliced flash-decode over the paged splice table)
against the fp64 oracle on identical rounded inputs. Tolerances are the
north_star's: 1e-3 relative (fp32 KV) and 2e-2 (bf16 KV), metric
|got - want| / max(1, |want|) (acceptance_test.cpp:107-109)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import cases as CS
from tests import splice_cases as SC
from tests.gpu_util import to_device, tol_for, torch_from_raw

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _check(o, lse, want_o, want_l, kv_dtype, units=None, Hq=None):
    o = o.float().cpu().numpy().astype(np.float64)
    lse = lse.cpu().numpy().astype(np.float64)
    if units is not None:
        sel = [(int(u) // Hq, int(u) % Hq) for u in units]
        o = np.stack([o[b, :, h] for b, h in sel])
        lse = np.stack([lse[b, :, h] for b, h in sel])
        want_o = np.stack([want_o[b, :, h] for b, h in sel])
        want_l = np.stack([want_l[b, :, h] for b, h in sel])
    err_o = CS.rel_err(o, want_o)
    fin = np.isfinite(want_l)
    assert np.array_equal(np.isfinite(lse), fin)
    err_l = CS.rel_err(lse[fin], want_l[fin])
    tol = tol_for(kv_dtype)
    assert err_o <= tol, f"out rel err {err_o:.3e} > {tol}"
    assert err_l <= 1e-4, f"lse rel err {err_l:.3e}"
    return err_o, err_l


@pytest.mark.parametrize("name", list(SC.SMALL_CASES))
def test_small_cases_vs_reference_golden(cuda_handle, name):
    gold = np.load(os.path.join(GOLD, "splice_golden.npz"))
    sb = SC.small_case(name)
    pool, table, attn, q = to_device(sb, cuda_handle)
    o, lse = attn(q, o_dtype=q.dtype)
    e1 = _check(o, lse, gold[f"{name}/out"], gold[f"{name}/lse"], sb.kv_dtype)
    # fp32 output path as well
    import torch
    o32, lse32 = attn(q, o_dtype=torch.float32)
    e2 = _check(o32, lse32, gold[f"{name}/out"], gold[f"{name}/lse"], sb.kv_dtype)
    print(name, "rel err (o, lse):", e1, e2)


def test_deterministic(cuda_handle):
    sb = SC.small_case("gqa4_bf16_decode")
    _, _, attn, q = to_device(sb, cuda_handle)
    o1, l1 = attn(q)
    o2, l2 = attn(q)
    assert bool((o1 == o2).all()) and bool((l1 == l2).all())


def _big_case(kv_dtype, Hq, Hkv, d, requests, n_q=1, seed=3):
    return SC.make_case(kv_dtype, Hq, Hkv, d, requests, n_q=n_q, seed=seed)


def test_config2_shape_full_size(cuda_handle):
    """BASELINE config 2: Hq=32, Hkv=8, d=128, bf16, private 4096 cloud + 512
    edge + self token per request, B=32. Checked on 96 random units."""
    reqs = [[(SC.CLOUD, 4096, None), (SC.EDGE, 512, None), (SC.GEN, 1, None)]] * 32
    sb = _big_case(O.DT_BF16, 32, 8, 128, reqs)
    _, _, attn, q = to_device(sb, cuda_handle)
    o, lse = attn(q)
    units = np.random.default_rng(0).choice(32 * 32, 96, replace=False)
    want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4, units=units)
    print("cfg2 rel err:", _check(o, lse, want_o, want_l, sb.kv_dtype, units, 32))
    print("plan (ctas, items, pages):", attn.info())


def test_config5_shared_prefix_ragged(cuda_handle):
    """BASELINE config 5 structure at reduced batch: requests share one 8192-token
    cloud segment (same pages) with ragged U{32..2048} edge segments."""
    r = O.SplitMix64(5)
    reqs = [[(SC.CLOUD, 8192, "cloud"), (SC.EDGE, 32 + r.next_u64() % 2017, None),
             (SC.GEN, 1, None)] for _ in range(24)]
    sb = _big_case(O.DT_BF16, 32, 8, 128, reqs, seed=4)
    _, _, attn, q = to_device(sb, cuda_handle)
    o, lse = attn(q)
    units = np.random.default_rng(1).choice(24 * 32, 64, replace=False)
    want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4, units=units)
    print("cfg5 rel err:", _check(o, lse, want_o, want_l, sb.kv_dtype, units, 32))


def test_config1_real_model_kv(cuda_handle):
    """Config 1 KV produced by the reference model itself (L=2, H=4, D=256,
    cloud 512 + edge 64), fp32 pages, MHA d=64; synthetic decode queries."""
    import json
    from tests.conftest import require_ref
    require_ref()
    g = json.load(open(os.path.join(GOLD, "model_golden.json")))
    m = O.RefModel(2, 4, 256, 256, 1024, 42)
    sess = m.session(g["cfg1_cloud"], g["cfg1_edge"])
    H, d, P = 4, 64, 64
    for layer in range(2):
        ks, vs, segs = [], [], []
        for s in range(sess.n_segments):
            k, v, pos, org = sess.segment(layer, s)
            segs.append((org, k.shape[0], pos))
            ks.append(k)
            vs.append(v)
        # one page-aligned pool: segment s occupies its own pages
        n_pages = sum(-(-n // P) for _, n, _ in segs) + 1
        kp = np.zeros((n_pages, H, P, d), np.float32)
        vp = np.zeros((n_pages, H, P, d), np.float32)
        recs, pt, page = [], [], 0
        for (org, n, pos), k, v in zip(segs, ks, vs):
            recs.append((org, n, pos, len(pt)))
            for t in range(n):
                kp[page + t // P, :, t % P] = k[t].reshape(H, d)
                vp[page + t // P, :, t % P] = v[t].reshape(H, d)
            npg = -(-n // P)
            pt.extend(range(page, page + npg))
            page += npg
        end = segs[-1][2] + segs[-1][1]
        q = O.fill_uniform(O.DT_F32, H * d, 77 + layer).reshape(1, 1, H, d)
        sb = O.HostSpliceBatch(O.DT_F32, H, H, d, P, kp, vp, np.array([0, len(recs)], np.int64),
                               np.array(recs, dtype=O.SEGMENT_DTYPE), np.array(pt, np.int32),
                               np.array([end - 1], np.int64), O.DT_F32, q, 1)
        want_o, want_l = O.spliced_attention(sb, n_threads=4)
        _, _, attn, qd = to_device(sb, cuda_handle)
        o, lse = attn(qd)
        print("cfg1 layer", layer, "rel err:", _check(o, lse, want_o, want_l, O.DT_F32))


def test_decode_loop_with_plan_update(cuda_handle):
    """Generated tokens appended page-slot by page-slot (no segment copy,
    cf. cache.cpp:55-80); the plan is updated in place each step."""
    import torch
    sb = SC.make_case(O.DT_BF16, 8, 2, 128, [[(SC.CLOUD, 190, None), (SC.EDGE, 40, None)],
                                              [(SC.EDGE, 63, None)]], seed=9, spare_pages=8)
    pool, table, attn, q = to_device(sb, cuda_handle)
    pool._free = [p for p in range(pool.num_pages - 1, -1, -1)
                  if p not in set(sb.page_table.tolist())]
    host_k, host_v = sb.k_pages.copy(), sb.v_pages.copy()
    for step in range(70):
        for b in range(table.batch):
            pages, start = table.append_generated_tokens(b, 1, pool)
            kv = O.fill_uniform(O.DT_BF16, 2 * 2 * 128, 1000 + step * 7 + b).reshape(2, 2, 128)
            pool.write(pages, torch_from_raw(kv[0:1].copy(), O.DT_BF16),
                       torch_from_raw(kv[1:2].copy(), O.DT_BF16), start=start)
            host_k[pages[0], :, start] = kv[0]
            host_v[pages[0], :, start] = kv[1]
            table.q_pos[b] = table.end_position(b) - 1
        attn.update()
        o, lse = attn(q)
        if step % 23 == 0 or step == 69:
            indptr, segs, pt = table.arrays()
            hb = O.HostSpliceBatch(sb.kv_dtype, 2, 8, 128, 64, host_k, host_v, indptr, segs, pt,
                                   table.q_pos.copy(), sb.q_dtype, sb.q, 1)
            want_o, want_l = O.spliced_attention(hb, n_threads=4)
            _check(o, lse, want_o, want_l, sb.kv_dtype)


def test_plan_rejects_bad_tables(cuda_handle):
    import ctypes as C
    from paper_2504_11729_b200 import _capi
    sb = SC.small_case("gqa4_bf16_decode")
    pool, table, attn, q = to_device(sb, cuda_handle)
    indptr, segs, pt = table.arrays()
    segs_bad = segs.copy()
    segs_bad[1]["pos_offset"] += 1  # gap (cache.cpp:37-41)
    plan = C.c_void_p()
    pd = pool.desc()
    rc = _capi.lib().ep_plan_create(cuda_handle.ptr, C.byref(pd), 8, 1, table.batch,
                                    indptr.ctypes.data, segs_bad.ctypes.data, pt.ctypes.data,
                                    table.q_pos.ctypes.data, 0, C.byref(plan))
    assert rc == _capi.EP_EINVAL and b"segment starts" in _capi.lib().ep_last_error()
    pt_bad = pt.copy()
    pt_bad[0] = pool.num_pages + 5
    rc = _capi.lib().ep_plan_create(cuda_handle.ptr, C.byref(pd), 8, 1, table.batch,
                                    indptr.ctypes.data, segs.ctypes.data, pt_bad.ctypes.data,
                                    table.q_pos.ctypes.data, 0, C.byref(plan))
    assert rc == _capi.EP_EINVAL
    # rows = 4 * 17 = 68 > 64: past K3, K1 takes it in query chunks
    rc = _capi.lib().ep_plan_create(cuda_handle.ptr, C.byref(pd), 8, 17, table.batch,
                                    indptr.ctypes.data, segs.ctypes.data, pt.ctypes.data,
                                    table.q_pos.ctypes.data, 0, C.byref(plan))
    assert rc == _capi.EP_OK
    _capi.lib().ep_plan_destroy(plan)
    pd_wide = pool.desc()
    pd_wide.d_head = 512   # the only shape without a kernel: d_head > 256
    rc = _capi.lib().ep_plan_create(cuda_handle.ptr, C.byref(pd_wide), 8, 1, table.batch,
                                    indptr.ctypes.data, segs.ctypes.data, pt.ctypes.data,
                                    table.q_pos.ctypes.data, 0, C.byref(plan))
    assert rc == _capi.EP_EUNSUPPORTED


# Every head shape the reference accepts (any n_heads, any d_head,
# attention.cpp:80-114, model.hpp:15-25) runs on the device: K1 with its row
# stride padded to a power of two (group 3 / 5 / 6, n_q*group = 5), K1 over
# query chunks of 8 / group tokens when a unit has more than 8 rows and K3
# does not apply (fp32 verify: 20 rows; config 1's k = 8 verify on MHA d 64:
# 9 rows), and the generic kernel for the rest (d_head 96 / 256 / 80, group
# 16 on fp32). Ragged segments, a shared cloud prompt, a request of only its
# own query tokens.
@pytest.mark.parametrize("kv,Hq,Hkv,d,n_q", [
    (O.DT_BF16, 12, 4, 128, 1),   # G 3 -> R 4
    (O.DT_F32, 10, 2, 64, 1),     # G 5 -> R 8
    (O.DT_BF16, 24, 4, 128, 1),   # G 6 -> R 8
    (O.DT_F32, 4, 4, 64, 5),      # MHA verify k = 4: 5 rows -> R 8
    (O.DT_F32, 4, 4, 64, 9),      # MHA verify k = 8: 9 rows -> chunks of 8 + 1 tokens
    (O.DT_F32, 16, 4, 128, 5),    # fp32 GQA verify: 20 rows -> chunks of 2 tokens
    (O.DT_BF16, 12, 4, 64, 7),    # bf16 d 64, 21 rows -> chunks of 2 tokens (K3 needs d 128)
    (O.DT_BF16, 8, 2, 96, 1),     # generic: d 96
    (O.DT_BF16, 4, 2, 256, 3),    # generic: d 256, multi-row
    (O.DT_F32, 32, 2, 64, 1),     # generic: group 16
    (O.DT_F32, 6, 3, 80, 2),      # generic: d 80
])
def test_any_head_shape(cuda_handle, kv, Hq, Hkv, d, n_q):
    import torch
    reqs = [[(SC.CLOUD, 300, "c"), (SC.EDGE, 37, None), (SC.GEN, 9, None)],
            [(SC.CLOUD, 300, "c"), (SC.EDGE, 130, None), (SC.GEN, 12, None)],
            [(SC.EDGE, 64, None)],
            [(SC.GEN, n_q, None)],
            [(SC.CLOUD, 70, None), (SC.EDGE, 1, None), (SC.GEN, n_q, None)]]
    sb = SC.make_case(kv, Hq, Hkv, d, reqs, n_q=n_q, seed=17 + d + Hq)
    _, _, attn, q = to_device(sb, cuda_handle)
    want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4)
    for o_dtype in (torch.float32, q.dtype):
        o, lse = attn(q, o_dtype=o_dtype)
        err = _check(o, lse, want_o, want_l, sb.kv_dtype)
        print(Hq, Hkv, d, n_q, o_dtype, err)


def test_cache_object_per_token_growth(cuda_handle):
    """Per-token growth through the C-ABI splice state (ep_cache): every step
    ep_cache_append_generated gives each request's new token a page slot
    (fresh pages at page boundaries), ep_kv_append writes the K/V rows there,
    ep_plan_update_cache re-plans from the cache (no host arrays), and the
    attention matches the oracle on the same pages; truncation (rejected
    drafts) shrinks the plan again."""
    import ctypes as C
    import torch
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.splice import SpliceCache, SplicedAttention
    sb = SC.make_case(O.DT_BF16, 8, 2, 128, [[(SC.CLOUD, 190, None), (SC.EDGE, 40, None)],
                                              [(SC.EDGE, 63, None)]], seed=19, spare_pages=8)
    pool, table, _, q = to_device(sb, cuda_handle)
    cache = SpliceCache(1, table.batch, 64)
    for b in range(table.batch):
        for s in table.requests[b]:
            cache.append(b, s.origin, s.pos_offset, s.length, s.pages)
    used = set(sb.page_table.tolist())
    free = [p for p in range(pool.num_pages) if p not in used]
    attn = SplicedAttention.from_cache(pool, cache, 8, 1, handle=cuda_handle)
    host_k, host_v = sb.k_pages.copy(), sb.v_pages.copy()
    lib = _capi.lib()
    pd = pool.desc()
    for step in range(70):
        newp = np.array([[free[0]], [free[1]]], np.int32)
        dp, ds, nused = cache.append_generated([1, 1], newp)
        taken = {int(newp[b, 0]) for b in range(2) if nused[b]}
        free = [p for p in free if p not in taken]
        kv = O.fill_uniform(O.DT_BF16, 2 * 2 * 2 * 128, 3000 + step).reshape(2, 2, 2, 128)  # [k|v][b][h][d]
        kd = torch_from_raw(np.ascontiguousarray(kv[0]), O.DT_BF16)
        vd = torch_from_raw(np.ascontiguousarray(kv[1]), O.DT_BF16)
        dpg = torch.from_numpy(dp.astype(np.int32)).cuda()
        dsl = torch.from_numpy(ds.astype(np.int32)).cuda()
        _capi.check(lib.ep_kv_append(cuda_handle.ptr, C.byref(pd), 2, dpg.data_ptr(), dsl.data_ptr(),
                                     kd.data_ptr(), vd.data_ptr(), None), "ep_kv_append")
        for b in range(2):
            host_k[dp[b], :, ds[b]] = kv[0, b]
            host_v[dp[b], :, ds[b]] = kv[1, b]
        if step == 40:   # a rejected draft of 3 tokens on request 1
            rel = cache.truncate(1, 3)
            free = list(rel) + free
        attn.update_from_cache()
        o, lse = attn(q)
        if step % 23 == 0 or step in (40, 69):
            indptr, segs, pt = cache.arrays(0)
            qp = np.array([cache.end_position(b) - 1 for b in range(2)], np.int64)
            hb = O.HostSpliceBatch(sb.kv_dtype, 2, 8, 128, 64, host_k, host_v, indptr, segs, pt,
                                   qp, sb.q_dtype, sb.q, 1)
            want_o, want_l = O.spliced_attention(hb, n_threads=4)
            _check(o, lse, want_o, want_l, sb.kv_dtype)
    assert cache.check_consistent() == ""


def test_cache_two_plans_alternating(cuda_handle):
    """The serving pattern of bench.py's e2e: two plans of one ep_cache used on
    alternate steps, so each plan follows the cache two tokens at a time
    (in-page growth through the device patch, a re-plan when a page fills,
    a truncation in between); every checked step matches the oracle on the
    cache's own pages."""
    import ctypes as C
    import torch
    from paper_2504_11729_b200 import _capi
    from paper_2504_11729_b200.splice import SpliceCache, SplicedAttention
    sb = SC.make_case(O.DT_BF16, 8, 2, 128, [[(SC.CLOUD, 130, None), (SC.EDGE, 61, None)],
                                              [(SC.EDGE, 7, None)]], seed=29, spare_pages=8)
    pool, table, _, q = to_device(sb, cuda_handle)
    cache = SpliceCache(1, table.batch, 64)
    for b in range(table.batch):
        for s in table.requests[b]:
            cache.append(b, s.origin, s.pos_offset, s.length, s.pages)
    used = set(sb.page_table.tolist())
    free = [p for p in range(pool.num_pages) if p not in used]
    plans = [SplicedAttention.from_cache(pool, cache, 8, 1, handle=cuda_handle) for _ in range(2)]
    host_k, host_v = sb.k_pages.copy(), sb.v_pages.copy()
    lib = _capi.lib()
    pd = pool.desc()
    for step in range(75):
        newp = np.array([[free[0]], [free[1]]], np.int32)
        dp, ds, nused = cache.append_generated([1, 1], newp)
        taken = {int(newp[b, 0]) for b in range(2) if nused[b]}
        free = [p for p in free if p not in taken]
        kv = O.fill_uniform(O.DT_BF16, 2 * 2 * 2 * 128, 5000 + step).reshape(2, 2, 2, 128)
        kd = torch_from_raw(np.ascontiguousarray(kv[0]), O.DT_BF16)
        vd = torch_from_raw(np.ascontiguousarray(kv[1]), O.DT_BF16)
        dpg = torch.from_numpy(dp.astype(np.int32)).cuda()
        dsl = torch.from_numpy(ds.astype(np.int32)).cuda()
        _capi.check(lib.ep_kv_append(cuda_handle.ptr, C.byref(pd), 2, dpg.data_ptr(), dsl.data_ptr(),
                                     kd.data_ptr(), vd.data_ptr(), None), "ep_kv_append")
        for b in range(2):
            host_k[dp[b], :, ds[b]] = kv[0, b]
            host_v[dp[b], :, ds[b]] = kv[1, b]
        if step == 33:   # a rejected draft of 2 tokens on request 0
            rel = cache.truncate(0, 2)
            free = list(rel) + free
        attn = plans[step & 1]
        attn.update_from_cache()
        o, lse = attn(q)
        if step % 11 == 0 or step in (33, 34, 74):
            indptr, segs, pt = cache.arrays(0)
            qp = np.array([cache.end_position(b) - 1 for b in range(2)], np.int64)
            hb = O.HostSpliceBatch(sb.kv_dtype, 2, 8, 128, 64, host_k, host_v, indptr, segs, pt,
                                   qp, sb.q_dtype, sb.q, 1)
            want_o, want_l = O.spliced_attention(hb, n_threads=4)
            _check(o, lse, want_o, want_l, sb.kv_dtype)
    assert cache.check_consistent() == ""


@pytest.mark.parametrize("P", [128, 192])
@pytest.mark.parametrize("kind", ["decode", "verify", "shared"])
def test_page_sizes_beyond_64(cuda_handle, P, kind):
    """Pages of 128 and 192 tokens (any multiple of 64 is legal, ep_plan
    splits them into 64-token pipeline blocks): K1 decode, K3 verify rows
    (n_q = 5) and the config-5 cascade (a cloud segment shared by every
    request), with ragged segment tails inside the larger pages; vs the oracle."""
    Hq, Hkv, d = 32, 8, 128
    n_q = 5 if kind == "verify" else 1
    r = O.SplitMix64(P + len(kind))
    if kind == "shared":
        reqs = [[(SC.CLOUD, 1000, "cloud"), (SC.EDGE, 40 + r.next_u64() % 300, None), (SC.GEN, 1, None)]
                for _ in range(40)]
    else:
        reqs = [[(SC.CLOUD, 300 + r.next_u64() % 700, None), (SC.EDGE, 1 + r.next_u64() % 250, None),
                 (SC.GEN, n_q, None)] for _ in range(6)]
    sb = SC.make_case(O.DT_BF16, Hq, Hkv, d, reqs, n_q=n_q, page_tokens=P, seed=70 + P)
    _, _, attn, q = to_device(sb, cuda_handle)
    o, lse = attn(q)
    want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4)
    _check(o, lse, want_o, want_l, sb.kv_dtype)
