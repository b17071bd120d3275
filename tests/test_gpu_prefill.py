"""GPU parity of the prefill tiles (ep_plan_create_prefill -> K3 on tcgen05):
the last n_new tokens of each request attend causally to every key up to
their own position — the cloud-prompt prefill (n_new = the whole prompt,
cloud.cpp:160-172 -> transformer_layer) and the edge prefill against a shared
cloud segment (edge.cpp:148-164) — against the fp64 oracle's spliced
attention with n_q = n_new causal rows (model.cpp:161-182 semantics) on
identical bf16 inputs."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import splice_cases as SC
from tests.cases import rel_err
from tests.gpu_util import to_device, torch_from_raw

pytestmark = pytest.mark.gpu

C, E = SC.CLOUD, SC.EDGE
CASES = {
    # G = 4 -> 32 query tokens per tile; a 300-token prompt = 10 ragged chunks
    "cloud_prefill_gqa4": dict(n_q_heads=32, n_kv_heads=8,
                               requests=[[(C, 300, None)], [(C, 77, None)]], n_new=[300, 77]),
    # edge prefill over one shared cloud prompt, ragged edges, a request with
    # no new tokens and a pure edge request
    "edge_prefill_shared_cloud": dict(n_q_heads=8, n_kv_heads=2,
                                      requests=[[(C, 256, "c"), (E, 70, None)],
                                                [(C, 256, "c"), (E, 129, None)],
                                                [(C, 256, "c"), (E, 1, None)],
                                                [(C, 256, "c"), (E, 5, None)],
                                                [(E, 40, None)]],
                                      n_new=[70, 129, 1, 0, 40]),
    # MHA (G = 1 -> 128 tokens per tile) and G = 8 (16 tokens per tile)
    "mha_prefill": dict(n_q_heads=4, n_kv_heads=4, requests=[[(C, 200, None), (E, 90, None)]],
                        n_new=[290]),
    "gqa8_edge_prefill": dict(n_q_heads=16, n_kv_heads=2, requests=[[(C, 130, None), (E, 33, None)]],
                              n_new=[33]),
}


def _oracle(sb, q, n_new):
    """Per request: n_q = n_new causal rows at the end of its cache."""
    outs, lses = [], []
    off = 0
    for b, nb in enumerate(n_new):
        if nb == 0:
            continue
        i0, i1 = int(sb.seg_indptr[b]), int(sb.seg_indptr[b + 1])
        segs = sb.segs[i0:i1].copy()
        end = int(segs[-1]["pos_offset"] + segs[-1]["len"])
        one = O.HostSpliceBatch(
            kv_dtype=sb.kv_dtype, n_kv_heads=sb.n_kv_heads, n_q_heads=sb.n_q_heads,
            d_head=sb.d_head, page_tokens=sb.page_tokens, k_pages=sb.k_pages, v_pages=sb.v_pages,
            seg_indptr=np.array([0, i1 - i0], dtype=np.int64), segs=segs,
            page_table=sb.page_table, q_pos=np.array([end - nb], dtype=np.int64),
            q_dtype=sb.q_dtype, q=np.ascontiguousarray(q[off:off + nb][None]), n_q=nb)
        o, l = O.spliced_attention(one, n_threads=8)
        outs.append(o[0])
        lses.append(l[0])
        off += nb
    return np.concatenate(outs), np.concatenate(lses)


@pytest.mark.parametrize("page_tokens", [64, 192])
@pytest.mark.parametrize("name", sorted(CASES))
def test_prefill_matches_oracle(cuda_handle, name, page_tokens):
    import torch
    from paper_2504_11729_b200.splice import SplicedPrefill
    cfg = CASES[name]
    sb = SC.make_case(O.DT_BF16, cfg["n_q_heads"], cfg["n_kv_heads"], 128, cfg["requests"],
                      n_q=1, page_tokens=page_tokens, seed=11)
    T = sum(cfg["n_new"])
    q_raw = O.fill_uniform(O.DT_BF16, T * cfg["n_q_heads"] * 128, 11_009).reshape(
        T, cfg["n_q_heads"], 128)
    want_o, want_l = _oracle(sb, q_raw, cfg["n_new"])
    pool, table, _, _ = to_device(sb, cuda_handle)
    pre = SplicedPrefill(pool, table, cfg["n_q_heads"], cfg["n_new"], handle=cuda_handle)
    q = torch_from_raw(np.ascontiguousarray(q_raw), O.DT_BF16)
    o16, l16 = pre(q)                            # bf16 out: single bf16 P
    o32, l32 = pre(q, o_dtype=torch.float32)     # fp32 out: P as bf16 hi + lo
    torch.cuda.synchronize()
    e16 = rel_err(o16.float().cpu().numpy(), want_o)
    e32 = rel_err(o32.cpu().numpy(), want_o)
    le = max(np.max(np.abs(l16.cpu().numpy() - want_l)), np.max(np.abs(l32.cpu().numpy() - want_l)))
    print(f"{name}: tokens {T}, plan {pre.info()}, rel err bf16 {e16:.2e} fp32 {e32:.2e}, lse {le:.2e}")
    assert e16 <= 2e-2 and e32 <= 1e-3 and le <= 1e-4


def test_prefill_equals_decode_rows(cuda_handle):
    """The last prefill row of a request equals a decode of that token over the
    same table (split == monolithic, acceptance criterion 2 in spirit)."""
    import torch
    from paper_2504_11729_b200.splice import SplicedPrefill
    sb = SC.make_case(O.DT_BF16, 32, 8, 128, [[(C, 190, None), (E, 66, None)]], n_q=1, seed=5)
    pool, table, attn, q1 = to_device(sb, cuda_handle)  # decode row at position end-1
    n_new = 66
    q_raw = O.fill_uniform(O.DT_BF16, n_new * 32 * 128, 77).reshape(n_new, 32, 128)
    q_raw[-1] = sb.q[0, 0]
    pre = SplicedPrefill(pool, table, 32, [n_new], handle=cuda_handle)
    o, _ = pre(torch_from_raw(np.ascontiguousarray(q_raw), O.DT_BF16), o_dtype=torch.float32)
    od, _ = attn(q1, o_dtype=torch.float32)
    torch.cuda.synchronize()
    err = (o[-1] - od[0, 0]).abs().max().item()
    assert err < 1e-4, err


def test_prefill_rejects_bad_n_new(cuda_handle):
    from paper_2504_11729_b200._capi import InvalidArgument
    from paper_2504_11729_b200.splice import SplicedPrefill
    sb = SC.make_case(O.DT_BF16, 8, 2, 128, [[(C, 64, None)]], n_q=1, seed=3)
    pool, table, _, _ = to_device(sb, cuda_handle)
    with pytest.raises(InvalidArgument):
        SplicedPrefill(pool, table, 8, [65], handle=cuda_handle)


K1_CASES = {
    # (kv dtype, q heads, kv heads, d_head): K3 has no instance for these, so
    # prefill runs as K1 chunks of 8/G query tokens; ragged n_new leaves a
    # short last chunk (valid-rows path)
    "f32_mha_d64": (O.DT_F32, 4, 4, 64),
    "bf16_gqa2_d64": (O.DT_BF16, 8, 4, 64),
    "f32_gqa4_d128": (O.DT_F32, 16, 4, 128),
    "f32_gqa8_d64": (O.DT_F32, 16, 2, 64),
}


@pytest.mark.parametrize("name", sorted(K1_CASES))
def test_prefill_cuda_core_chunks(cuda_handle, name):
    import torch
    from paper_2504_11729_b200.splice import SplicedPrefill
    dt, hq, hkv, d = K1_CASES[name]
    reqs = [[(C, 150, None), (E, 37, None)], [(C, 64, None)], [(C, 21, None), (E, 9, None)]]
    n_new = [37, 64, 13]
    sb = SC.make_case(dt, hq, hkv, d, reqs, n_q=1, seed=21)
    T = sum(n_new)
    q_raw = O.fill_uniform(dt, T * hq * d, 21_013).reshape(T, hq, d)
    want_o, want_l = _oracle(sb, q_raw, n_new)
    pool, table, _, _ = to_device(sb, cuda_handle)
    pre = SplicedPrefill(pool, table, hq, n_new, handle=cuda_handle)
    q = torch_from_raw(np.ascontiguousarray(q_raw), dt)
    o, l = pre(q, o_dtype=torch.float32)
    torch.cuda.synchronize()
    err = rel_err(o.cpu().numpy(), want_o)
    le = float(np.max(np.abs(l.cpu().numpy() - want_l)))
    print(f"{name}: plan {pre.info()}, rel err {err:.2e}, lse {le:.2e}")
    assert err <= (1e-3 if dt == O.DT_F32 else 2e-2) and le <= 1e-4
