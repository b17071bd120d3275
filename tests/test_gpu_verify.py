"""GPU parity of K3 (tcgen05 multi-row verify attention): n_q = k+1 causal
rows per request (k = 4, 8) with GQA group 4 -> 20 / 36 rows per kv-head,
against the fp64 oracle on identical bf16 inputs (2e-2 relative, north_star)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests import splice_cases as SC
from tests.gpu_util import to_device
from tests.test_gpu_decode import _check

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("k", [4, 8])
def test_config3_shape_subset(cuda_handle, k):
    """BASELINE config 3 structure (cloud 14336 + edge 1536 + generated 512
    = 16384 keys, drafts causal at the end) at batch 4, checked on 24 units."""
    reqs = [[(SC.CLOUD, 14336, None), (SC.EDGE, 1536, None), (SC.GEN, 512, None)]] * 4
    sb = SC.make_case(O.DT_BF16, 32, 8, 128, reqs, n_q=k + 1, seed=31)
    _, _, attn, q = to_device(sb, cuda_handle)
    o, lse = attn(q)
    units = np.random.default_rng(k).choice(4 * 32, 24, replace=False)
    want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4, units=units)
    print(f"cfg3 k={k} rel err:", _check(o, lse, want_o, want_l, sb.kv_dtype, units, 32))


def test_tc_path_on_decode_rows_matches_golden():
    """EP_FORCE_TC=1 routes a 4-row decode through the tcgen05 kernel: it must
    reproduce the reference goldens like the CUDA-core kernel does."""
    code = (
        "import numpy as np, os, sys; sys.path.insert(0, %r)\n"
        "from tests import splice_cases as SC\n"
        "from tests.gpu_util import to_device\n"
        "from tests.cases import rel_err\n"
        "g = np.load(os.path.join(%r, 'tests/golden/splice_golden.npz'))\n"
        "for name in ['gqa4_bf16_decode', 'gqa2_f32_d128_nq2']:\n"
        "    sb = SC.small_case(name)\n"
        "    if sb.kv_dtype != 1: continue\n"
        "    _, _, attn, q = to_device(sb)\n"
        "    import torch\n"
        "    o, l = attn(q, o_dtype=torch.float32)\n"
        "    e = rel_err(o.cpu().numpy(), g[name + '/out'])\n"
        "    assert e <= 2e-2, (name, e)\n"
        "    print(name, e)\n" % (ROOT, ROOT))
    env = dict(os.environ, EP_FORCE_TC="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    print(r.stdout)


@pytest.mark.parametrize("k", [4, 8])
def test_verify_greedy_accept_bit_exact(cuda_handle, k):
    """Full verify step (K3 attention + K4 score/argmax/accept) against the
    fp64 oracle (spliced attention -> LN -> @W_score -> argmax -> accept rule).
    Drafts follow the oracle's own targets with a seeded forced mismatch per
    request, so every acceptance length 0..k occurs. Rows whose oracle top-2
    logit gap is below 8x the measured max |logit error| are margin-guarded
    (SURVEY §8a); all other target ids and every accepted count must be
    bit-exact."""
    import torch
    from paper_2504_11729_b200.verify import VerifyGreedy
    from tests.gpu_util import torch_from_raw
    B, Hq, Hkv, d, V = 8, 32, 8, 128, 4096
    n_q = k + 1
    reqs = [[(SC.CLOUD, 1024 + 64 * b, None), (SC.EDGE, 200 + b, None), (SC.GEN, 64, None)]
            for b in range(B)]
    sb = SC.make_case(O.DT_BF16, Hq, Hkv, d, reqs, n_q=n_q, seed=33 + k)
    _, _, attn, q = to_device(sb, cuda_handle)
    o, _ = attn(q, o_dtype=torch.float32)  # [B][n_q][Hq][d], scored as bf16 hi+lo

    W = O.fill_uniform(O.DT_BF16, Hq * d * V, 33).reshape(Hq * d, V)   # [width][vocab]
    w_t = torch_from_raw(np.ascontiguousarray(W.T), O.DT_BF16)         # [vocab][width]
    ver = VerifyGreedy(w_t, handle=cuda_handle)

    want_o, _ = O.spliced_attention(sb, n_threads=os.cpu_count() or 4)
    attn64 = want_o.reshape(B, n_q, Hq * d)
    W64 = O.bf16_to_f64(W)
    g_ref, _, gap = O.verify_greedy(attn64, W64, np.zeros((B, k), np.int32))
    drafts = g_ref[:, :k].copy()
    for b in range(B):
        a = b % (k + 1)              # force acceptance length a
        if a < k:
            drafts[b, a] = (g_ref[b, a] + 1) % V
            drafts[b, a + 1:] = (g_ref[b, a + 1:k] + 7) % V
    g_ref, nacc_ref, gap = O.verify_greedy(attn64, W64, drafts)

    tgt, nacc, logits = ver(o, torch.from_numpy(drafts).cuda(), logits=True)
    torch.cuda.synchronize()
    tgt, nacc = tgt.cpu().numpy(), nacc.cpu().numpy()
    # oracle logits for the margin guard
    ref_logits = np.zeros((B, n_q, V))
    for b in range(B):
        for j in range(n_q):
            x = attn64[b, j]
            xn = (x - x.mean()) / np.sqrt(x.var() + 1e-5)
            ref_logits[b, j] = xn @ W64
    err = float(np.max(np.abs(logits.cpu().numpy() - ref_logits)))
    guarded = gap < 8 * err
    print(f"k={k}: max |logit err| {err:.3e}, guarded rows {int(guarded.sum())}/{B * n_q}")
    assert guarded.mean() < 0.1
    ok_rows = ~guarded
    assert np.array_equal(tgt[ok_rows], g_ref[ok_rows])
    # accepted counts: bit-exact wherever no guarded row decides them
    for b in range(B):
        if not guarded[b, :min(nacc_ref[b] + 1, k)].any():
            assert nacc[b] == nacc_ref[b], (b, nacc[b], nacc_ref[b])
    assert sorted(set(nacc_ref.tolist())) == list(range(min(B, k + 1)))


def _oracle_argmax(x, W64):
    """argmax_token(LN(x) @ W) in fp64, first index of the maximum."""
    xn = (x - x.mean(axis=-1, keepdims=True)) / np.sqrt(x.var(axis=-1, keepdims=True) + 1e-5)
    return np.argmax(xn @ W64, axis=-1)


@pytest.mark.parametrize("case,B,n_q", [
    ("tie_pair", 4, 3), ("all_equal", 4, 3), ("random", 4, 3), ("zero_max", 4, 3),
    ("random", 43, 3), ("random", 64, 5), ("random", 64, 9), ("tie_pair", 64, 9),
    ("zero_max", 64, 5)])
def test_score_refinement_edge_cases(cuda_handle, case, B, n_q):
    """K4's hi-only GEMM + exact refinement against the fp64 argmax on crafted
    rows: exact ties between two vocab entries (argmax_token keeps the lower
    id), a W whose columns are all identical (every logit ties: the candidate
    overflow path must still return id 0), a maximum of exactly zero shared
    by two all-zero vocab columns, and random rows — at 12 rows (one M tile)
    and at 129 / 320 / 576 rows (2 / 3 / 5 M tiles, partial last tile)."""
    import torch
    from paper_2504_11729_b200.verify import VerifyGreedy
    from tests.gpu_util import torch_from_raw
    width, V = 4096, 4096
    rng = np.random.default_rng({"tie_pair": 1, "all_equal": 2, "random": 3, "zero_max": 4}[case] + B)
    W = O.fill_uniform(O.DT_BF16, width * V, 77).reshape(width, V)  # raw bf16 [width][vocab]
    x = rng.uniform(-1.0, 1.0, size=(B, n_q, width)).astype(np.float32) * 0.01
    if case == "tie_pair":
        # columns 17 and 1000: the same bf16 vector, aligned with the rows'
        # shared direction u, so they tie for the maximum in every row
        u = rng.uniform(-1.0, 1.0, size=width).astype(np.float32)
        x = x + 0.05 * u
        col = O.f64_to_bf16(0.5 * u.astype(np.float64))
        W[:, 17] = col
        W[:, 1000] = col
    elif case == "all_equal":
        W[:, :] = W[:, :1]
    elif case == "zero_max":
        # every column anti-aligned with the rows' shared direction (logits
        # < 0) except columns 40 and 41, which are zero: the maximum is an
        # exact 0 tie and argmax_token keeps id 40
        u = rng.uniform(-1.0, 1.0, size=width).astype(np.float32)
        x = x + 0.05 * u
        scale = rng.uniform(0.2, 1.0, size=V)
        wf = (-np.outer(u.astype(np.float64) - u.mean(), scale)).astype(np.float32).view(np.uint32)
        W[:, :] = ((wf + 0x7FFF + ((wf >> 16) & 1)) >> 16).astype(np.uint16)   # RNE to bf16
        W[:, 40] = 0
        W[:, 41] = 0
    w_t = torch_from_raw(np.ascontiguousarray(W.T), O.DT_BF16)
    ver = VerifyGreedy(w_t, handle=cuda_handle)
    xt = torch.from_numpy(x).cuda().view(B, n_q, 32, 128)
    drafts = torch.zeros((B, n_q - 1), dtype=torch.int32, device="cuda")
    tgt, _, _ = ver(xt, drafts)
    want = _oracle_argmax(x.astype(np.float64), O.bf16_to_f64(W))
    got = tgt.cpu().numpy()
    if case == "tie_pair":
        assert (want == 17).all()
    if case == "all_equal":
        assert (want == 0).all()
    if case == "zero_max":
        assert (want == 40).all()
    assert np.array_equal(got, want), (got, want)


def _cfg3_setup(k, h):
    """BASELINE config 3 at full size, built like the bench (tools/verify_bench.py):
    B = 64 requests, private KV, cloud 14336 + edge 1536 + generated 512 =
    16384 keys, Hq 32 / Hkv 8 / d 128 bf16, W_score 4096 x 4096 bf16; pool, q
    and W drawn on the device by ep_fill_uniform (the SplitMix64 stream of
    oracle.fill_uniform, so the host can regenerate any slice)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import verify_bench as VB
    return VB, VB.setup(k, h)


@pytest.mark.parametrize("k", [4, 8])
def test_config3_verify_production_path(cuda_handle, k):
    """The path the bench times (K3 attention -> K4 hi-only GEMM + candidate
    refinement + fused accept, logits=None) at config 3's full shape: 64 x
    (k+1) = 320 / 576 score rows, i.e. 3 / 5 M tiles of 128 with a partial
    last tile. Attention is checked against the fp64 oracle on sampled
    requests (all their units); every target id against argmax_token(LN(x) @
    W) in fp64 over the GPU's own fp32 attention rows (model.cpp:238-255),
    outside the margin guard; every accepted count against the acceptance rule
    on the oracle ids (drafts force every acceptance length 0..k)."""
    import torch
    from tests.cases import rel_err
    VB, st = _cfg3_setup(k, cuda_handle)
    B, HQ, HKV, D, V, P = VB.B, VB.HQ, VB.HKV, VB.D, VB.V, VB.P
    n_q = k + 1
    attn, q, ver, o, lse = st["attn"], st["q"], st["ver"], st["o"], st["lse"]
    attn(q, o=o, lse=lse)
    torch.cuda.synchronize()
    x = o.cpu().numpy().astype(np.float64).reshape(B, n_q, HQ * D)

    # (1) attention of sampled requests vs the oracle on the same pages
    ppr = VB.S // P
    pool = st["pool"]
    for b in (0, 37, 63):
        pages = np.arange(b * ppr, (b + 1) * ppr)
        kp = pool.k[torch.from_numpy(pages).cuda()].view(torch.int16).cpu().numpy().view(np.uint16)
        vp = pool.v[torch.from_numpy(pages).cuda()].view(torch.int16).cpu().numpy().view(np.uint16)
        segs = np.array([(0, VB.CLOUD, 0, 0), (1, VB.EDGE, VB.CLOUD, VB.CLOUD // P),
                         (2, VB.GEN, VB.CLOUD + VB.EDGE, (VB.CLOUD + VB.EDGE) // P)],
                        dtype=O.SEGMENT_DTYPE)
        qb = q[b:b + 1].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        sb = O.HostSpliceBatch(kv_dtype=O.DT_BF16, n_kv_heads=HKV, n_q_heads=HQ, d_head=D,
                               page_tokens=P, k_pages=np.ascontiguousarray(kp),
                               v_pages=np.ascontiguousarray(vp),
                               seg_indptr=np.array([0, 3], np.int64), segs=segs,
                               page_table=np.arange(ppr, dtype=np.int32),
                               q_pos=np.array([VB.S - n_q], np.int64), q_dtype=O.DT_BF16,
                               q=np.ascontiguousarray(qb), n_q=n_q)
        want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4)
        e_o = rel_err(o[b:b + 1].cpu().numpy(), want_o)
        e_l = rel_err(lse[b:b + 1].cpu().numpy(), want_l)
        print(f"cfg3 k={k} request {b}: attention rel err {e_o:.2e}, lse {e_l:.2e}")
        assert e_o <= 1e-3 and e_l <= 1e-4   # fp32 output of bf16 KV: far inside 2e-2

    # (2) target ids over all B * n_q rows, fp64 oracle on the GPU's rows
    W = O.fill_uniform(O.DT_BF16, V * HQ * D, 33).reshape(V, HQ * D)   # W^T as on the device
    W64 = np.ascontiguousarray(O.bf16_to_f64(W).T)                     # [width][vocab]
    g_ref, _, gap = O.verify_greedy(x, W64, np.zeros((B, k), np.int32))
    drafts = g_ref[:, :k].copy()
    for b in range(B):
        a = b % (k + 1)
        if a < k:
            drafts[b, a] = (g_ref[b, a] + 1) % V
            drafts[b, a + 1:] = (g_ref[b, a + 1:k] + 7) % V
    g_ref, nacc_ref, gap = O.verify_greedy(x, W64, drafts)
    dr = torch.from_numpy(drafts.astype(np.int32)).cuda()
    tgt, nacc, _ = ver(o, dr)                      # the timed path: logits=None
    torch.cuda.synchronize()
    tgt, nacc = tgt.cpu().numpy(), nacc.cpu().numpy()
    # margin guard from the exact-logits path (a separate call)
    _, _, lg = ver(o, dr, logits=True)
    xn = (x - x.mean(-1, keepdims=True)) / np.sqrt(x.var(-1, keepdims=True) + 1e-5)
    err = float(np.max(np.abs(lg.cpu().numpy().astype(np.float64) - xn @ W64)))
    guarded = gap < 8 * err
    print(f"cfg3 k={k}: {B * n_q} rows, max |logit err| {err:.2e}, guarded {int(guarded.sum())}")
    assert guarded.mean() < 0.1
    assert np.array_equal(tgt[~guarded], g_ref[~guarded])
    checked = 0
    for b in range(B):
        if not guarded[b, :min(nacc_ref[b] + 1, k)].any():
            assert nacc[b] == nacc_ref[b], (b, nacc[b], nacc_ref[b])
            checked += 1
    assert checked >= B - 4
    assert sorted(set(nacc_ref.tolist())) == list(range(k + 1))


@pytest.mark.parametrize("V", [16384, 40960])
def test_score_large_vocab_candidate_path(cuda_handle, V):
    """Vocabularies past 64 (and past 256) tiles of 128: the refinement keeps
    using the candidate list (sized by the gathered count, tiles read in
    strides of the block) instead of scoring every entry; ids equal the fp64
    argmax_token(LN(x) @ W) (model.cpp:238-255)."""
    import torch
    from paper_2504_11729_b200.verify import VerifyGreedy
    from tests.gpu_util import torch_from_raw
    B, n_q, width = 4, 3, 4096
    rng = np.random.default_rng(V)
    W = O.fill_uniform(O.DT_BF16, width * V, 91).reshape(width, V)
    x = rng.uniform(-1.0, 1.0, size=(B, n_q, width)).astype(np.float32)
    ver = VerifyGreedy(torch_from_raw(np.ascontiguousarray(W.T), O.DT_BF16), handle=cuda_handle)
    tgt, _, _ = ver(torch.from_numpy(x).cuda().view(B, n_q, 32, 128),
                    torch.zeros((B, n_q - 1), dtype=torch.int32, device="cuda"))
    want = _oracle_argmax(x.astype(np.float64), O.bf16_to_f64(W))
    assert np.array_equal(tgt.cpu().numpy(), want)


@pytest.mark.parametrize("B,n_q,width,V", [
    (64, 9, 1024, 4096),   # 5 x 16 tiles of 16 k-blocks over 148 CTAs: tiles span 2-3 CTAs (1-2 partials)
    (7, 3, 2048, 1024),    # 1 M tile x 4 vocab tiles x 32 k-blocks: 128 k-blocks < 148 CTAs (one per CTA)
    (1, 1, 64, 256),       # a single k-block: one CTA, no partials
    (43, 5, 4096, 8192),   # 2 M tiles x 32 vocab tiles: partial last M tile, ~28 k-blocks per CTA
])
def test_score_streamk_partition_shapes(cuda_handle, B, n_q, width, V):
    """K4's stream-K GEMM (score_argmax_streamk_kernel): ranges of the flattened
    (tile, k-block) space that start / end inside tiles, tiles covered by 1-3
    CTAs (owner + published partial tiles), fewer k-blocks than SMs, a single
    k-block; target ids equal the fp64 argmax_token(LN(x) @ W)
    (model.cpp:238-255)."""
    import torch
    from paper_2504_11729_b200.verify import VerifyGreedy
    from tests.gpu_util import torch_from_raw
    rng = np.random.default_rng(B * 7919 + width + V)
    W = O.fill_uniform(O.DT_BF16, width * V, 1234).reshape(width, V)
    x = rng.uniform(-1.0, 1.0, size=(B, n_q, width)).astype(np.float32)
    ver = VerifyGreedy(torch_from_raw(np.ascontiguousarray(W.T), O.DT_BF16), handle=cuda_handle)
    drafts = torch.zeros((B, max(n_q - 1, 0)), dtype=torch.int32, device="cuda")
    tgt, _, _ = ver(torch.from_numpy(x).cuda().view(B, n_q, width), drafts)
    want = _oracle_argmax(x.astype(np.float64), O.bf16_to_f64(W))
    assert np.array_equal(tgt.cpu().numpy(), want)
    # a second launch on the same verifier: the partial-tile flags were
    # cleared by their consumers, so the owners wait for fresh partials
    x2 = rng.uniform(-1.0, 1.0, size=(B, n_q, width)).astype(np.float32)
    tgt2, _, _ = ver(torch.from_numpy(x2).cuda().view(B, n_q, width), drafts)
    assert np.array_equal(tgt2.cpu().numpy(), _oracle_argmax(x2.astype(np.float64), O.bf16_to_f64(W)))


@pytest.mark.parametrize("B,n_q", [(4, 3), (64, 9)])
def test_score_bf16_rows_folded_ln(cuda_handle, B, n_q):
    """bf16 attention rows (the prefill / bf16-output path of ep_verify_greedy):
    one bf16 GEMM with LayerNorm folded into the epilogue (z = x.w - mean *
    colsum(w)), no refinement, the acceptance rule in accept_kernel. Logits
    (rstd * z) within a measured error of the fp64 LN(x) @ W; target ids
    bit-exact on every row whose fp64 top-2 gap exceeds 8x that error, and
    accepted counts bit-exact where no guarded row decides them
    (model.cpp:238-255)."""
    import torch
    from paper_2504_11729_b200.verify import VerifyGreedy
    from tests.gpu_util import torch_from_raw
    width, V = 4096, 4096
    rng = np.random.default_rng(B * 31 + n_q)
    W = O.fill_uniform(O.DT_BF16, width * V, 555).reshape(width, V)
    x = rng.uniform(-1.0, 1.0, size=(B, n_q, width)).astype(np.float32) + 0.25  # nonzero mean: the fold matters
    xb = torch.from_numpy(x).to(torch.bfloat16)
    x64 = xb.to(torch.float64).numpy()
    W64 = O.bf16_to_f64(W)
    g_ref, _, _ = O.verify_greedy(x64, W64, np.zeros((B, n_q - 1), np.int32))
    drafts = g_ref[:, :n_q - 1].copy()
    for b in range(B):
        a = b % n_q
        if a < n_q - 1:
            drafts[b, a] = (g_ref[b, a] + 1) % V
    g_ref, nacc_ref, _ = O.verify_greedy(x64, W64, drafts)
    ver = VerifyGreedy(torch_from_raw(np.ascontiguousarray(W.T), O.DT_BF16), handle=cuda_handle)
    tgt, nacc, lg = ver(xb.cuda().view(B, n_q, width), torch.from_numpy(drafts).cuda(), logits=True)
    torch.cuda.synchronize()
    tgt, nacc, lg = tgt.cpu().numpy(), nacc.cpu().numpy(), lg.cpu().numpy().reshape(B, n_q, V)
    xn = (x64 - x64.mean(-1, keepdims=True)) / np.sqrt(x64.var(-1, keepdims=True) + 1e-5)
    ref = xn @ W64
    err = float(np.max(np.abs(lg - ref)))
    assert err < 1e-2 * float(np.max(np.abs(ref)))
    top2 = np.sort(ref, axis=-1)[..., -2:]
    guarded = (top2[..., 1] - top2[..., 0]) < 8 * err
    assert guarded.mean() < 0.2
    assert np.array_equal(tgt[~guarded], g_ref[~guarded])
    for b in range(B):
        if not guarded[b, :min(nacc_ref[b] + 1, n_q - 1)].any():
            assert nacc[b] == nacc_ref[b], (b, nacc[b], nacc_ref[b])
