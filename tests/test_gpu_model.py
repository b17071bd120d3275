"""GPU parity of the decoder on the device (ep_model)
against the reference's own goldens (tests/golden/model_golden.json, written
by the unmodified reference) and the numpy restatement of model.cpp
(oracle/model_oracle.py, pinned to the reference by test_model_oracle.py).

fp64 models reproduce the reference's tests at the reference's tolerances
(model_test.cpp: golden tokens, weight_sum golden, decode logits 1e-9,
split == monolithic; acceptance criterion 2). fp32 models (BASELINE config 1:
fp32, d_head 64 -> the K1 spliced decode / prefill kernels) are held to the
north-star fp32 tolerance (1e-3, |got - want| / max(1, |want|)) with greedy
tokens bit-exact wherever the oracle's top-2 logit gap exceeds the logit
error bound."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import model_oracle as MO
from oracle import oracle as O
from tests.cases import rel_err

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "model_golden.json")))
CFG1 = (2, 4, 256, 256, 1024, 42)
TINY = (2, 2, 8, 32, 512, 42)


def _mod():
    from paper_2504_11729_b200 import model as M
    return M


def tiny_prompts():
    r = O.SplitMix64(7)
    cloud = [r.next_u64() % 32 for _ in range(16)]
    edge = [r.next_u64() % 32 for _ in range(8)]
    return cloud, edge


def make(cfg, dtype="f64", kv=None, **kw):
    M = _mod()
    return M.Model(M.ModelConfig(*cfg), dtype=dtype, kv_dtype=kv, **kw)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_weight_sum_goldens(cuda_handle, dtype):
    # model_test.cpp:156-160 (Approx epsilon 1e-15); the fp64 draws are summed
    # in generation order, so the value is bit-identical to the reference's
    assert make(TINY, dtype).weight_sum() == GOLD["tiny_weight_sum"]
    assert make(CFG1, dtype).weight_sum() == GOLD["cfg1_weight_sum"]


def _read_device(ptr, n, tdtype):
    """n elements at a raw device pointer -> numpy (cudaMemcpy, cuda-python)."""
    import torch
    from cuda.bindings import runtime as rt
    out = torch.empty(n, dtype=tdtype, device="cuda")
    torch.cuda.synchronize()
    (err,) = rt.cudaMemcpy(out.data_ptr(), ptr, n * out.element_size(),
                           rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
    assert err == rt.cudaError_t.cudaSuccess
    return out.cpu().to(torch.float64).numpy()


def test_weights_are_the_reference_draws(cuda_handle):
    """init_model's stream, element by element: bit-identical in fp64, the
    fp64 draw rounded to nearest in fp32."""
    ref = MO.Model(MO.Config(*TINY))
    for dtype in ("f64", "f32"):
        m = make(TINY, dtype)
        for name, layer, want in (("embedding", 0, ref.embedding), ("unembed", 0, ref.unembed),
                                  ("wq", 0, ref.layers[0].wq), ("w1", 1, ref.layers[1].w1),
                                  ("b1", 1, ref.layers[1].b1), ("b2", 0, ref.layers[0].b2)):
            ptr, n = m.weight_ptr(name, layer)
            assert n == want.size
            w = want.ravel() if dtype == "f64" else want.ravel().astype(np.float32).astype(np.float64)
            np.testing.assert_array_equal(_read_device(ptr, n, m.tdtype), w)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_tiny_rollout_golden(cuda_handle, dtype):
    # model_test.cpp:341-355: split == monolithic == {30,30,24,7,7,7,30,30}
    M = _mod()
    m = make(TINY, dtype)
    cloud, edge = tiny_prompts()
    for loop in (True, False):  # device-resident rollout (CUDA graph) / one decode_step per token
        assert M.generate_split(m, cloud, edge, 8, device_loop=loop) == GOLD["tiny_rollout"]
        assert M.generate_monolithic(m, cloud + edge, 8, device_loop=loop) == GOLD["tiny_rollout"]
    assert m.last_attention_path() == "generic"  # d_head 4
    assert m.pages.free_pages == m.num_pages  # caches released their pages


def test_criterion2_configs_fp64(cuda_handle):
    # acceptance_test.cpp:159-242 (50 random configs, split == monolithic)
    M = _mod()
    for c in GOLD["criterion2_configs"]:
        m = make((c["L"], c["H"], c["D"], c["V"], 256, int(c["seed"])), "f64")
        assert M.generate_split(m, c["cloud"], c["edge"], 16) == c["tokens"], c


def test_cfg1_rollout_fp64(cuda_handle):
    M = _mod()
    m = make(CFG1, "f64")
    got = M.generate_split(m, GOLD["cfg1_cloud"], GOLD["cfg1_edge"], 64)
    assert got == GOLD["cfg1_rollout64"]


def _teacher_forced(m, cfg, n_steps, tol):
    """Prefill cloud then edge, then n_steps decode steps fed with the
    ORACLE's tokens; every step's logits within tol of the oracle and the
    greedy token equal wherever the oracle's top-2 gap exceeds 2x the
    measured logit error."""
    M = _mod()
    ses = MO.Session(MO.Model(MO.Config(*cfg)))
    cloud, edge = GOLD["cfg1_cloud"], GOLD["cfg1_edge"]
    cache = M.SegmentedCache(m)
    pf = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, cache)
    h_c = ses.prefill(cloud)
    assert rel_err(pf.hidden.cpu().numpy(), h_c) <= tol
    cache.append(pf.segments)
    pf = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), cache)
    h_e = ses.prefill(edge)
    assert rel_err(pf.hidden.cpu().numpy(), h_e) <= tol
    cache.append(pf.segments)
    want = ses.model.unembed_logits(h_e[-1])
    got = pf.logits.cpu().numpy()
    errs, guarded = [rel_err(got, want)], 0
    tok = MO.Model.argmax_token(want)
    for _ in range(n_steps):
        r = M.decode_step(m, cache, tok)
        nt, lg = ses.decode_step(tok)
        e = rel_err(r.logits, lg)
        errs.append(e)
        top2 = np.sort(lg)[-2:]
        if top2[1] - top2[0] > 2 * e * max(1.0, abs(top2[1])):
            assert r.next_token == nt
        else:
            guarded += 1
        tok = nt
    cache.release()
    assert max(errs) <= tol, max(errs)
    assert guarded <= n_steps // 8
    return max(errs)


@pytest.mark.parametrize("persist", ["0", "1"])
def test_cfg1_fp32_spliced_kernels(cuda_handle, persist, monkeypatch):
    # decode_step logits of the fp32 serving path against the fp64 reference:
    # K1 spliced decode inside the layer-by-layer forward, or (persist=1, the
    # batch-1 default) the K9 persistent kernel
    monkeypatch.setenv("EP_MODEL_PERSIST", persist)
    m = make(CFG1, "f32", "f32")
    err = _teacher_forced(m, CFG1, 24, 1e-3)
    assert m.last_attention_path() == ("persistent" if persist == "1" else "spliced")  # d_head 64
    assert err <= 1e-4


@pytest.mark.parametrize("persist", ["0", "1"])
def test_cfg1_fp32_rollout_matches_golden(cuda_handle, persist, monkeypatch):
    # fp32 serving path (CUDA-graph rollout, or the K9 persistent kernel that a
    # batch-1 rollout takes by default) = the reference's fp64 greedy tokens
    M = _mod()
    monkeypatch.setenv("EP_MODEL_PERSIST", persist)
    m = make(CFG1, "f32", "f32")
    got = M.generate_split(m, GOLD["cfg1_cloud"], GOLD["cfg1_edge"], 64)
    assert got == GOLD["cfg1_rollout64"]
    assert (m.last_attention_path() == "persistent") == (persist == "1")


def test_cfg1_bf16_kv(cuda_handle):
    m = make(CFG1, "f32", "bf16")  # bf16 pages: never the K9 kernel
    _teacher_forced(m, CFG1, 8, 2e-2)
    assert m.last_attention_path() == "spliced"


def test_cfg1_fp64_decode_logits_1e9(cuda_handle):
    # model_test.cpp:302-333 tolerance on decode_step logits
    M = _mod()
    m = make(CFG1, "f64")
    ses = MO.Session(MO.Model(MO.Config(*CFG1)))
    cloud, edge = GOLD["cfg1_cloud"][:200], GOLD["cfg1_edge"][:30]
    cache = M.SegmentedCache(m)
    for toks, org, pos in ((cloud, M.ORIGIN_CLOUD, 0), (edge, M.ORIGIN_EDGE, len(cloud))):
        pf = M.prefill(m, toks, org, pos, cache)
        cache.append(pf.segments)
        h = ses.prefill(toks)
        assert rel_err(pf.hidden.cpu().numpy(), h) <= 1e-10
    tok = 5
    for _ in range(5):
        r = M.decode_step(m, cache, tok)
        nt, lg = ses.decode_step(tok)
        assert rel_err(r.logits, lg) <= 1e-9
        assert r.next_token == nt
        tok = nt


@pytest.mark.parametrize("dtype,kv", [("f64", "f64"), ("f32", "f32")])
def test_batched_decode_equals_per_session(cuda_handle, dtype, kv):
    """decode_batch over 4 sessions that share one cloud prompt's pages and
    have ragged edge segments = each session's own decode_step on a model of
    its own."""
    M = _mod()
    edges_n = (1, 17, 64, 100)
    rng = O.SplitMix64(11)
    cloud = [rng.next_u64() % 256 for _ in range(130)]
    edges = [[rng.next_u64() % 256 for _ in range(n)] for n in edges_n]

    m = make(CFG1, dtype, kv, num_pages=256)
    pf = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, M.SegmentedCache(m))
    caches, firsts = [], []
    for edge in edges:
        c = M.SegmentedCache(m)
        m.pages.retain(pf.segment.pages)
        c.append(pf.segments)  # the cloud prompt's pages are shared
        e = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), c)
        c.append(e.segments)
        caches.append(c)
        firsts.append(e.next_token)
    nxt, lg = M.decode_batch(m, caches, firsts, want_logits=True)
    for c, n in zip(caches, edges_n):
        assert c.end_position() == len(cloud) + n + 1
    nxt2, lg2 = M.decode_batch(m, caches, [int(t) for t in nxt], want_logits=True)

    tol = 1e-12 if dtype == "f64" else 1e-5
    for b, edge in enumerate(edges):
        m2 = make(CFG1, dtype, kv, num_pages=32)
        c = M.SegmentedCache(m2)
        p0 = M.prefill(m2, cloud, M.ORIGIN_CLOUD, 0, c)
        c.append(p0.segments)
        e = M.prefill(m2, edge, M.ORIGIN_EDGE, len(cloud), c)
        c.append(e.segments)
        assert e.next_token == firsts[b]
        r = M.decode_step(m2, c, firsts[b])
        assert rel_err(r.logits, lg[b]) <= tol
        assert r.next_token == int(nxt[b])
        r = M.decode_step(m2, c, int(nxt[b]))
        assert rel_err(r.logits, lg2[b]) <= tol
        assert r.next_token == int(nxt2[b])


def test_errors_mirror_the_reference(cuda_handle):
    M = _mod()
    m = make(TINY, "f64")
    cache = M.SegmentedCache(m)
    with pytest.raises(ValueError):
        M.decode_step(m, cache, 1)  # model_test.cpp: decode_step rejects an empty cache
    with pytest.raises(ValueError):
        M.prefill(m, [], M.ORIGIN_CLOUD, 0, cache)
    with pytest.raises(ValueError):
        M.prefill(m, [1, 99], M.ORIGIN_CLOUD, 0, cache)  # unknown token id
    with pytest.raises(ValueError):
        M.prefill(m, [1, 2], M.ORIGIN_CLOUD, 3, cache)  # pos_offset != cache end
    pf = M.prefill(m, [1] * 510, M.ORIGIN_CLOUD, 0, cache)
    cache.append(pf.segments)
    M.decode_step(m, cache, 3)
    M.decode_step(m, cache, 3)  # position 511 = max_positions - 1
    with pytest.raises(ValueError):
        M.decode_step(m, cache, 3)  # embed: position overflow
    assert cache.end_position() == 512
    with pytest.raises(ValueError):
        M.ModelConfig(2, 3, 8, 32).validate()


@pytest.mark.parametrize("dtype,kv,persist", [("f64", "f64", "0"), ("f32", "f32", "0"), ("f32", "bf16", "0"),
                                               ("f32", "f32", "1")])
def test_device_rollout_equals_decode_steps(cuda_handle, dtype, kv, persist, monkeypatch):
    """generate_batch (one CUDA graph per step, positions advanced on the
    device, K1 plan built for the final length; or, persist=1, the K9
    persistent kernel) = decode_step per token, for 3 sessions sharing a
    cloud prompt; the cached K/V are the same too."""
    import torch
    M = _mod()
    monkeypatch.setenv("EP_MODEL_PERSIST", persist)
    rng = O.SplitMix64(5)
    cloud = [rng.next_u64() % 256 for _ in range(100)]
    edges = [[rng.next_u64() % 256 for _ in range(n)] for n in (3, 40, 70)]
    n_steps = 70  # crosses a page boundary for every session

    def sessions(m):
        pf = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, M.SegmentedCache(m))
        out = []
        for edge in edges:
            c = M.SegmentedCache(m)
            m.pages.retain(pf.segment.pages)
            c.append(pf.segments)
            e = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), c)
            c.append(e.segments)
            out.append((c, e.next_token))
        return out

    m1 = make(CFG1, dtype, kv, num_pages=64)
    s1 = sessions(m1)
    got = M.generate_batch(m1, [c for c, _ in s1], [t for _, t in s1], n_steps)
    assert (m1.last_attention_path() == "persistent") == (persist != "0")
    m2 = make(CFG1, dtype, kv, num_pages=64)
    s2 = sessions(m2)
    for b, (c, t) in enumerate(s2):
        toks = []
        for _ in range(n_steps):
            t = M.decode_step(m2, c, t).next_token
            toks.append(t)
        assert got[b] == toks, b
        assert s1[b][0].end_position() == c.end_position()
    # cached K: bit-identical in fp64 (same kernels, same order); in fp32 /
    # bf16 the spliced-decode plan of the rollout (built once for the final
    # length) splits the keys differently from the per-step plans, so the fp32
    # summation order differs in the last bits
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[kv]
    for layer in range(CFG1[0]):
        p1, p2 = m1.kv_pool(layer), m2.kv_pool(layer)
        n = p1.num_pages * p1.n_kv_heads * p1.page_tokens * p1.d_head
        a = _read_device(p1.k_pages, n, tdt)
        b2 = _read_device(p2.k_pages, n, tdt)
        if kv == "f64":
            np.testing.assert_array_equal(a, b2)
        else:
            assert rel_err(a, b2) <= (1e-5 if kv == "f32" else 1e-2)


def test_persistent_rollout_batch8_equals_graph_rollout(cuda_handle, monkeypatch):
    """K9 at its largest batch (8 sessions with ragged edges sharing a cloud
    prompt, EP_MODEL_PERSIST=1) = the CUDA-graph rollout, token for token;
    the logits of a following decode_batch agree within fp32 rounding."""
    M = _mod()
    rng = O.SplitMix64(23)
    cloud = [rng.next_u64() % 256 for _ in range(150)]
    edges = [[rng.next_u64() % 256 for _ in range(n)] for n in (1, 5, 31, 32, 33, 64, 65, 120)]
    n_steps = 40

    def run(persist):
        monkeypatch.setenv("EP_MODEL_PERSIST", persist)
        m = make(CFG1, "f32", "f32", num_pages=96)
        pf = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, M.SegmentedCache(m))
        caches, firsts = [], []
        for edge in edges:
            c = M.SegmentedCache(m)
            m.pages.retain(pf.segment.pages)
            c.append(pf.segments)
            e = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), c)
            c.append(e.segments)
            caches.append(c)
            firsts.append(e.next_token)
        toks = M.generate_batch(m, caches, firsts, n_steps)
        path = m.last_attention_path()
        _, lg = M.decode_batch(m, caches, [t[-1] for t in toks], want_logits=True)
        return toks, path, lg

    t1, p1, l1 = run("1")
    t0, p0, l0 = run("0")
    assert (p1, p0) == ("persistent", "spliced")
    assert t1 == t0
    assert rel_err(l1, l0) <= 1e-5


@pytest.mark.parametrize("cfg,n_cloud", [((3, 8, 256, 300, 1024, 7), 70),     # d_head 32, vocab not a multiple of 32
                                         ((1, 2, 128, 250, 1024, 9), 70),     # d_head 64, one layer
                                         ((2, 2, 128, 256, 4096, 5), 2200)])  # > 32 partials per (row, head)
def test_persistent_rollout_other_shapes(cuda_handle, cfg, n_cloud, monkeypatch):
    """K9 on shapes other than config 1 (the d_head 32 attention task, ragged
    column splits, more than 32 key halves per row) = the layer-by-layer
    path: same greedy tokens, logits within fp32 rounding."""
    M = _mod()
    rng = O.SplitMix64(31)
    V = cfg[3]
    cloud = [rng.next_u64() % V for _ in range(n_cloud)]
    edges = [[rng.next_u64() % V for _ in range(n)] for n in (2, 40, 95)]

    def run(persist):
        monkeypatch.setenv("EP_MODEL_PERSIST", persist)
        m = make(cfg, "f32", "f32", num_pages=96)
        pf = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, M.SegmentedCache(m))
        caches, firsts = [], []
        for edge in edges:
            c = M.SegmentedCache(m)
            m.pages.retain(pf.segment.pages)
            c.append(pf.segments)
            e = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), c)
            c.append(e.segments)
            caches.append(c)
            firsts.append(e.next_token)
        toks = M.generate_batch(m, caches, firsts, 24)
        path = m.last_attention_path()
        _, lg = M.decode_batch(m, caches, [t[-1] for t in toks], want_logits=True)
        one = M.decode_step(m, caches[2], 1)  # batch 1: every CTA merges the row itself
        return toks, path, lg, one

    t1, p1, l1, o1 = run("1")
    t0, p0, l0, o0 = run("0")
    assert p1 == "persistent" and p0 != "persistent"
    assert t1 == t0
    assert rel_err(l1, l0) <= 1e-5
    assert o1.next_token == o0.next_token and rel_err(o1.logits, o0.logits) <= 1e-5


@pytest.mark.parametrize("dtype,kv", [("f64", "f64"), ("f32", "f32")])
def test_verify_matches_reference_prefill(cuda_handle, dtype, kv):
    """Greedy speculative verify on config 1's decoder (the
    rest of it): per round, [last, d1..dk] (k = 4 / 8, drafts from the
    reference's own rollout with a forced mismatch at a varying place) go
    through ep_model_verify; every row's target must equal the reference's
    own construction — prefill(model, [last, d1..dk], generated, end, cache)
    + unembed_logits + argmax_token per row (oracle/_ref, unmodified
    sources) — and the accepted count its acceptance rule. fp64: bit-exact
    everywhere; fp32: logits within 1e-3 and ids bit-exact outside the
    margin guard. The cache then keeps last, d1..dn, so the rounds stay in
    step with a reference session advanced by n + 1 decode_steps."""
    M = _mod()
    if not O.available("ref"):
        pytest.skip("oracle/_ref not built")
    m = make(CFG1, dtype, kv, num_pages=64)
    cloud, edge = GOLD["cfg1_cloud"], GOLD["cfg1_edge"]
    ref = O.RefModel(*CFG1[:4], max_positions=CFG1[4], seed=CFG1[5])
    ses = ref.session(cloud, edge)
    cache = M.SegmentedCache(m)
    pf = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, cache, want_hidden=False)
    cache.append(pf.segments)
    pf = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), cache, want_hidden=False)
    cache.append(pf.segments)
    last = ses.first_token()
    assert pf.next_token == last
    roll = list(GOLD["cfg1_rollout64"])  # the reference's greedy continuation (roll[0] == last)
    assert roll[0] == last
    pos = 0                                 # index of `last` in roll
    checked, guarded = 0, 0
    for rnd, (k, a) in enumerate([(4, 4), (4, 1), (8, 0), (8, 5), (4, 2), (8, 8), (4, 3)]):
        drafts = list(roll[pos + 1:pos + 1 + k])
        if a < k:                           # force the first mismatch at draft a+1
            drafts[a] = (drafts[a] + 1) % CFG1[3]
        want_t, want_lg = ses.verify([last] + drafts)
        want_n = 0
        while want_n < k and drafts[want_n] == want_t[want_n]:
            want_n += 1
        r = M.verify_greedy(m, cache, last, drafts, want_logits=True)
        err = rel_err(r.logits, want_lg)
        if dtype == "f64":
            assert err <= 1e-9
            assert np.array_equal(r.targets, want_t), (rnd, r.targets, want_t)
            assert len(r.accepted) == want_n
        else:
            assert err <= 1e-3, err
            top2 = np.sort(want_lg, axis=1)[:, -2:]
            safe = (top2[:, 1] - top2[:, 0]) > 4 * err * np.maximum(1.0, np.abs(top2[:, 1]))
            guarded += int((~safe).sum())
            assert np.array_equal(r.targets[safe], want_t[safe]), (rnd, r.targets, want_t)
            if safe[:want_n + 1].all():
                assert len(r.accepted) == want_n
        assert r.next_token == want_t[len(r.accepted)]
        checked += k + 1
        # the reference session takes last, d1..dn as n + 1 decode steps
        n = len(r.accepted)
        for t in [last] + drafts[:n]:
            ses.decode_step(t)
        assert cache.end_position() == ses.end_position
        last = r.next_token
        pos += n + 1
        assert roll[pos] == last            # accepted + bonus = the greedy rollout
    # a decode step after the verify rounds still matches the reference
    d = M.decode_step(m, cache, last)
    nt, _ = ses.decode_step(last)
    assert d.next_token == nt
    cache.release()
    assert guarded <= checked // 10
