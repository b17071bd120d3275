"""Pins the CPU oracle (oracle/ep_oracle.c, the "port") against the reference:
its own known answers, the real reference code (oracle/_ref) on identical
inputs, and the committed golden fixtures generated from the reference."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import cases as CS
from tests import splice_cases as SC
from tests.conftest import require_ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def attn_gold():
    return np.load(os.path.join(GOLD, "attention_golden.npz"))


# ---------------------------------------------------- reference known answers

def test_known_answers_port():
    for c in CS.attention_test_cases():
        if "expect" in c:
            got = O.full_attention(c["q"], c["k"], c["v"], *c["span"])
            assert np.allclose(got, c["expect"], rtol=1e-12, atol=0), c["name"]


def test_log_add_exp_identities():
    # matrix_test.cpp:115-129: -inf is the identity, symmetric, no overflow
    assert O.log_add_exp(-np.inf, 3.0) == 3.0
    assert O.log_add_exp(2.0, -np.inf) == 2.0
    assert O.log_add_exp(-np.inf, -np.inf) == -np.inf
    assert abs(O.log_add_exp(1000.0, 1000.0) - (1000.0 + np.log(2))) < 1e-12
    assert O.log_add_exp(0.5, 1.5) == O.log_add_exp(1.5, 0.5)


def test_argmax_tie_break():
    # model_test.cpp: ties break toward the lowest token id
    assert O.argmax([1.0, 3.0, 3.0, -2.0]) == 1
    assert O.argmax([0.5, 0.5, 0.5]) == 0


def test_masked_rows_and_errors():
    q = np.zeros((2, 3))
    o, l = O.partial_attention(q, np.zeros((0, 3)), np.zeros((0, 3)), 0, 0)
    assert np.all(l == -np.inf) and np.all(o == 0)
    o, l = O.partial_attention(q, np.ones((2, 3)), np.ones((2, 3)), 0, 9)
    assert l[0] == -np.inf
    with pytest.raises(O.DomainError):
        O.full_attention(np.zeros((1, 2)), np.zeros((1, 2)), np.zeros((1, 2)), 0, 5)
    with pytest.raises(O.DomainError):
        e = (np.zeros((2, 3)), np.full(2, -np.inf))
        O.fuse_partials([e, e])
    with pytest.raises(O.InvalidArgument):
        O.fuse_partials([])


# -------------------------------------------------- port == reference itself

def test_port_matches_reference_single_calls():
    require_ref()
    for c in CS.attention_test_cases():
        if c["kind"] in ("full",):
            a = O.full_attention(c["q"], c["k"], c["v"], *c["span"], impl="port")
            b = O.full_attention(c["q"], c["k"], c["v"], *c["span"], impl="ref")
            assert np.array_equal(a, b), c["name"]
        elif c["kind"] == "partial":
            a = O.partial_attention(c["q"], c["k"], c["v"], *c["span"], impl="port")
            b = O.partial_attention(c["q"], c["k"], c["v"], *c["span"], impl="ref")
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_port_matches_reference_bitwise_on_all_fusion_cases():
    """Same operation order as the reference -> identical fp64 bits."""
    require_ref()
    for c in CS.all_fuse_cases():
        pp = [O.partial_attention(c["q"], k, v, *sp, impl="port") for k, v, sp in c["segments"]]
        pr = [O.partial_attention(c["q"], k, v, *sp, impl="ref") for k, v, sp in c["segments"]]
        for (a, b), (x, y) in zip(pp, pr):
            assert np.array_equal(a, x) and np.array_equal(b, y), c["name"]
        ma = O.merge_partials(pp, impl="port")
        mb = O.merge_partials(pr, impl="ref")
        assert np.array_equal(ma[0], mb[0]) and np.array_equal(ma[1], mb[1]), c["name"]


def test_port_matches_golden_fixtures(attn_gold):
    for c in CS.attention_test_cases() + CS.all_fuse_cases():
        n = c["name"]
        if c["kind"] == "full":
            got = O.full_attention(c["q"], c["k"], c["v"], *c["span"])
            assert np.array_equal(got, attn_gold[f"{n}/out"]), n
        elif c["kind"] == "partial":
            o, l = O.partial_attention(c["q"], c["k"], c["v"], *c["span"])
            assert np.array_equal(o, attn_gold[f"{n}/out"]) and np.array_equal(
                l, attn_gold[f"{n}/lse"]), n
        else:
            parts = [O.partial_attention(c["q"], k, v, *sp) for k, v, sp in c["segments"]]
            o, l = O.merge_partials(parts)
            assert np.array_equal(o, attn_gold[f"{n}/out"]), n
            assert np.array_equal(l, attn_gold[f"{n}/lse"]), n


def test_fusion_equals_monolithic_acceptance_criterion_1():
    """acceptance_test.cpp:67-129: max rel err <= 1e-9, |sum(alpha)-1| <= 1e-12."""
    max_rel = max_alpha = 0.0
    for c in CS.acceptance_fusion_cases():
        parts = [O.partial_attention(c["q"], k, v, *sp) for k, v, sp in c["segments"]]
        fused = O.fuse_partials(parts)
        k, v, sp = c["full"]
        mono = O.full_attention(c["q"], k, v, *sp)
        max_rel = max(max_rel, CS.rel_err(fused, mono))
        lses = np.stack([l for _, l in parts])
        total = np.full(lses.shape[1], -np.inf)
        for l in lses:
            total = np.array([O.log_add_exp(a, b) for a, b in zip(total, l)])
        alpha = np.where(np.isneginf(lses), 0.0, np.exp(lses - total))
        max_alpha = max(max_alpha, float(np.max(np.abs(alpha.sum(0) - 1.0))))
    assert max_rel <= 1e-9 and max_alpha <= 1e-12


# ------------------------------------------------ batched splice oracle

@pytest.mark.parametrize("name", list(SC.SMALL_CASES))
def test_spliced_batch_port_matches_golden(name):
    gold = np.load(os.path.join(GOLD, "splice_golden.npz"))
    sb = SC.small_case(name)
    from tests.golden.make_golden import digest
    assert str(gold[f"{name}/digest"]) == digest(sb.k_pages, sb.v_pages, sb.q, sb.segs,
                                                  sb.page_table, sb.q_pos)
    o, l = O.spliced_attention(sb, n_threads=4)
    assert np.array_equal(o, gold[f"{name}/out"])
    assert np.array_equal(l, gold[f"{name}/lse"])


def test_spliced_batch_unit_subset_and_threads():
    sb = SC.small_case("gqa4_bf16_decode")
    full_o, full_l = O.spliced_attention(sb, n_threads=1)
    units = np.array([3, 17, 30], dtype=np.int64)
    o, l = O.spliced_attention(sb, n_threads=3, units=units)
    Hq = sb.n_q_heads
    for u in units:
        b, h = divmod(int(u), Hq)
        assert np.array_equal(o[b, :, h], full_o[b, :, h])
    assert np.isnan(o[0, 0, 0]).all()


def test_fill_uniform_matches_splitmix():
    r = O.SplitMix64(99)
    want = [r.uniform(-1, 1) for _ in range(64)]
    assert np.array_equal(O.fill_uniform(O.DT_F64, 64, 99), np.array(want))
    f32 = O.fill_uniform(O.DT_F32, 64, 99)
    assert np.array_equal(f32, np.array(want, dtype=np.float32))
    bf = O.fill_uniform(O.DT_BF16, 64, 99)
    assert np.max(np.abs(O.bf16_to_f64(bf) - f32)) <= 2 ** -8


# ------------------------------------------------ verify (constructed a16)

def test_verify_accept_rule():
    rng = np.random.default_rng(0)
    B, k, W, V = 3, 4, 16, 11
    attn = rng.standard_normal((B, k + 1, W))
    w = rng.standard_normal((W, V))
    tgt, _, _ = O.verify_greedy(attn, w, np.zeros((B, k), np.int32))
    drafts = np.zeros((B, k), np.int32)
    drafts[0] = tgt[0, :k]                                   # all accepted
    drafts[1] = tgt[1, :k]; drafts[1, 2] = (tgt[1, 2] + 1) % V  # reject at 3rd
    drafts[2] = (tgt[2, :k] + 1) % V                         # reject first
    tgt2, nacc, gap = O.verify_greedy(attn, w, drafts)
    assert np.array_equal(tgt, tgt2)
    assert nacc.tolist() == [4, 2, 0]
    assert np.all(gap >= 0)


# ------------------------------------------------ reference model goldens

def test_model_goldens_reproduce():
    require_ref()
    g = json.load(open(os.path.join(GOLD, "model_golden.json")))
    m = O.RefModel(2, 2, 8, 32, 512, 42)
    assert m.weight_sum() == pytest.approx(0.96434447830977787, rel=1e-15)
    assert g["tiny_rollout"] == [30, 30, 24, 7, 7, 7, 30, 30]
    r = O.SplitMix64(7)
    cloud = [r.next_u64() % 32 for _ in range(16)]
    edge = [r.next_u64() % 32 for _ in range(8)]
    assert m.generate_split(cloud, edge, 8) == g["tiny_rollout"]
    assert m.generate_monolithic(cloud + edge, 8) == g["tiny_rollout"]
