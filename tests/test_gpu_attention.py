"""GPU parity: the C-ABI drop-in entry points (fp64 host buffers and device
pointers) against the reference goldens, with the reference's OWN tolerances
(1e-9 / 1e-12 in fp64), and the error behaviour of attention.cpp."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import cases as CS

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "attention_golden.npz"))


@pytest.fixture(scope="module")
def ep(cuda_handle):
    import paper_2504_11729_b200 as ep
    return ep


def test_known_answers(ep, cuda_handle, gold):
    for c in CS.attention_test_cases():
        span = ep.CausalSpan(*c["span"]) if "span" in c else None
        if c["kind"] == "full":
            got = ep.full_attention(c["q"], c["k"], c["v"], span, handle=cuda_handle)
            if "expect" in c:
                assert CS.rel_err(got, c["expect"]) <= 1e-12, c["name"]
            assert CS.rel_err(got, gold[f"{c['name']}/out"]) <= 1e-12, c["name"]
        elif c["kind"] == "partial":
            p = ep.partial_attention(c["q"], c["k"], c["v"], span, handle=cuda_handle)
            assert CS.rel_err(p.out, gold[f"{c['name']}/out"]) <= 1e-12
            assert CS.rel_err(p.lse, gold[f"{c['name']}/lse"]) <= 1e-10


def test_all_fusion_cases_match_reference_fp64(ep, cuda_handle, gold):
    """attention_test 3+7 / 13+9 / invariance / pairwise and acceptance
    criterion 1 on the GPU, reference tolerance 1e-9 vs monolithic."""
    worst = 0.0
    for c in CS.all_fuse_cases():
        parts = [ep.partial_attention(c["q"], k, v, ep.CausalSpan(*sp), handle=cuda_handle)
                 for k, v, sp in c["segments"]]
        m = ep.merge_partials(parts, handle=cuda_handle)
        worst = max(worst, CS.rel_err(m.out, gold[f"{c['name']}/out"]))
        assert CS.rel_err(m.out, gold[f"{c['name']}/out"]) <= 1e-9, c["name"]
        lse_g = gold[f"{c['name']}/lse"]
        fin = np.isfinite(lse_g)
        assert np.array_equal(np.isfinite(m.lse), fin)
        assert CS.rel_err(m.lse[fin], lse_g[fin]) <= 1e-10
        if f"{c['name']}/full" in gold:
            fused = ep.fuse_partials(parts, handle=cuda_handle)
            assert CS.rel_err(fused, gold[f"{c['name']}/full"]) <= 1e-9, c["name"]
    print(f"max rel err vs reference over all fusion cases: {worst:.3e}")


def test_pairwise_merge_equals_one_shot(ep, cuda_handle):
    for c in CS.pairwise_merge_cases():
        a, b, cc = [ep.partial_attention(c["q"], k, v, ep.CausalSpan(*sp), handle=cuda_handle)
                    for k, v, sp in c["segments"]]
        one = ep.fuse_partials([a, b, cc], handle=cuda_handle)
        ab = ep.merge_partials([a, b], handle=cuda_handle)
        step = ep.fuse_partials([ab, cc], handle=cuda_handle)
        assert np.max(np.abs(one - step)) <= 1e-12


def test_error_behaviour(ep, cuda_handle):
    q = np.zeros((2, 3))
    p = ep.partial_attention(q, np.zeros((0, 3)), np.zeros((0, 3)), ep.CausalSpan(0, 0),
                             handle=cuda_handle)
    assert p.n_keys == 0 and np.all(p.lse == -np.inf) and np.all(p.out == 0)
    m = ep.partial_attention(q, np.ones((2, 3)), np.ones((2, 3)), ep.CausalSpan(0, 9),
                             handle=cuda_handle)
    assert m.lse[0] == -np.inf
    with pytest.raises(ep.DomainError):
        ep.full_attention(np.zeros((1, 2)), np.zeros((1, 2)), np.zeros((1, 2)),
                          ep.CausalSpan(0, 5), handle=cuda_handle)
    with pytest.raises(ep.DomainError):
        ep.fuse_partials([p, p], handle=cuda_handle)
    with pytest.raises(ep.InvalidArgument):
        ep.fuse_partials([], handle=cuda_handle)
    with pytest.raises(ep.InvalidArgument):
        ep.full_attention(q, np.zeros((1, 4)), np.zeros((1, 4)), handle=cuda_handle)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_device_path(ep, cuda_handle, gold, dtype):
    import torch
    tdt = getattr(torch, dtype)
    tol = 1e-9 if dtype == "float64" else 1e-3
    for c in CS.splitting_invariance_cases()[:60]:
        parts = []
        for k, v, sp in c["segments"]:
            parts.append(ep.partial_attention(torch.tensor(c["q"], dtype=tdt, device="cuda"),
                                              torch.tensor(k, dtype=tdt, device="cuda"),
                                              torch.tensor(v, dtype=tdt, device="cuda"),
                                              ep.CausalSpan(*sp), handle=cuda_handle))
        fused = ep.fuse_partials(parts, handle=cuda_handle)
        assert CS.rel_err(fused.cpu().numpy(), gold[f"{c['name']}/full"]) <= tol, c["name"]


def test_larger_heads_and_keys(ep, cuda_handle):
    """Model-scale per-head calls (d = 64/128/256, thousands of keys)."""
    r = O.SplitMix64(5)
    for d, n_k, n_q in [(64, 577, 1), (128, 4609, 3), (256, 1000, 2)]:
        q = O.fill_uniform(O.DT_F64, n_q * d, r.next_u64()).reshape(n_q, d)
        k = O.fill_uniform(O.DT_F64, n_k * d, r.next_u64()).reshape(n_k, d)
        v = O.fill_uniform(O.DT_F64, n_k * d, r.next_u64()).reshape(n_k, d)
        want_o, want_l = O.partial_attention(q, k, v, n_k - n_q, 0)
        p = ep.partial_attention(q, k, v, ep.CausalSpan(n_k - n_q, 0), handle=cuda_handle)
        assert CS.rel_err(p.out, want_o) <= 1e-11
        assert CS.rel_err(p.lse, want_l) <= 1e-12
