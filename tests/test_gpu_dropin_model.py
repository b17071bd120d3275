"""The drop-in proof: the reference's own model/cache code (model.cpp,
cache.cpp, matrix.cpp compiled unmodified) linked against
paper_2504_11729_b200/csrc/dropin/attention_dropin.cpp INSTEAD of
attention.cpp (oracle/_ref/libep_ref_dropin.so), so every partial_attention /
merge_partials of prefill and decode_step runs on the B200 through the C-ABI.
The reference's golden tokens and token-equality invariants must still hold."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    if not O.available("dropin"):
        pytest.skip("oracle/_ref/libep_ref_dropin.so not built")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return json.load(open(os.path.join(GOLD, "model_golden.json")))


def test_tiny_golden_rollout(gold):
    """model_test.cpp:341-355: {30,30,24,7,7,7,30,30}, split == monolithic."""
    m = O.RefModel(2, 2, 8, 32, 512, 42, impl="dropin")
    assert m.weight_sum() == pytest.approx(0.96434447830977787, rel=1e-15)
    r = O.SplitMix64(7)
    cloud = [r.next_u64() % 32 for _ in range(16)]
    edge = [r.next_u64() % 32 for _ in range(8)]
    assert m.generate_split(cloud, edge, 8) == [30, 30, 24, 7, 7, 7, 30, 30]
    assert m.generate_monolithic(cloud + edge, 8) == [30, 30, 24, 7, 7, 7, 30, 30]


def test_criterion2_token_equality(gold):
    """acceptance_test.cpp:159-242 in process: 50 random configs, split and
    monolithic tokens equal the reference's, attention on the GPU."""
    mism = 0
    for c in gold["criterion2_configs"]:
        m = O.RefModel(c["L"], c["H"], c["D"], c["V"], 256, int(c["seed"]), impl="dropin")
        split = m.generate_split(c["cloud"], c["edge"], 16)
        mono = m.generate_monolithic(c["cloud"] + c["edge"], 16)
        mism += int(split != c["tokens"]) + int(mono != c["tokens"])
    assert mism == 0


def test_config1_rollout(gold):
    """BASELINE config 1 (L=2, H=4, D=256, cloud 512 + edge 64): 64 greedy
    tokens identical to the reference CPU run."""
    m = O.RefModel(2, 4, 256, 256, 1024, 42, impl="dropin")
    assert m.generate_split(gold["cfg1_cloud"], gold["cfg1_edge"], 64) == gold["cfg1_rollout64"]


def test_decode_step_logits_match_reference(gold):
    """model_test.cpp:302-333: decode_step logits within 1e-9 of the CPU path."""
    from tests.conftest import require_ref
    require_ref()
    ref = O.RefModel(2, 4, 256, 256, 1024, 42, impl="ref").session(gold["cfg1_cloud"],
                                                                    gold["cfg1_edge"])
    gpu = O.RefModel(2, 4, 256, 256, 1024, 42, impl="dropin").session(gold["cfg1_cloud"],
                                                                      gold["cfg1_edge"])
    tok_r, tok_g = ref.first_token(), gpu.first_token()
    assert tok_r == tok_g
    for _ in range(8):
        nr, lr = ref.decode_step(tok_r)
        ng, lg = gpu.decode_step(tok_g)
        assert nr == ng
        assert np.max(np.abs(lg - lr) / np.maximum(1.0, np.abs(lr))) <= 1e-9
        tok_r, tok_g = nr, ng
