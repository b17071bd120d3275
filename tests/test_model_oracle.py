"""CPU: the numpy decoder oracle (oracle/model_oracle.py) pinned against the
reference's goldens (tests/golden/model_golden.json, written by the unmodified
reference) and, where oracle/_ref is built, against the reference itself."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import model_oracle as MO
from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "model_golden.json")))


def tiny_prompts():
    r = O.SplitMix64(7)  # model_test.cpp:341-355
    cloud = [r.next_u64() % 32 for _ in range(16)]
    edge = [r.next_u64() % 32 for _ in range(8)]
    return cloud, edge


def test_weight_sum_goldens():
    m = MO.Model(MO.Config(2, 2, 8, 32, 512, 42))
    assert m.weight_sum() == GOLD["tiny_weight_sum"]  # model_test.cpp:156-160
    m1 = MO.Model(MO.Config(2, 4, 256, 256, 1024, 42))
    assert m1.weight_sum() == GOLD["cfg1_weight_sum"]


def test_tiny_rollout_golden_split_and_monolithic():
    m = MO.Model(MO.Config(2, 2, 8, 32, 512, 42))
    cloud, edge = tiny_prompts()
    assert MO.generate_split(m, cloud, edge, 8) == GOLD["tiny_rollout"] == [30, 30, 24, 7, 7, 7, 30, 30]
    assert MO.generate_monolithic(m, cloud + edge, 8) == GOLD["tiny_rollout"]


def test_criterion2_configs():
    for c in GOLD["criterion2_configs"]:
        m = MO.Model(MO.Config(c["L"], c["H"], c["D"], c["V"], 256, int(c["seed"])))
        assert MO.generate_split(m, c["cloud"], c["edge"], 16) == c["tokens"]


def test_cfg1_rollout_golden():
    m = MO.Model(MO.Config(2, 4, 256, 256, 1024, 42))
    got = MO.generate_split(m, GOLD["cfg1_cloud"], GOLD["cfg1_edge"], 64)
    assert got == GOLD["cfg1_rollout64"]


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
def test_decode_logits_match_reference():
    for cfg, cloud, edge in [((2, 2, 8, 32, 512, 42), *tiny_prompts()),
                             ((2, 4, 256, 256, 1024, 42), GOLD["cfg1_cloud"][:96],
                              GOLD["cfg1_edge"][:16])]:
        ref = O.RefModel(*cfg).session(cloud, edge)
        ses = MO.Session(MO.Model(MO.Config(*cfg)))
        ses.prefill(cloud)
        h = ses.prefill(edge)
        tok = MO.Model.argmax_token(ses.model.unembed_logits(h[-1]))
        assert tok == ref.first_token()
        for _ in range(4):
            nt, lg = ses.decode_step(tok)
            rt, rl = ref.decode_step(tok)
            assert nt == rt
            assert np.max(np.abs(lg - rl) / np.maximum(1.0, np.abs(rl))) <= 1e-10
            tok = nt
