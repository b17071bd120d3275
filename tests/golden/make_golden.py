"""Generates the committed golden fixtures from the REAL reference.

    make -C oracle ref && python tests/golden/make_golden.py

Runs the unmodified reference sources (oracle/_ref/libep_ref.so, compiled from
/root/reference/proj/core by oracle/Makefile) on the inputs of tests/cases.py
and tests/splice_cases.py and stores the outputs. The GPU box has no
/root/reference, so the parity tests read these files instead.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests import cases as CS  # noqa: E402
from tests import splice_cases as SC  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def attention_golden() -> dict:
    out = {}
    for c in CS.attention_test_cases() + CS.all_fuse_cases():
        n = c["name"]
        if n in out or f"{n}/out" in out:
            continue
        if c["kind"] == "full":
            out[f"{n}/out"] = O.full_attention(c["q"], c["k"], c["v"], *c["span"], impl="ref")
            out[f"{n}/digest"] = np.array(digest(c["q"], c["k"], c["v"]))
        elif c["kind"] == "partial":
            o, l = O.partial_attention(c["q"], c["k"], c["v"], *c["span"], impl="ref")
            out[f"{n}/out"], out[f"{n}/lse"] = o, l
            out[f"{n}/digest"] = np.array(digest(c["q"], c["k"], c["v"]))
        else:
            parts = [O.partial_attention(c["q"], k, v, *sp, impl="ref") for k, v, sp in
                     c["segments"]]
            mo, ml = O.merge_partials(parts, impl="ref")
            out[f"{n}/out"], out[f"{n}/lse"] = mo, ml
            out[f"{n}/part_lse"] = np.stack([l for _, l in parts])
            out[f"{n}/digest"] = np.array(digest(c["q"], *[x for k, v, _ in c["segments"]
                                                           for x in (k, v)]))
            if c.get("full") is not None:
                k, v, sp = c["full"]
                out[f"{n}/full"] = O.full_attention(c["q"], k, v, *sp, impl="ref")
    return out


def splice_golden() -> dict:
    out = {}
    for name in SC.SMALL_CASES:
        sb = SC.small_case(name)
        o, l = O.spliced_attention(sb, n_threads=8, impl="ref")
        out[f"{name}/out"], out[f"{name}/lse"] = o, l
        out[f"{name}/digest"] = np.array(digest(sb.k_pages, sb.v_pages, sb.q, sb.segs,
                                                sb.page_table, sb.q_pos))
    return out


def model_golden() -> dict:
    g = {}
    m = O.RefModel(2, 2, 8, 32, 512, 42)
    g["tiny_weight_sum"] = m.weight_sum()
    r = O.SplitMix64(7)
    cloud = [r.next_u64() % 32 for _ in range(16)]
    edge = [r.next_u64() % 32 for _ in range(8)]
    g["tiny_rollout"] = m.generate_split(cloud, edge, 8)
    assert g["tiny_rollout"] == [30, 30, 24, 7, 7, 7, 30, 30]
    # config 1: L=2, H=4, D=256, V=256, seed 42; cloud 512 + edge 64 tokens
    # drawn from SplitMix64(1) mod V.
    m1 = O.RefModel(2, 4, 256, 256, 1024, 42)
    r = O.SplitMix64(1)
    toks = [r.next_u64() % 256 for _ in range(576)]
    g["cfg1_cloud"], g["cfg1_edge"] = toks[:512], toks[512:]
    g["cfg1_weight_sum"] = m1.weight_sum()
    g["cfg1_rollout64"] = m1.generate_split(toks[:512], toks[512:], 64)
    # acceptance criterion 2 in-process (acceptance_test.cpp:159-242, seed 202)
    rng = O.SplitMix64(202)
    cfgs = []
    for _ in range(50):
        L = 1 + rng.next_u64() % 4
        H = 1 + rng.next_u64() % 4
        D = H * (1 + rng.next_u64() % (32 // H))
        V = 8 + rng.next_u64() % 57
        seed = rng.next_u64()
        cl = [rng.next_u64() % V for _ in range(1 + rng.next_u64() % 64)]
        ed = [rng.next_u64() % V for _ in range(4 + rng.next_u64() % 29)]
        mm = O.RefModel(L, H, D, V, 256, seed)
        toks_split = mm.generate_split(cl, ed, 16)
        assert toks_split == mm.generate_monolithic(cl + ed, 16)
        cfgs.append(dict(L=L, H=H, D=D, V=V, seed=str(seed), cloud=cl, edge=ed,
                         tokens=toks_split))
    g["criterion2_configs"] = cfgs
    return g


def main() -> None:
    if not O.available("ref"):
        O.build(with_ref=True)
    np.savez_compressed(os.path.join(HERE, "attention_golden.npz"), **attention_golden())
    np.savez_compressed(os.path.join(HERE, "splice_golden.npz"), **splice_golden())
    with open(os.path.join(HERE, "model_golden.json"), "w") as f:
        json.dump(model_golden(), f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
