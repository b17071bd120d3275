"""Deterministic input cases mirroring the reference's own tests.

Each generator reproduces the seeds and draw order of a reference test so the
inputs are bit-identical to what that test feeds the reference:

* attention_test.cpp:19-23 random_matrix = U(-2, 2) row-major;
* acceptance_test.cpp:50-56 random_matrix = U(-1, 1) row-major.

A case is a dict: kind ("partial" | "full" | "fuse" | "merge"), q, segments
[(k, v, span)], plus what the reference test asserts.
"""
from __future__ import annotations

import numpy as np

from oracle.oracle import SplitMix64


def _m(rng: SplitMix64, r: int, c: int, lo: float, hi: float) -> np.ndarray:
    return rng.matrix(r, c, lo, hi)


def attention_test_cases():
    """Known-answer and oracle cases of attention_test.cpp (file:line in 'src')."""
    cases = []
    # :83-90 single key -> 7.0
    cases.append(dict(name="single_key", src="attention_test.cpp:83-90", kind="full",
                      q=np.array([[1.0]]), k=np.array([[1.0]]), v=np.array([[7.0]]),
                      span=(0, 0), expect=np.array([[7.0]])))
    # :92-103 identical keys -> mean of visible values 2.0
    q = np.array([[0.3, -1.1]])
    k = np.tile(np.array([[0.5, 0.25]]), (3, 1))
    v = np.array([[1.0], [2.0], [3.0]])
    # the reference case has v with one column; our ABI takes one head width,
    # so the single value column is padded with a zero column (same math).
    cases.append(dict(name="identical_keys", src="attention_test.cpp:92-103", kind="full",
                      q=q, k=k, v=np.hstack([v, np.zeros((3, 1))]), span=(2, 0),
                      expect=np.array([[2.0, 0.0]])))
    rng = SplitMix64(11)  # :105-116
    q, k, v = _m(rng, 4, 8, -2, 2), _m(rng, 6, 8, -2, 2), _m(rng, 6, 8, -2, 2)
    cases.append(dict(name="no_mask", src="attention_test.cpp:105-116", kind="full", q=q, k=k,
                      v=v, span=(10, 0)))
    rng = SplitMix64(12)  # :118-128
    q, k, v = _m(rng, 5, 4, -2, 2), _m(rng, 5, 4, -2, 2), _m(rng, 5, 4, -2, 2)
    cases.append(dict(name="causal", src="attention_test.cpp:118-128", kind="full", q=q, k=k,
                      v=v, span=(0, 0)))
    rng = SplitMix64(13)  # :140-152
    q, k, v = _m(rng, 3, 4, -2, 2), _m(rng, 7, 4, -2, 2), _m(rng, 7, 4, -2, 2)
    cases.append(dict(name="partial_eq_full", src="attention_test.cpp:140-152", kind="partial",
                      q=q, k=k, v=v, span=(6, 0)))
    rng = SplitMix64(14)  # :168-190
    q, k, v = _m(rng, 4, 5, -2, 2), _m(rng, 10, 5, -2, 2), _m(rng, 10, 5, -2, 2)
    cases.append(dict(name="split_3_7", src="attention_test.cpp:168-190", kind="fuse", q=q,
                      segments=[(k[:3], v[:3], (9, 0)), (k[3:], v[3:], (9, 3))], full=(k, v, (9, 0))))
    rng = SplitMix64(15)  # :192-202
    q, k, v = _m(rng, 3, 4, -2, 2), _m(rng, 5, 4, -2, 2), _m(rng, 5, 4, -2, 2)
    cases.append(dict(name="single_partial", src="attention_test.cpp:192-202", kind="fuse", q=q,
                      segments=[(k, v, (4, 0))], full=(k, v, (4, 0))))
    rng = SplitMix64(16)  # :204-218
    q, k, v = _m(rng, 2, 4, -2, 2), _m(rng, 3, 4, -2, 2), _m(rng, 3, 4, -2, 2)
    cases.append(dict(name="identical_segments", src="attention_test.cpp:204-218", kind="fuse",
                      q=q, segments=[(k, v, (5, 0)), (k, v, (5, 0))], full=None))
    rng = SplitMix64(17)  # :220-234
    q, k, v = _m(rng, 6, 8, -2, 2), _m(rng, 22, 8, -2, 2), _m(rng, 22, 8, -2, 2)
    cases.append(dict(name="cloud13_edge9", src="attention_test.cpp:220-234", kind="fuse", q=q,
                      segments=[(k[:13], v[:13], (21, 0)), (k[13:], v[13:], (21, 13))],
                      full=(k, v, (21, 0))))
    return cases


def splitting_invariance_cases():
    """attention_test.cpp:244-287 (seed 18, 200 random partitions)."""
    rng = SplitMix64(18)
    cases = []
    while len(cases) < 200:
        n_q = 1 + rng.next_u64() % 16
        n_k = 1 + rng.next_u64() % 64
        d = 1 + rng.next_u64() % 16
        n_seg = 1 + rng.next_u64() % 4
        span = (n_k - 1, 0)
        q, k, v = _m(rng, n_q, d, -2, 2), _m(rng, n_k, d, -2, 2), _m(rng, n_k, d, -2, 2)
        cuts = [0, n_k] + [rng.next_u64() % (n_k + 1) for _ in range(1, n_seg)]
        cuts.sort()
        segs = [(k[lo:hi], v[lo:hi], (span[0], lo)) for lo, hi in zip(cuts[:-1], cuts[1:])]
        cases.append(dict(name=f"invariance_{len(cases)}", src="attention_test.cpp:244-287",
                          kind="fuse", q=q, segments=segs, full=(k, v, span)))
    return cases


def acceptance_fusion_cases():
    """acceptance_test.cpp:67-129 (criterion 1, seed 101, 500 cases, U(-1,1)).
    Empty cuts become identity partials (acceptance_test.cpp:97-100)."""
    rng = SplitMix64(101)
    cases = []
    for it in range(500):
        n_q = 1 + rng.next_u64() % 16
        n_k = 1 + rng.next_u64() % 64
        d = 1 + rng.next_u64() % 16
        causal = it % 2 == 1
        if causal and n_k < n_q:
            n_k = n_q
        q_off = n_k - n_q if causal else n_k
        q, k, v = _m(rng, n_q, d, -1, 1), _m(rng, n_k, d, -1, 1), _m(rng, n_k, d, -1, 1)
        n_seg = 1 + rng.next_u64() % 4
        cuts = [0, n_k] + [rng.next_u64() % (n_k + 1) for _ in range(1, n_seg)]
        cuts.sort()
        segs = [(k[lo:hi], v[lo:hi], (q_off, lo)) for lo, hi in zip(cuts[:-1], cuts[1:])]
        cases.append(dict(name=f"accept_{it}", src="acceptance_test.cpp:67-129", kind="fuse",
                          q=q, segments=segs, full=(k, v, (q_off, 0))))
    return cases


def pairwise_merge_cases():
    """attention_test.cpp:289-315 (seed 19, 40 rounds): merge({a,b}) then fuse
    with c equals one-shot fuse({a,b,c})."""
    rng = SplitMix64(19)
    cases = []
    for _ in range(40):
        d = 1 + rng.next_u64() % 8
        n_q = 1 + rng.next_u64() % 6
        n_k = 3 + rng.next_u64() % 20
        q_off = n_k - 1
        q, k, v = _m(rng, n_q, d, -2, 2), _m(rng, n_k, d, -2, 2), _m(rng, n_k, d, -2, 2)
        c1 = 1 + rng.next_u64() % (n_k - 2)
        c2 = c1 + 1 + rng.next_u64() % (n_k - c1 - 1)
        segs = [(k[:c1], v[:c1], (q_off, 0)), (k[c1:c2], v[c1:c2], (q_off, c1)),
                (k[c2:], v[c2:], (q_off, c2))]
        cases.append(dict(name=f"pairwise_{len(cases)}", src="attention_test.cpp:289-315",
                          kind="fuse", q=q, segments=segs, full=(k, v, (q_off, 0))))
    return cases


def all_fuse_cases():
    return ([c for c in attention_test_cases() if c["kind"] == "fuse"] +
            splitting_invariance_cases() + acceptance_fusion_cases() + pairwise_merge_cases())


def rel_err(got, want) -> float:
    """|got - want| / max(1, |want|) (acceptance_test.cpp:107-109, attention_test.cpp:73-79)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))))
