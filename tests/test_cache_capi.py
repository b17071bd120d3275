"""ep_cache (the C-ABI SegmentedCache, include/ep/ep_attn.h §2b) on CPU: the
reference's own cache tests (/root/reference/proj/tests/cache_test.cpp)
restated on the paged form — append invariants and atomicity, origin order,
generated-token growth without copies, cross-layer consistency — plus the
paged specifics (page slots of new tokens, truncation of rejected drafts,
the plan-layout export). Host-only calls: no GPU needed."""
import numpy as np
import pytest

from paper_2504_11729_b200._capi import InvalidArgument
from paper_2504_11729_b200.splice import (ORIGIN_CLOUD, ORIGIN_EDGE, ORIGIN_GENERATED, SpliceCache)

P = 4  # tokens per page (small, so page boundaries are exercised)


def pages(n, start=0):
    return np.arange(start, start + n, dtype=np.int32)


def test_empty_cache():
    # cache_test.cpp "empty cache reports empty and position zero"
    c = SpliceCache(3, 1, P)
    assert c.end_position(0) == 0
    assert c.check_consistent() == ""
    indptr, segs, pt = c.arrays(0)
    assert list(indptr) == [0, 0] and segs.size == 0


def test_zero_layers_rejected():
    with pytest.raises(InvalidArgument):
        SpliceCache(0, 1, P)


def test_append_keeps_layers_aligned_and_gapless():
    # cache_test.cpp "append keeps layers aligned and positions gapless"
    c = SpliceCache(2, 1, P)
    c.append(0, ORIGIN_CLOUD, 0, 3, pages(1))
    assert c.end_position(0) == 3
    c.append(0, ORIGIN_EDGE, 3, 2, pages(1, 1))
    assert c.end_position(0) == 5
    assert c.check_consistent() == ""
    for layer in range(2):
        _, segs, pt = c.arrays(layer)
        assert [int(s["origin"]) for s in segs] == [ORIGIN_CLOUD, ORIGIN_EDGE]
        assert int(segs[1]["pos_offset"]) == 3 and list(pt) == [0, 1]


def test_append_rejects_gaps_overlaps_empty_and_is_atomic():
    # cache_test.cpp "append rejects gaps, overlaps, and malformed batches"
    c = SpliceCache(2, 1, P)
    c.append(0, ORIGIN_CLOUD, 0, 3, pages(1))
    for pos, n in ((4, 1), (2, 1), (3, 0)):         # gap, overlap, empty segment
        with pytest.raises(InvalidArgument):
            c.append(0, ORIGIN_EDGE, pos, n, pages(1, 5))
    with pytest.raises(InvalidArgument):           # fewer pages than tokens
        c.append(0, ORIGIN_EDGE, 3, 9, pages(2, 5))
    assert c.end_position(0) == 3                  # nothing was appended by any failed call
    assert c.check_consistent() == ""


def test_origin_order():
    # cache_test.cpp "origin order is cloud then edge then generated"
    c = SpliceCache(1, 1, P)
    c.append(0, ORIGIN_EDGE, 0, 2, pages(1))
    with pytest.raises(InvalidArgument):
        c.append(0, ORIGIN_CLOUD, 2, 1, pages(1, 1))
    c.append_generated([1], [[7]])
    _, segs, _ = c.arrays(0)
    assert int(segs[-1]["origin"]) == ORIGIN_GENERATED


def test_generated_tokens_extend_in_place_with_page_slots():
    # cache_test.cpp "generated tokens extend one position at a time", paged:
    # the new tokens take the last page's free slots, then fresh pages
    c = SpliceCache(2, 2, P)
    c.append(0, ORIGIN_EDGE, 0, 2, pages(1, 0))
    c.append(1, ORIGIN_CLOUD, 0, 4, pages(1, 1))
    dp, ds, used = c.append_generated([1, 1], [[10, 11], [12, 13]])
    assert (c.end_position(0), c.end_position(1)) == (3, 5)
    assert list(dp) == [10, 12] and list(ds) == [0, 0] and list(used) == [1, 1]
    assert c.check_consistent() == ""
    dp, ds, used = c.append_generated([5, 0], [[20, 21], [22, 23]])
    assert c.end_position(0) == 8 and c.end_position(1) == 5
    assert list(dp) == [10, 10, 10, 20, 20] and list(ds) == [1, 2, 3, 0, 1] and list(used) == [1, 0]
    for layer in range(2):   # one generated segment per layer, grown in place
        indptr, segs, pt = c.arrays(layer)
        s = segs[indptr[0]:indptr[1]]
        assert len(s) == 2 and int(s[1]["len"]) == 6 and int(s[1]["pos_offset"]) == 2
    with pytest.raises(InvalidArgument):           # a full page and no new page supplied
        c.append_generated([9, 0], None)


def test_truncate_rejected_drafts():
    c = SpliceCache(2, 1, P)
    c.append(0, ORIGIN_EDGE, 0, 3, pages(1))
    c.append_generated([7], [[5, 6]])              # positions 3..9: pages 0 (slot 3), 5, 6
    assert c.end_position(0) == 10
    rel = c.truncate(0, 5)                         # keep positions 3..4
    assert c.end_position(0) == 5 and list(rel) == [6]
    rel = c.truncate(0, 2)
    assert c.end_position(0) == 3 and list(rel) == [5]
    with pytest.raises(InvalidArgument):
        c.truncate(0, 1)                           # no generated tokens left
    assert c.check_consistent() == ""


def test_check_consistent_flags_per_layer_divergence():
    # cache_test.cpp check_consistent: counts / ranges must agree across layers
    c = SpliceCache(2, 1, P)
    c.append(0, ORIGIN_CLOUD, 0, 4, pages(1), layer=0)   # layer 0's frame arrived, layer 1's not yet
    msg = c.check_consistent()
    assert "layer segment counts differ" in msg
    c.append(0, ORIGIN_CLOUD, 0, 3, pages(1), layer=1)   # different length
    assert "layers cover different position ranges" in c.check_consistent()
    c2 = SpliceCache(2, 1, P)
    c2.append(0, ORIGIN_CLOUD, 0, 4, pages(1), layer=0)
    c2.append(0, ORIGIN_CLOUD, 0, 4, pages(1, 3), layer=1)  # own page ids per layer are fine
    assert c2.check_consistent() == ""


def test_plan_layout_export_matches_splice_table():
    from paper_2504_11729_b200.splice import SpliceTable
    c = SpliceCache(1, 3, P)
    t = SpliceTable(3, P)
    for b, segs in enumerate([[(0, 5), (1, 3)], [(1, 9)], [(0, 2), (1, 1), (2, 6)]]):
        pos, pg = 0, 100 * b
        for origin, n in segs:
            pl = pages(-(-n // P), pg)
            c.append(b, origin, pos, n, pl)
            t.append(b, origin, pos, n, pl)
            pos += n
            pg += pl.size
    a1, a2 = c.arrays(0), t.arrays()
    for x, y in zip(a1, a2):
        assert np.array_equal(x, y)
