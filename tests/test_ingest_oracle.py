"""KV ingest oracle, CPU: the C restatement of the EPKV
kv-frame decode (oracle/ep_oracle.c, wire.cpp:138-221) against the
UNMODIFIED reference codec compiled from /root/reference (oracle/_ref):
identical values and identical WireError kinds on valid, edge-case and
malformed frames; the reference test's golden header bytes; correctly
rounded f64 -> bf16."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")


def _frame(seq=70, H=4, d=64, seed=1, session=9, layer=3):
    rng = np.random.default_rng(seed)
    k = rng.uniform(-2, 2, (seq, H, d))
    v = rng.uniform(-2, 2, (seq, H, d))
    return O.kv_frame_encode(session, layer, k, v), k, v


def test_end_of_prefill_golden():
    # wire_test.cpp:52-55 ("end-of-prefill is the golden 10-byte header")
    assert list(O.end_of_prefill_frame()) == [ord("E"), ord("P"), ord("K"), ord("V"), 1, 3, 0, 0, 0, 0]


@pytest.mark.parametrize("seq,H,d", [(1, 1, 2), (70, 4, 64), (129, 8, 128)])
def test_decode_port_equals_reference(seq, H, d):
    fr, k, v = _frame(seq, H, d, seed=seq)
    for impl in ("port", "ref"):
        code, info, k2, v2 = O.kv_frame_decode(fr, impl)
        assert code == O.WIRE_OK
        assert (info.seq_len, info.n_heads, info.d_head, info.layer, info.session_id) == (seq, H, d, 3, 9)
        assert np.array_equal(k2, k) and np.array_equal(v2, v)
    assert fr.size == 10 + 14 + 16 * seq * H * d  # "expected 14 + 16 * n" (wire.cpp:192-197)


def _mutations(fr):
    out = {}
    b = fr.copy(); b[0] = ord("X"); out["bad_magic"] = b
    b = fr.copy(); b[4] = 2; out["bad_version"] = b
    out["short_header"] = fr[:7].copy()
    out["truncated_body"] = fr[:-3].copy()
    out["trailing_byte"] = np.concatenate([fr, np.zeros(1, np.uint8)])
    b = fr.copy(); b[6:10] = np.frombuffer(np.uint32((1 << 30) + 1).tobytes(), np.uint8); out["length_overflow"] = b
    b = fr.copy(); b[5] = 9; out["unknown_type"] = b
    b = fr.copy(); b[16] ^= 1; out["shape_mismatch"] = b          # seq_len no longer matches the payload
    b = fr.copy(); b[5] = 1; out["ack_typed"] = b                  # decodes as an ack -> trailing bytes
    out["payload_under_14"] = np.concatenate([fr[:6], np.frombuffer(np.uint32(5).tobytes(), np.uint8),
                                              fr[10:15]])
    out["end_of_prefill"] = O.end_of_prefill_frame()
    return out


def test_malformed_kinds_match_reference():
    fr, _, _ = _frame()
    kinds = {}
    for name, b in _mutations(fr).items():
        want = O.kv_frame_decode(b, "ref")[0]
        got = O.kv_frame_decode(b, "port")[0]
        assert got == want, (name, got, want)
        kinds[name] = got
    assert kinds["bad_magic"] == O.WIRE_BAD_MAGIC and kinds["bad_version"] == O.WIRE_BAD_VERSION
    assert kinds["truncated_body"] == O.WIRE_TRUNCATED and kinds["length_overflow"] == O.WIRE_LENGTH_OVERFLOW
    assert kinds["shape_mismatch"] == O.WIRE_MALFORMED and kinds["end_of_prefill"] == O.WIRE_NOT_KV


def _bf16_value(bits: int) -> Fraction:
    x = np.array([bits << 16], dtype=np.uint32).view(np.float32)[0]
    return Fraction(float(x))


def test_f64_to_bf16_correctly_rounded():
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.uniform(-3, 3, 600), rng.standard_normal(200) * 1e-39,
                         rng.standard_normal(100) * 1e30,
                         # exact ties between two bf16 neighbours -> even
                         np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 2 ** -140 * 1.5])])
    got = O.f64_to_bf16(xs)
    for x, g in zip(xs, got):
        g = int(g)
        fx = Fraction(float(x))
        best = abs(_bf16_value(g) - fx)
        for nb in (g - 1, g + 1):
            if 0 <= nb < 0x7F80 or 0x8000 <= nb < 0xFF80:
                dn = abs(_bf16_value(nb) - fx)
                assert dn > best or (dn == best and g % 2 == 0), (x, hex(g), hex(nb))
    assert O.f64_to_bf16([np.inf, -np.inf, 1e300])[0] == 0x7F80
    assert O.f64_to_bf16([np.nan])[0] & 0x7FC0 == 0x7FC0


def test_ingest_port_layout():
    """The port scatters frame token t / head h into pages[page_table[t//P]][h][t%P]."""
    fr, k, v = _frame(seq=130, H=2, d=64)
    pt = np.array([5, 0, 3], dtype=np.int32)
    code, info, kp, vp = O.kv_ingest(fr, O.DT_F32, 64, pt, 6)
    assert code == O.WIRE_OK
    for t in (0, 63, 64, 129):
        for h in range(2):
            assert np.array_equal(kp[pt[t // 64], h, t % 64], k[t, h].astype(np.float32))
            assert np.array_equal(vp[pt[t // 64], h, t % 64], v[t, h].astype(np.float32))
