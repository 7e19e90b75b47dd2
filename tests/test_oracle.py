"""Pin the CPU oracle (oracle/kitty_oracle.py) before trusting it.

Two anchors: the golden vectors generated from the reference itself
(tests/golden/make_golden.py) and the reference's own known-answer tests
(pkg/tests/test_quant.py, test_pages.py, test_cache.py, test_cli.py),
restated here against the oracle.
"""

import numpy as np
import pytest

from oracle import kitty_oracle as ko


# -- golden vectors from the reference ---------------------------------------


def test_pages_match_reference_golden(golden):
    for ci in range(int(golden["num_page_cases"][0])):
        x = golden[f"page{ci}_x"]
        d, g, db = (int(v) for v in golden[f"page{ci}_meta"])
        frac = float(golden[f"page{ci}_frac"][0])
        scores = ko.channel_scores(x)
        assert np.array_equal(scores, golden[f"page{ci}_scores"]), ci
        sel = ko.select_boost(scores, frac)
        assert np.array_equal(sel, golden[f"page{ci}_sel"]), ci
        kp = ko.pack_key_page(x, sel)
        vp = ko.pack_value_page(x)
        assert ko.key_page_body(kp) == golden[f"page{ci}_kbody"].tobytes(), ci
        assert ko.value_page_body(vp) == golden[f"page{ci}_vbody"].tobytes(), ci
        assert np.array_equal(ko.dequantize_key_page(kp), golden[f"page{ci}_kdeq"])
        assert np.array_equal(ko.dequantize_value_page(vp), golden[f"page{ci}_vdeq"])
        assert np.array_equal(
            ko.dequantize_key_page(ko.f16_roundtrip(kp)), golden[f"page{ci}_kdeq16"]
        )
        assert np.array_equal(
            ko.dequantize_value_page(ko.f16_roundtrip(vp)), golden[f"page{ci}_vdeq16"]
        )
        assert len(ko.key_page_body(kp)) == ko.key_slot_bytes(d, g, db)


def test_explicit_selection_matches_golden(golden):
    kp = ko.pack_key_page(golden["explicit_x"], golden["explicit_sel"])
    assert ko.key_page_body(kp) == golden["explicit_kbody"].tobytes()


@pytest.mark.parametrize("ci", range(5))
def test_cache_matches_reference_golden(golden, ci):
    s, r, g, d, h_kv, h_q, db, n = (int(v) for v in golden[f"cache{ci}_cfg"])
    frac = float(golden[f"cache{ci}_frac"][0])
    st = ko.OracleCache(s, r, g, d, h_kv, h_q, frac)
    keys, values = golden[f"cache{ci}_keys"], golden[f"cache{ci}_values"]
    for t in range(n):
        st.insert_token(keys[:, t], values[:, t])
    assert [st.key_pack_events, st.value_pack_events] == list(golden[f"cache{ci}_events"])
    for h in range(h_kv):
        kb, vb = st.page_bodies(h)
        gk, gv = golden[f"cache{ci}_h{h}_kpages"], golden[f"cache{ci}_h{h}_vpages"]
        assert len(kb) == len(gk) and len(vb) == len(gv)
        for a, b in zip(kb, gk):
            assert a == b.tobytes()
        for a, b in zip(vb, gv):
            assert a == b.tobytes()
        assert np.array_equal(st.flatten_keys(h), golden[f"cache{ci}_h{h}_flatk"])
        assert np.array_equal(st.flatten_values(h), golden[f"cache{ci}_h{h}_flatv"])
    out = st.attend(golden[f"cache{ci}_q"])
    np.testing.assert_allclose(out, golden[f"cache{ci}_out"], rtol=1e-5, atol=1e-6)
    assert ko.memory_total_bytes(s, r, g, d, h_kv, db, n) == int(golden[f"cache{ci}_total_bytes"][0])


def test_memory_kat(golden):
    c = ko.component_counts(32, 128, 128, 8192)
    assert c["key_pages"] == 63 and c["value_pages"] == 62  # test_cli.py:203-204
    assert ko.memory_total_bytes(32, 128, 128, 128, 1, 16, 8192) == 714624  # test_cli.py:205
    assert list(golden["mem8192"]) == [63, 62, 714624]


# -- the reference's own known-answer tests, restated --------------------------


def test_half_even_kat():
    # test_quant.py:128-136
    codes, scale, zero = ko.quantize_columns(np.array([[-1.0], [0.4], [1.0]], np.float32), 3.0)
    assert list(codes[:, 0]) == [0, 2, 3]
    assert zero[0] == -1.0


def test_constant_group_kat():
    # test_quant.py:121-125
    codes, scale, zero = ko.quantize_columns(np.full((3, 1), 5.0, np.float32), 15.0)
    assert scale[0] == 0.0 and zero[0] == 5.0 and list(codes[:, 0]) == [0, 0, 0]


def test_tie_break_kat():
    # test_quant.py:74-76
    assert list(ko.select_boost(np.array([5.0, 1.0, 5.0, 0.0]), 0.5)) == [0, 2]
    assert list(ko.select_boost(np.array([5.0, 5.0, 5.0, 0.0]), 0.5)) == [0, 1]
    assert ko.boost_count(0.25, 128) == 32  # test_quant.py:62-65
    assert ko.boost_count(0.125, 128) == 16


def test_select_matches_sort_oracle():
    # test_quant.py:58-59,79-87
    rng = np.random.default_rng(7)
    for _ in range(50):
        d = int(rng.integers(1, 40))
        scores = rng.choice([0.0, 1.0, 2.0, 3.5], size=d)
        frac = float(rng.random())
        want = sorted(sorted(range(d), key=lambda i: (-scores[i], i))[: round(frac * d)])
        assert list(ko.select_boost(scores, frac)) == want


def test_bit_split_kat():
    # test_pages.py:48-69
    g, d = 16, 4
    x = np.zeros((g, d), np.float32)
    x[:, 2] = np.arange(16)
    p = ko.pack_key_page(x, [2])
    low = ko.unpack2(p.dense_low)[2]
    high = ko.unpack2(p.high_bits)[0]
    assert list(low) == [c & 3 for c in range(16)]
    assert list(high) == [c >> 2 for c in range(16)]
    assert p.boost_idx[2] == 0 and all(p.boost_idx[i] == 255 for i in (0, 1, 3))
    assert np.array_equal(ko.dequantize_key_page(p)[2], np.arange(16, dtype=np.float32))


def test_pack_matches_fake_quant():
    # test_pages.py:81-91
    rng = np.random.default_rng(3)
    for d, g in [(4, 4), (8, 16), (64, 32), (128, 128)]:
        for frac in (0.0, 0.125, 0.5, 1.0):
            x = rng.normal(0, 4, (g, d)).astype(np.float32)
            sel = np.sort(rng.choice(d, size=round(frac * d), replace=False))
            w = np.full(d, 2)
            w[sel] = 4
            got = ko.dequantize_key_page(ko.pack_key_page(x, sel)).T
            assert np.array_equal(got, ko.fake_quantize_matrix(x, "per_channel", w))
    x = rng.normal(0, 3, (128, 128)).astype(np.float32)
    got = ko.dequantize_value_page(ko.pack_value_page(x))
    assert np.array_equal(got, ko.fake_quantize_matrix(x, "per_token", np.full(128, 2)))


def test_sentinel_corruption_detected():
    # test_pages.py:116-129
    rng = np.random.default_rng(7)
    p = ko.pack_key_page(rng.normal(0, 1, (8, 8)).astype(np.float32), [2, 6])
    p.boost_idx = p.boost_idx.copy()
    p.boost_idx[2] = 255
    with pytest.raises(ko.OraclePageFormatError):
        ko.dequantize_key_page(p)


def test_order_reconstruction_fuzz():
    # test_cache.py:353-375 (quantized mode: check counts and fp segments)
    rng = np.random.default_rng(13)
    for _ in range(60):
        s, r, g = int(rng.integers(0, 4)), int(rng.integers(1, 6)), int(rng.integers(1, 3)) * 4
        st = ko.OracleCache(s, r, g, 4, 1, 1)
        n = int(rng.integers(1, 40))
        for t in range(n):
            st.insert_token(np.full(4, t, np.float32), np.full(4, t + 0.5, np.float32))
        c = ko.component_counts(s, r, g, n)
        hd = st.heads[0]
        assert len(hd["kpages"]) == c["key_pages"] and len(hd["kq"]) == c["key_qbuf"]
        assert len(hd["vpages"]) == c["value_pages"] and len(hd["vq"]) == c["value_qbuf"]
        assert len(hd["local"]) == c["local"]


@pytest.mark.parametrize("s,r,g,n", [(4, 8, 8, 0), (4, 8, 8, 3), (4, 8, 8, 100), (0, 5, 4, 37), (32, 128, 128, 700), (4, 256, 128, 1004)])
def test_bulk_state_equals_fold(s, r, g, n):
    # bulk_unit_state (the closed-form state used by the long-context GPU tests)
    # must equal the fold of insert_token, page bytes and flattened rows alike
    rng = np.random.default_rng(n + s)
    d = 16 if g < 128 else 128
    k = rng.normal(0, 1, (1, n, d)).astype(np.float32)
    v = rng.normal(0, 1, (1, n, d)).astype(np.float32)
    oc = ko.OracleCache(s, r, g, d, 1, 1, 0.125, metadata16=True)
    oc.prefill(k, v)
    kf, vf, kb, vb = ko.bulk_unit_state(k[0], v[0], s, r, g, 0.125, metadata16=True)
    assert np.array_equal(kf.reshape(-1, d), oc.flatten_keys(0).reshape(-1, d))
    assert np.array_equal(vf.reshape(-1, d), oc.flatten_values(0).reshape(-1, d))
    okb, ovb = oc.page_bodies(0)
    assert kb == okb and vb == ovb
    if n:
        q = rng.normal(0, 1, (1, d)).astype(np.float32)
        np.testing.assert_array_equal(ko.attend_rows(kf, vf, q), oc.attend(q))
