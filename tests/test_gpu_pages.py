"""GPU parity of the page codec (K1/K2/K6) through the C ABI.

Bar: bit-exact.  Device slot bytes == KTYP body of the reference page
(golden vectors from the reference; the oracle at larger sizes); dequantised
values == the reference's (f32 metadata) or the KTYP round trip (f16)."""

import numpy as np
import pytest
import torch

from oracle import kitty_oracle as ko

pytestmark = pytest.mark.gpu


def _bf16(rng, shape, outliers=(), gain=8.0):
    m = rng.normal(0.0, 1.0, size=shape).astype(np.float32)
    if len(outliers):
        m[..., list(outliers)] *= gain
    return torch.from_numpy(m).bfloat16().float().numpy()


def test_golden_pages_bit_exact(cuda, golden):
    for ci in range(int(golden["num_page_cases"][0])):
        x = golden[f"page{ci}_x"]
        d, g, db = (int(v) for v in golden[f"page{ci}_meta"])
        xt = torch.from_numpy(x).cuda()[None]
        # fused magnitude selection
        slots = cuda.pack_key_pages(xt, db)
        assert slots[0].cpu().numpy().tobytes() == golden[f"page{ci}_kbody"].tobytes(), ci
        vs = cuda.pack_value_pages(xt)
        assert vs[0].cpu().numpy().tobytes() == golden[f"page{ci}_vbody"].tobytes(), ci
        # scores and selection entry points
        sc = cuda.channel_scores_batch(xt)[0].cpu().numpy()
        assert np.array_equal(sc, golden[f"page{ci}_scores"])
        if db:
            sel = cuda.select_boost_batch(torch.from_numpy(sc).cuda()[None], db)[0].cpu().numpy()
            assert np.array_equal(sel, golden[f"page{ci}_sel"])
        # dequant from the slot (f16 metadata) == reference deserialize(serialize(page))
        kd = cuda.dequant_key_pages(slots, g, d, db)[0].cpu().numpy()
        assert np.array_equal(kd, golden[f"page{ci}_kdeq16"])
        vd = cuda.dequant_value_pages(vs, g, d)[0].cpu().numpy()
        assert np.array_equal(vd, golden[f"page{ci}_vdeq16"])
        # bf16 input path gives the same bytes (inputs are bf16-representable)
        assert cuda.pack_key_pages(xt.bfloat16(), db)[0].cpu().numpy().tobytes() == golden[f"page{ci}_kbody"].tobytes()


def test_reference_single_page_api(cuda, golden):
    for ci in range(int(golden["num_page_cases"][0])):
        x = golden[f"page{ci}_x"]
        frac = float(golden[f"page{ci}_frac"][0])
        sel = cuda.select_boost(cuda.channel_scores(x), frac)
        kp = cuda.pack_key_page(x, sel)
        assert cuda.serialize_page(kp)[11:] == golden[f"page{ci}_kbody"].tobytes()
        assert np.array_equal(cuda.dequantize_key_page(kp), golden[f"page{ci}_kdeq"])
        vp = cuda.pack_value_page(x)
        assert np.array_equal(cuda.dequantize_value_page(vp), golden[f"page{ci}_vdeq"])


def test_explicit_selection(cuda, golden):
    x = torch.from_numpy(golden["explicit_x"]).cuda()[None]
    sel = torch.from_numpy(golden["explicit_sel"])[None]
    slots = cuda.pack_key_pages(x, sel.shape[1], sel)
    assert slots[0].cpu().numpy().tobytes() == golden["explicit_kbody"].tobytes()


@pytest.mark.parametrize("frac", [0.0, 0.0625, 0.125, 0.25])
def test_many_pages_match_oracle(cuda, frac):
    # SPEC AC1 asks for >= 1000 pages; 1024 default-shape pages per fraction
    rng = np.random.default_rng(int(frac * 1000) + 1)
    pages = 1024
    x = _bf16(rng, (pages, 128, 128), rng.choice(128, 16, replace=False))
    x[7, :, 5] = 1.5  # constant channel -> scale 0
    x[9, 3, :] = x[9, 2, :]
    db = ko.boost_count(frac, 128)
    xt = torch.from_numpy(x).cuda().bfloat16()
    ks = cuda.pack_key_pages(xt, db).cpu().numpy()
    vs = cuda.pack_value_pages(xt).cpu().numpy()
    for p in list(range(16)) + list(rng.choice(pages, 48, replace=False)):
        op = ko.pack_key_page(x[p], ko.select_boost(ko.channel_scores(x[p]), frac))
        assert ks[p].tobytes() == ko.key_page_body(op), p
        assert vs[p].tobytes() == ko.value_page_body(ko.pack_value_page(x[p])), p


def test_pack_dequantize_matches_fake_quant(cuda):
    # test_pages.py:81-91 with the device codec (f32 metadata path)
    for d, g in [(4, 4), (8, 16), (64, 32), (128, 128)]:
        for fraction in (0.0, 0.125, 0.5, 1.0):
            rng = np.random.default_rng(d * 1000 + g + int(fraction * 8))
            for _ in range(3):
                x = rng.normal(0, 4, (g, d)).astype(np.float32)
                k = round(fraction * d)
                sel = cuda.BoostSelection(boosted=np.array(sorted(rng.choice(d, size=k, replace=False)), np.int64), d_boost=k)
                got = cuda.dequantize_key_page(cuda.pack_key_page(x, sel)).T
                w = np.full(d, 2)
                w[sel.boosted] = 4
                assert np.array_equal(got, ko.fake_quantize_matrix(x, "per_channel", w))


def test_value_page_matches_per_token_oracle(cuda):
    rng = np.random.default_rng(8)
    x = rng.normal(0, 3, (128, 128)).astype(np.float32)
    got = cuda.dequantize_value_page(cuda.pack_value_page(x))
    assert np.array_equal(got, ko.fake_quantize_matrix(x, "per_token", np.full(128, 2)))
    c = np.full((8, 8), -1.75, dtype=np.float32)
    assert np.array_equal(cuda.dequantize_value_page(cuda.pack_value_page(c)), c)


def test_bit_split_kat(cuda):
    # test_pages.py:48-69
    x = np.zeros((16, 4), dtype=np.float32)
    x[:, 2] = np.arange(16)
    page = cuda.pack_key_page(x, cuda.BoostSelection(boosted=np.array([2]), d_boost=1))
    low = ko.unpack2(page.dense_low)[2]
    high = ko.unpack2(page.high_bits)[0]
    assert list(low) == [c & 3 for c in range(16)]
    assert list(high) == [c >> 2 for c in range(16)]
    assert page.boost_idx[2] == 0
    assert np.array_equal(cuda.dequantize_key_page(page)[2], np.arange(16, dtype=np.float32))


def test_constant_page(cuda):
    x = np.full((8, 4), 3.25, dtype=np.float32)
    page = cuda.pack_key_page(x, cuda.BoostSelection(boosted=np.array([1]), d_boost=1))
    assert np.all(page.scales == 0.0)
    assert np.array_equal(cuda.dequantize_key_page(page), np.full((4, 8), 3.25, dtype=np.float32))


def test_sentinel_corruption_detected(cuda):
    import dataclasses

    rng = np.random.default_rng(7)
    x = rng.normal(0, 1, (8, 8)).astype(np.float32)
    page = cuda.pack_key_page(x, cuda.BoostSelection(boosted=np.array([2, 6]), d_boost=2))
    bad = page.boost_idx.copy()
    bad[2] = 255
    with pytest.raises(cuda.PageFormatError):
        cuda.dequantize_key_page(dataclasses.replace(page, boost_idx=bad))
    bad = page.boost_idx.copy()
    bad[2] = bad[6]
    with pytest.raises(cuda.PageFormatError):
        cuda.dequantize_key_page(dataclasses.replace(page, boost_idx=bad))


def test_pack_validation(cuda):
    sel0 = cuda.BoostSelection(boosted=np.zeros(0, np.int64), d_boost=0)
    with pytest.raises(cuda.KittyError):
        cuda.pack_key_page(np.zeros((6, 4), np.float32), sel0)
    with pytest.raises(cuda.KittyError):
        cuda.pack_key_page(np.zeros((4, 4), np.float32), cuda.BoostSelection(boosted=np.array([4]), d_boost=1))
    with pytest.raises(cuda.KittyError):
        cuda.pack_key_page(np.full((4, 4), np.nan, np.float32), sel0)
    with pytest.raises(cuda.KittyError):
        cuda.pack_value_page(np.zeros((4, 6), np.float32))
    with pytest.raises(cuda.KittyError):
        cuda.pack_value_page(np.full((4, 4), np.inf, np.float32))


def test_tie_breaking_on_device(cuda):
    assert list(cuda.select_boost(np.array([5.0, 1.0, 5.0, 0.0]), 0.5).boosted) == [0, 2]
    assert list(cuda.select_boost(np.array([5.0, 5.0, 5.0, 0.0]), 0.5).boosted) == [0, 1]
    rng = np.random.default_rng(7)
    for _ in range(30):
        d = int(rng.integers(1, 40))
        scores = rng.choice([0.0, 1.0, 2.0, 3.5], size=d)
        frac = float(rng.random())
        assert list(cuda.select_boost(scores, frac).boosted) == list(ko.select_boost(scores, frac))
