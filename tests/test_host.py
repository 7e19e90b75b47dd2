"""Host-side logic on CPU: the config mirror, byte accounting, KTYP wire
format, sharding plans and the algorithmic-bytes formula.  Checked against
the oracle (itself pinned to the reference) and the reference's KATs."""

import numpy as np
import pytest

import paper_2511_18643_b200 as kb
from paper_2511_18643_b200 import sharding
from oracle import kitty_oracle as ko


@pytest.mark.parametrize("kwargs", [
    dict(s=-1), dict(r=0), dict(g=6), dict(d=10), dict(h_kv=2, h_q=3), dict(key_bits=4),
    dict(value_bits=8), dict(boost_fraction=1.5), dict(heuristic="oracle"),
])
def test_config_validation(kwargs):
    # test_cache.py:32-48
    with pytest.raises(kb.ConfigError):
        kb.KittyConfig(**kwargs)


def test_config_defaults():
    cfg = kb.KittyConfig()
    assert (cfg.s, cfg.r, cfg.g, cfg.d_boost) == (32, 128, 128, 16)
    assert kb.config_from_mapping({"s": "8", "boost_fraction": "0.25"}).d_boost == 32
    with pytest.raises(kb.ConfigError):
        kb.config_from_mapping({"sink": 8})


def test_boost_count_half_even():
    for frac in (0.0, 0.0625, 0.125, 0.25, 0.3, 0.5, 1.0):
        for d in (4, 8, 10, 64, 128):
            assert kb.boost_count(frac, d) == ko.boost_count(frac, d)


def test_page_byte_size_kat():
    cfg = kb.KittyConfig()
    key = kb.page_byte_size("key", cfg)
    assert (key.payload, key.metadata, key.index, key.total) == (4608, 512, 128, 5248)
    assert kb.page_byte_size("value", cfg).total == 4608


def test_memory_report_matches_oracle_and_kat():
    rep = kb.memory_report(kb.KittyConfig(), 8192)
    assert (rep.key_page_count, rep.value_page_count, rep.total_bytes) == (63, 62, 714624)
    rng = np.random.default_rng(10)
    for _ in range(50):
        s, r, g, d = int(rng.integers(0, 8)), int(rng.integers(1, 12)), int(rng.integers(1, 5)) * 4, int(rng.integers(1, 5)) * 4
        frac = float(rng.choice([0.0, 0.125, 0.25, 1.0]))
        cfg = kb.KittyConfig(s=s, r=r, g=g, d=d, h_kv=2, h_q=2, boost_fraction=frac)
        length = int(rng.integers(0, 150))
        assert kb.memory_report(cfg, length).total_bytes == ko.memory_total_bytes(s, r, g, d, 2, cfg.d_boost, length)


def test_kv_data_ratio_approaches_8x():
    cfg = kb.KittyConfig(boost_fraction=0.0)
    assert kb.memory_report(cfg, 2**22).kv_data_ratio == pytest.approx(8.0, abs=0.05)


def test_algorithmic_bytes_match_survey_table():
    # bytes per unit at the BASELINE configs
    c = kb.KittyConfig(h_kv=8, h_q=32)
    assert kb.algorithmic_bytes_per_unit(c, 4096) == 399232 + 2048
    assert kb.algorithmic_bytes_per_unit(c, 32768) == 2606976 + 2048
    assert kb.algorithmic_bytes_per_unit(c, 131072) == 10176384 + 2048
    c5 = kb.KittyConfig(h_kv=8, h_q=64)
    assert kb.algorithmic_bytes_per_unit(c5, 16384) == 1345408 + 4096
    for frac, want in ((0.0, 682368), (0.0625, 698496), (0.125, 714624), (0.25, 746880)):
        assert kb.algorithmic_bytes_per_unit(kb.KittyConfig(h_kv=8, h_q=32, boost_fraction=frac), 8192) == want + 2048
    assert kb.algorithmic_bytes_per_unit(c, 4096) == ko.algorithmic_bytes_per_unit(32, 128, 128, 128, 16, 4, 4096)


def test_wire_format_roundtrip_against_oracle():
    rng = np.random.default_rng(9)
    x = rng.normal(0, 1, (16, 8)).astype(np.float32)
    op = ko.pack_key_page(x, [0, 3])
    raw = ko.serialize_page(op)
    page = kb.deserialize_page(raw)
    assert kb.serialize_page(page) == raw
    assert np.array_equal(page.boost_idx, op.boost_idx)
    vraw = ko.serialize_page(ko.pack_value_page(x))
    assert kb.serialize_page(kb.deserialize_page(vraw)) == vraw
    with pytest.raises(kb.BadMagicError):
        kb.deserialize_page(b"XXXX" + vraw[4:])
    with pytest.raises(kb.TruncatedFileError):
        kb.deserialize_page(vraw[:-3])
    with pytest.raises(kb.PageFormatError):
        kb.deserialize_page(vraw + b"\x00")
    assert kb.serialize_slot(raw[11:], "key", 8, 16, 2) == raw


def test_golden_bodies_roundtrip_through_wire_format(golden):
    for ci in range(int(golden["num_page_cases"][0])):
        d, g, db = (int(v) for v in golden[f"page{ci}_meta"])
        body = golden[f"page{ci}_kbody"].tobytes()
        raw = kb.serialize_slot(body, "key", d, g, db)
        assert kb.serialize_page(kb.deserialize_page(raw)) == raw


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_request_and_head_shards_partition(world):
    for batch in (1, 7, 16, 64, 256):
        seen = []
        for r in range(world):
            s = sharding.shard_by_request(batch, 8, world, r)
            seen.extend(range(s.seq_begin, s.seq_end))
            assert (s.kv_begin, s.kv_end) == (0, 8)
        assert seen == list(range(batch))
    heads = []
    for r in range(world):
        s = sharding.shard_by_kv_head(256, 8, world, r)
        heads.extend(range(s.kv_begin, s.kv_end))
    assert heads == list(range(8))
