"""GPU parity of the cache runtime (append K3 + fused pack, prefill) and the
decode attention (K4/K5) through the C ABI.

Bars: page bytes bit-exact vs the reference (golden) / oracle; flattened
K/V bit-exact vs the oracle with the device's f16 page metadata; attention
within max-abs 1e-2 of the reference's bf16-rounded outputs (north_star) and
within 1e-5 relative of the oracle's f32 attention on the same (f16-metadata)
pages, the reference's own tolerance (test_cache.py:231-304)."""

import numpy as np
import pytest
import torch

from oracle import kitty_oracle as ko

pytestmark = pytest.mark.gpu

SMALL = dict(s=4, r=8, g=8, d=8)


def _rel(got, want):
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30))


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def _golden_cfg(golden, ci):
    s, r, g, d, h_kv, h_q, db, n = (int(v) for v in golden[f"cache{ci}_cfg"])
    return dict(s=s, r=r, g=g, d=d, h_kv=h_kv, h_q=h_q, boost_fraction=float(golden[f"cache{ci}_frac"][0])), n


@pytest.mark.parametrize("ci", range(5))
def test_golden_cache_step_by_step(cuda, golden, ci):
    kw, n = _golden_cfg(golden, ci)
    cfg = cuda.KittyConfig(**kw)
    st = cuda.KittyCacheState(cfg, max_tokens=64)  # forces grow() for the long cases
    keys, values = golden[f"cache{ci}_keys"], golden[f"cache{ci}_values"]
    for t in range(n):
        st.insert_token(keys[:, t], values[:, t])
    assert [st.key_pack_events, st.value_pack_events] == list(golden[f"cache{ci}_events"])
    # KittyCacheState keeps the reference's precision: f32 rows, f32 page metadata
    oc = ko.OracleCache(kw["s"], kw["r"], kw["g"], kw["d"], kw["h_kv"], kw["h_q"], kw["boost_fraction"], metadata16=False)
    oc.prefill(keys, values)
    for h in range(cfg.h_kv):
        kb_, vb_ = st.export_pages(h)
        gk, gv = golden[f"cache{ci}_h{h}_kpages"], golden[f"cache{ci}_h{h}_vpages"]
        assert len(kb_) == len(gk) and len(vb_) == len(gv)
        for a, b in zip(kb_, gk):
            assert a[11:] == b.tobytes()
        for a, b in zip(vb_, gv):
            assert a[11:] == b.tobytes()
        assert np.array_equal(st.flatten_keys(h), oc.flatten_keys(h))
        assert np.array_equal(st.flatten_values(h), oc.flatten_values(h))
    q = golden[f"cache{ci}_q"]
    got = st.attend(q).outputs
    # the reference's own tolerance (test_cache.py:291-304)
    assert _rel(got, oc.attend(q)) <= 1e-5
    # north_star bar against the reference itself (f32 page metadata)
    ref = golden[f"cache{ci}_out"]
    assert np.max(np.abs(_bf16(got) - ref)) <= 1e-2


@pytest.mark.parametrize("n", [0, 3, 4, 11, 12, 13, 29, 40])
def test_prefill_equals_fold_of_inserts(cuda, n):
    # test_cache.py:108-120 on the device: bulk prefill == n appends, field by field
    cfg = cuda.KittyConfig(h_kv=2, h_q=2, **SMALL)
    rng = np.random.default_rng(n)
    k = _bf16(rng.normal(0, 1, (2, n, cfg.d)))
    v = _bf16(rng.normal(0, 1, (2, n, cfg.d)))
    bulk = cuda.KittyCacheState(cfg)
    if n:
        bulk.prefill(k, v)
    stepped = cuda.KittyCacheState(cfg)
    for t in range(n):
        stepped.insert_token(k[:, t], v[:, t])
    assert bulk.total_tokens == stepped.total_tokens == n
    assert (bulk.key_pack_events, bulk.value_pack_events) == (stepped.key_pack_events, stepped.value_pack_events)
    for h in range(2):
        assert bulk.export_pages(h) == stepped.export_pages(h)
        assert np.array_equal(bulk.flatten_keys(h), stepped.flatten_keys(h))
        assert np.array_equal(bulk.flatten_values(h), stepped.flatten_values(h))


@pytest.mark.parametrize("ci", [3, 4])
def test_prefill_default_shape_matches_reference(cuda, golden, ci):
    # d = g = 128: the bulk packer (kitty_pack_fast.cuh) against the reference's bytes
    kw, n = _golden_cfg(golden, ci)
    cfg = cuda.KittyConfig(**kw)
    for rd in (torch.bfloat16, torch.float32):  # the bulk packer (bf16 rows) and the generic one
        st = cuda.KittyCacheState(cfg, max_tokens=n, row_dtype=rd)
        st.prefill(golden[f"cache{ci}_keys"], golden[f"cache{ci}_values"])
        for h in range(cfg.h_kv):
            kb_, vb_ = st.export_pages(h)
            assert [a[11:] for a in kb_] == [b.tobytes() for b in golden[f"cache{ci}_h{h}_kpages"]]
            assert [a[11:] for a in vb_] == [b.tobytes() for b in golden[f"cache{ci}_h{h}_vpages"]]


@pytest.mark.parametrize("frac", [0.0, 0.125, 0.25])
def test_bulk_packer_matches_append_packer(cuda, frac):
    # prefill and insert_token (both on the kitty_pack_fast.cuh routines at
    # d = g = 128, the value ring wrapping) must write the oracle's bytes on
    # adversarial pages: constant
    # channels / rows (scale 0), tied channel scores, quotients at exact
    # half-integers (round-half-even), signed zeros, outliers, tiny values
    cfg = cuda.KittyConfig(s=4, r=128, g=128, d=128, h_kv=2, h_q=4, boost_fraction=frac)
    rng = np.random.default_rng(77)
    n = 4 + 3 * 128 + 128 + 9
    k = rng.normal(0, 1, (2, n, 128)).astype(np.float32)
    v = rng.normal(0, 1, (2, n, 128)).astype(np.float32)
    k[:, :, 3] = 0.75                                   # constant channel
    k[:, :, 9] = k[:, :, 10]                            # tied scores
    k[:, :, 20] = rng.integers(0, 7, (2, n))            # integer grid: (x - mn) / 2 hits .5
    k[:, :, 21] = rng.choice([-0.0, 0.0], (2, n))       # signed zeros only
    k[:, ::37, 30] = 300.0                              # outliers
    k[:, :, 40] *= 1e-30                                # tiny magnitudes
    v[:, 50, :] = -1.25                                 # constant row
    v[:, 60, :] = rng.integers(0, 7, 128)               # half-integer quotients per row
    v[:, 70, ::2] = -0.0
    k, v = _bf16(k), _bf16(v)
    bulk = cuda.KittyCacheState(cfg, max_tokens=n, row_dtype=torch.bfloat16)
    bulk.prefill(k, v)
    stepped = cuda.KittyCacheState(cfg, max_tokens=n, row_dtype=torch.bfloat16)
    for t in range(n):
        stepped.insert_token(k[:, t], v[:, t])
    for h in range(2):
        kb_, vb_ = bulk.export_pages(h)
        ks_, vs_ = stepped.export_pages(h)
        assert len(kb_) == 4 and len(vb_) == 3
        assert kb_ == ks_
        assert vb_ == vs_
    # and against the oracle's packer (pages.py:81-118, 146-162)
    oc = ko.OracleCache(4, 128, 128, 128, 2, 4, frac, metadata16=True)
    oc.prefill(k, v)
    for h in range(2):
        kb_, vb_ = bulk.export_pages(h)
        assert [a[11:] for a in kb_] == [ko.key_page_body(p) for p in oc.heads[h]["kpages"]]
        assert [a[11:] for a in vb_] == [ko.value_page_body(p) for p in oc.heads[h]["vpages"]]


@pytest.mark.parametrize("d,g", [(8, 8), (128, 128)])
def test_signed_zero_zero_points(cuda, d, g):
    # a lane whose min / max is zero stores the sign of its last zero, as
    # np.minimum.reduce does (quant.py:109); both packers, append and bulk
    cfg = cuda.KittyConfig(s=2, r=g, g=g, d=d, h_kv=1, h_q=1, boost_fraction=0.25)
    rng = np.random.default_rng(11)
    n = 2 + 3 * g + 1
    k = rng.choice(np.array([0.0, -0.0, 0.5, 1.0], np.float32), (1, n, d))
    v = rng.choice(np.array([0.0, -0.0, 0.25, -1.0], np.float32), (1, n, d))
    k[0, :, 1] = rng.choice(np.array([0.0, -0.0], np.float32), n)
    v[0, 7, :] = rng.choice(np.array([0.0, -0.0], np.float32), d)
    oc = ko.OracleCache(2, g, g, d, 1, 1, 0.25, metadata16=True)
    oc.prefill(k[0], v[0])
    for bulk in (True, False):
        st = cuda.KittyCacheState(cfg, max_tokens=n, row_dtype=torch.bfloat16)
        if bulk:
            st.prefill(k, v)
        else:
            for t in range(n):
                st.insert_token(k[:, t], v[:, t])
        kb_, vb_ = st.export_pages(0)
        assert [a[11:] for a in kb_] == [ko.key_page_body(p) for p in oc.heads[0]["kpages"]]
        assert [a[11:] for a in vb_] == [ko.value_page_body(p) for p in oc.heads[0]["vpages"]]


def test_bulk_packer_flags_nonfinite(cuda):
    cfg = cuda.KittyConfig(s=4, r=128, g=128, d=128, h_kv=1, h_q=1)
    n = 4 + 2 * 128 + 128
    rng = np.random.default_rng(5)
    for where in ("key", "value"):
        k = _bf16(rng.normal(0, 1, (1, n, 128)))
        v = _bf16(rng.normal(0, 1, (1, n, 128)))
        (k if where == "key" else v)[0, 10, 5] = np.nan if where == "key" else np.inf
        st = cuda.KittyCacheState(cfg, max_tokens=n, row_dtype=torch.bfloat16)
        with pytest.raises(cuda.KittyError):
            st.prefill(k, v)


def test_attend_after_every_step_boundary_sweep(cuda):
    # boundaries S, S+1, S+G, S+G+1, S+G+R, S+2G+R+3 (test_cache.py:231-244), quantized
    cfg = cuda.KittyConfig(h_kv=2, h_q=4, boost_fraction=0.25, **SMALL)
    rng = np.random.default_rng(31)
    length = 4 + 2 * 8 + 8 + 3
    k = _bf16(rng.normal(0, 1, (2, length, 8)))
    v = _bf16(rng.normal(0, 1, (2, length, 8)))
    q = _bf16(rng.normal(0, 1, (4, 8)))
    st = cuda.KittyCacheState(cfg)
    oc = ko.OracleCache(4, 8, 8, 8, 2, 4, 0.25, metadata16=False)
    for t in range(length):
        st.insert_token(k[:, t], v[:, t])
        oc.insert_token(k[:, t], v[:, t])
        assert _rel(st.attend(q).outputs, oc.attend(q)) <= 1e-5, t


def test_singleton_softmax(cuda):
    cfg = cuda.KittyConfig(**SMALL)
    st = cuda.KittyCacheState(cfg)
    v0 = np.arange(cfg.d, dtype=np.float32)
    st.insert_token(np.ones(cfg.d, np.float32), v0)
    assert np.array_equal(st.attend(np.ones(cfg.d, np.float32)).outputs[0], v0)


def test_attend_empty_cache_rejected(cuda):
    st = cuda.KittyCacheState(cuda.KittyConfig(**SMALL))
    with pytest.raises(cuda.KittyError):
        st.attend(np.zeros(8, np.float32))


def test_gqa_identical_queries_identical_outputs(cuda):
    cfg = cuda.KittyConfig(h_kv=2, h_q=6, **SMALL)
    st = cuda.KittyCacheState(cfg)
    rng = np.random.default_rng(10)
    st.prefill(_bf16(rng.normal(0, 1, (2, 20, 8))), _bf16(rng.normal(0, 1, (2, 20, 8))))
    q = np.tile(_bf16(rng.normal(0, 1, 8)), (6, 1))
    out = st.attend(q).outputs
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[1], out[2])
    assert np.array_equal(out[3], out[4]) and np.array_equal(out[4], out[5])
    assert not np.array_equal(out[0], out[3])


def test_per_page_selection_is_dynamic(cuda):
    # test_cache.py:194-209
    cfg = cuda.KittyConfig(s=0, r=4, g=8, d=8, boost_fraction=0.25)
    st = cuda.KittyCacheState(cfg)
    rng = np.random.default_rng(6)
    first = _bf16(rng.normal(0, 0.1, (8, 8)))
    first[:, 1] += 50
    second = _bf16(rng.normal(0, 0.1, (8, 8)))
    second[:, 6] += 50
    for t in range(8):
        st.insert_token(first[t], first[t])
    for t in range(8):
        st.insert_token(second[t], second[t])
    pages = [cuda.deserialize_page(p) for p in st.export_pages(0)[0]]
    assert pages[0].boost_idx[1] != 255 and pages[1].boost_idx[6] != 255
    assert pages[0].boost_idx[6] == 255 and pages[1].boost_idx[1] == 255


def test_order_reconstruction_fuzz(cuda):
    # test_cache.py:353-375 with the quantized device store: the flattened
    # order must equal the oracle's (token-index-encoded rows)
    rng = np.random.default_rng(13)
    for _ in range(40):
        s, r, g = int(rng.integers(0, 4)), int(rng.integers(1, 6)), int(rng.integers(1, 3)) * 4
        h_kv = int(rng.integers(1, 3))
        cfg = cuda.KittyConfig(s=s, r=r, g=g, d=4, h_kv=h_kv, h_q=h_kv)
        n = int(rng.integers(1, 40))
        p = int(rng.integers(0, n + 1))
        ks = np.tile(np.arange(n, dtype=np.float32)[None, :, None], (h_kv, 1, 4))
        ks[:, :, 1] *= -1
        vs = ks + 0.5
        st = cuda.KittyCacheState(cfg)
        oc = ko.OracleCache(s, r, g, 4, h_kv, h_kv, 0.125, metadata16=False)
        if p:
            st.prefill(ks[:, :p], vs[:, :p])
            oc.prefill(ks[:, :p], vs[:, :p])
        for t in range(p, n):
            st.insert_token(ks[:, t], vs[:, t])
            oc.insert_token(ks[:, t], vs[:, t])
        for h in range(h_kv):
            assert np.array_equal(st.flatten_keys(h), oc.flatten_keys(h))
            assert np.array_equal(st.flatten_values(h), oc.flatten_values(h))


def test_amortization_bound(cuda):
    cfg = cuda.KittyConfig(**SMALL)
    st = cuda.KittyCacheState(cfg)
    rng = np.random.default_rng(4)
    n = 10 * cfg.g
    for _ in range(n):
        st.insert_token(_bf16(rng.normal(0, 1, cfg.d)), _bf16(rng.normal(0, 1, cfg.d)))
    bound = -(-n // cfg.g) + 1
    assert st.key_pack_events <= bound and st.value_pack_events <= bound
    rep = cuda.measure_cache_bytes(st)
    assert rep == cuda.memory_report(cfg, n)


@pytest.mark.parametrize("bits", [(16, 16), (2, 16), (16, 2)])
@pytest.mark.parametrize("row_dtype", ["f32", "bf16"])
def test_passthrough_pages(cuda, bits, row_dtype):
    # key_bits / value_bits 16 (cache.py:150-153,167-170): a full group becomes a
    # page holding its rows as they are; order, attention and the pages against
    # the dense reference over the same rows
    rng = np.random.default_rng(sum(bits) + len(row_dtype))
    cfg = cuda.KittyConfig(key_bits=bits[0], value_bits=bits[1], h_kv=2, h_q=4, **SMALL)
    dt = torch.float32 if row_dtype == "f32" else torch.bfloat16
    st = cuda.KittyCacheState(cfg, max_tokens=16, row_dtype=dt)
    n = 45
    k = _bf16(rng.normal(0, 1, (2, n, cfg.d)))
    v = _bf16(rng.normal(0, 1, (2, n, cfg.d)))
    st.prefill(k[:, :20], v[:, :20])
    for t in range(20, n):
        st.insert_token(k[:, t], v[:, t])
    q = _bf16(rng.normal(0, 1, (cfg.h_q, cfg.d)))
    for h in range(2):
        kf, vf = st.flatten_keys(h), st.flatten_values(h)
        if bits[0] == 16:
            assert np.array_equal(kf, k[h])
        if bits[1] == 16:
            assert np.array_equal(vf, v[h])
        pages = st.heads[h].key_pages if bits[0] == 16 else st.heads[h].value_pages
        for i, pg in enumerate(pages):  # pass-through pages are the stored (g, d) rows
            src = k[h] if bits[0] == 16 else v[h]
            assert np.array_equal(pg, src[cfg.s + i * cfg.g: cfg.s + (i + 1) * cfg.g])
    got = st.attend(q).outputs
    want = np.stack([ko.attend_rows(st.flatten_keys(i // 2), st.flatten_values(i // 2), q[i:i + 1])[0] for i in range(4)])
    assert _rel(got, want) <= 1e-5


def test_dense_oracle_attend_on_device(cuda):
    rng = np.random.default_rng(12)
    keys = rng.normal(0, 1, (2, 300, 16)).astype(np.float32)
    values = rng.normal(0, 1, (2, 300, 16)).astype(np.float32)
    q = rng.normal(0, 1, (6, 16)).astype(np.float32)
    got = cuda.oracle_attend(keys, values, q).outputs
    assert _rel(got, ko.oracle_attend(keys, values, q)) <= 1e-5
    # test_cache.py:325-329: uniform keys -> output is the mean of the values
    k1 = np.ones((10, 4), np.float32)
    v1 = rng.normal(0, 1, (10, 4)).astype(np.float32)
    np.testing.assert_allclose(cuda.oracle_attend(k1, v1, np.ones(4, np.float32)).outputs[0], v1.mean(0), rtol=1e-5, atol=1e-6)


def _c1_like(rng, b, h_kv, h_q, n, d=128):
    outl = rng.choice(d, 16, replace=False)
    k = rng.normal(0, 1, (b, h_kv, n, d)).astype(np.float32)
    k[..., outl] *= 8
    v = rng.normal(0, 1, (b, h_kv, n, d)).astype(np.float32)
    q = rng.normal(0, 1, (b, h_q, d)).astype(np.float32)
    return _bf16(k), _bf16(v), _bf16(q)


@pytest.mark.parametrize("n,group", [(4096, 4), (1000, 8), (160, 4), (33, 4), (290, 8), (700, 1), (1500, 2)])
def test_batched_attention_default_shape_vs_oracle(cuda, n, group):
    # C1 (1 seq, 8 kv / 32 q, 4K) and ragged-page lengths; bf16 out, max-abs <= 1e-2
    rng = np.random.default_rng(n + group)
    b, h_kv = 2, 8 if n == 4096 else 2
    h_q = h_kv * group
    cfg = cuda.KittyConfig(h_kv=h_kv, h_q=h_q)
    k, v, q = _c1_like(rng, b, h_kv, h_q, n)
    cache = cuda.KittyBatchCache(cfg, b, n + 8)
    cache.prefill(torch.from_numpy(k), torch.from_numpy(v))
    # one decode step: append then attend (pack-before-attend ordering)
    kn, vn, _ = _c1_like(rng, b, h_kv, h_q, 1)
    cache.append(torch.from_numpy(kn[:, :, 0]), torch.from_numpy(vn[:, :, 0]))
    out = cache.attend(torch.from_numpy(q).cuda()).float().cpu().numpy()
    cache.check()
    for bi in range(b):
        oc = ko.OracleCache(32, 128, 128, 128, h_kv, h_q, 0.125, metadata16=False)
        oc.prefill(np.concatenate([k[bi], kn[bi]], axis=1), np.concatenate([v[bi], vn[bi]], axis=1))
        want = oc.attend(q[bi])
        assert np.max(np.abs(out[bi] - want)) <= 1e-2, bi
        oc16 = ko.OracleCache(32, 128, 128, 128, h_kv, h_q, 0.125, metadata16=True)
        oc16.prefill(np.concatenate([k[bi], kn[bi]], axis=1), np.concatenate([v[bi], vn[bi]], axis=1))
        assert np.max(np.abs(out[bi] - oc16.attend(q[bi]))) <= 1e-2


def test_decode_loop_matches_oracle(cuda):
    # simulate-decode (cli.py:304-315) on the device: prompt, then steps of
    # append + attend, crossing key and value pack boundaries
    rng = np.random.default_rng(77)
    h_kv, h_q, prompt, steps = 2, 8, 32 + 128 + 100, 40
    cfg = cuda.KittyConfig(h_kv=h_kv, h_q=h_q)
    k, v, _ = _c1_like(rng, 1, h_kv, h_q, prompt + steps)
    cache = cuda.KittyBatchCache(cfg, 1, prompt + steps)
    cache.prefill(torch.from_numpy(k[:, :, :prompt]), torch.from_numpy(v[:, :, :prompt]))
    oc = ko.OracleCache(32, 128, 128, 128, h_kv, h_q, 0.125, metadata16=True)
    oc.prefill(k[0, :, :prompt], v[0, :, :prompt])
    for t in range(prompt, prompt + steps):
        cache.append(torch.from_numpy(k[:, :, t]), torch.from_numpy(v[:, :, t]))
        oc.insert_token(k[0, :, t], v[0, :, t])
        q = _bf16(rng.normal(0, 1, (1, h_q, 128)))
        got = cache.attend(torch.from_numpy(q), out_dtype=torch.float32)[0].cpu().numpy()
        assert _rel(got, oc.attend(q[0])) <= 5e-3, t
    cache.check()
    assert cache.key_pack_events[0] == oc.key_pack_events
    assert cache.value_pack_events[0] == oc.value_pack_events


def test_merge_width_tiers(cuda):
    # the split-KV merge picks its CTA width from the partial-slot count and
    # the grid size (kitty_attention_fast.cu launch_t): 64 sequences x 8 KV
    # heads at group 2 and ~16K tokens give 1 024 (unit, row) CTAs with 33-128
    # slots each -> the 4-warp tier; sampled units against dense attention
    # over the cache's own dequantised rows
    torch.manual_seed(7)
    B, h_kv, h_q = 64, 8, 16
    lens = [16000 + 37 * (b % 9) for b in range(B)]
    cfg = cuda.KittyConfig(h_kv=h_kv, h_q=h_q)
    cache = cuda.KittyBatchCache(cfg, B, max(lens) + 8)
    k = torch.randn(B, h_kv, max(lens), 128, device="cuda").bfloat16()
    v = torch.randn(B, h_kv, max(lens), 128, device="cuda").bfloat16()
    cache.prefill(k, v, lengths=lens)
    del k, v
    q = torch.randn(B, h_q, 128).bfloat16()
    out = cache.attend(q.cuda()).float().cpu().numpy()
    cache.check()
    g = h_q // h_kv
    for b in (0, 21, 63):
        for h in (0, 5):
            kf, vf = (t.double() for t in cache.flatten(b, h))
            qq = q[b, h * g:(h + 1) * g].double().cuda()
            p = torch.softmax((qq @ kf.T) / np.sqrt(128.0), dim=-1)
            ref = (p @ vf).float().cpu().numpy()
            assert np.max(np.abs(out[b, h * g:(h + 1) * g] - ref)) <= 1e-2, (b, h)


@pytest.mark.parametrize("group", [4, 8])
def test_long_units_on_both_schedule_rules(cuda, group):
    # units of >= 512 pages take the other level split (kitty_attention_fast.cu
    # level_begin): a ragged batch straddling the switch (70 000 / 65 000 /
    # 20 000 tokens = 546 / 507 / 155 pages), attention against dense fp32
    # attention over the cache's own dequantised rows (flatten, a15)
    rng = np.random.default_rng(3 + group)
    h_kv, h_q = 1, group
    lens = [70000, 65000, 20000]
    cfg = cuda.KittyConfig(h_kv=h_kv, h_q=h_q)
    k = torch.randn(len(lens), h_kv, max(lens), 128).bfloat16()
    v = torch.randn(len(lens), h_kv, max(lens), 128).bfloat16()
    cache = cuda.KittyBatchCache(cfg, len(lens), max(lens) + 8)
    cache.prefill(k, v, lengths=lens)
    q = torch.randn(len(lens), h_q, 128).bfloat16()
    out = cache.attend(q.cuda()).float().cpu().numpy()
    cache.check()
    for bi in range(len(lens)):
        kf, vf = (t.double() for t in cache.flatten(bi, 0))
        logits = (q[bi].double().cuda() @ kf.T) / np.sqrt(128.0)
        p = torch.softmax(logits, dim=-1)
        ref = (p @ vf).float().cpu().numpy()
        assert np.max(np.abs(out[bi] - ref)) <= 1e-2, bi


@pytest.mark.parametrize("group", [4, 8])
def test_ragged_batch_matches_oracle(cuda, group):
    # a ragged batch -- every sequence has its own length,
    # page count and pack triggers -- through prefill, decode steps and attend
    rng = np.random.default_rng(11 + group)
    h_kv, h_q = 2, 2 * group
    lens = [40, 700, 1337, 2100]
    b, steps, pmax = len(lens), 3, max(lens)
    cfg = cuda.KittyConfig(h_kv=h_kv, h_q=h_q)
    k, v, _ = _c1_like(rng, b, h_kv, h_q, pmax + steps)
    cache = cuda.KittyBatchCache(cfg, b, pmax + steps + 8)
    cache.prefill(torch.from_numpy(k[:, :, :pmax]), torch.from_numpy(v[:, :, :pmax]), lengths=lens)
    ocs = []
    for bi, n in enumerate(lens):
        oc = ko.OracleCache(32, 128, 128, 128, h_kv, h_q, 0.125, metadata16=True)
        oc.prefill(k[bi, :, :n], v[bi, :, :n])
        ocs.append(oc)
    for s in range(steps):
        kn = np.stack([k[bi, :, lens[bi] + s] for bi in range(b)])
        vn = np.stack([v[bi, :, lens[bi] + s] for bi in range(b)])
        cache.append(torch.from_numpy(kn), torch.from_numpy(vn))
        for bi in range(b):
            ocs[bi].insert_token(kn[bi], vn[bi])
        q = _bf16(rng.normal(0, 1, (b, h_q, 128)))
        out = cache.attend(torch.from_numpy(q).cuda()).float().cpu().numpy()
        cache.check()
        for bi in range(b):
            assert cache.lengths[bi] == lens[bi] + s + 1
            assert np.max(np.abs(out[bi] - ocs[bi].attend(q[bi]))) <= 1e-2, (s, bi)
