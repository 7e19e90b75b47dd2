"""Generate golden vectors from the REFERENCE implementation (kittykv).

Run in the build container, where the read-only reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It writes ``tests/golden/golden.npz``.  The fixture pins the CPU oracle
(``oracle/kitty_oracle.py``) and, transitively, the CUDA path: the GPU tests
compare device page bytes / dequant / attention against these arrays and
against the oracle at sizes beyond the fixture.  Nothing here is imported at
run time on the GPU box.

All inputs are bf16-representable float32 (the device stores bf16 rows), so
the reference and the device see identical values.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import kittykv as kv  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (RNE) and back to float32."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def synth(rng, shape, outliers=(), gain=8.0, std=1.0):
    """SyntheticSpec-style draw (tensor_io.py:89-124): Gaussian with outlier
    channels multiplied by ``gain``; rounded to bf16."""
    m = rng.normal(0.0, std, size=shape)
    if len(outliers):
        m[..., list(outliers)] *= gain
    return bf16_round(m.astype(np.float32))


def main():
    rng = np.random.default_rng(20251118)
    g = {}

    # -- pages: (d, g, fraction) sweep incl. the default 128x128 ------------
    page_cases = []
    for d, gg in [(8, 8), (16, 32), (64, 32), (128, 128)]:
        for frac in (0.0, 0.0625, 0.125, 0.25, 1.0):
            page_cases.append((d, gg, frac))
    for ci, (d, gg, frac) in enumerate(page_cases):
        outl = rng.choice(d, size=max(1, d // 8), replace=False)
        x = synth(rng, (gg, d), outl)
        if ci % 5 == 3:
            x[:, 1] = 2.5  # a constant channel -> scale 0
            x[3, :] = x[2, :]  # duplicate rows for ties in value pages
        scores = kv.channel_scores(x)
        sel = kv.select_boost(scores, frac)
        kp = kv.pack_key_page(x, sel)
        vp = kv.pack_value_page(x)
        kraw = kv.serialize_page(kp)
        vraw = kv.serialize_page(vp)
        g[f"page{ci}_x"] = x
        g[f"page{ci}_meta"] = np.array([d, gg, sel.d_boost], np.int64)
        g[f"page{ci}_frac"] = np.array([frac])
        g[f"page{ci}_scores"] = scores
        g[f"page{ci}_sel"] = sel.boosted
        g[f"page{ci}_kbody"] = np.frombuffer(kraw[11:], np.uint8)
        g[f"page{ci}_vbody"] = np.frombuffer(vraw[11:], np.uint8)
        g[f"page{ci}_kdeq"] = kv.dequantize_key_page(kp)
        g[f"page{ci}_vdeq"] = kv.dequantize_value_page(vp)
        g[f"page{ci}_kdeq16"] = kv.dequantize_key_page(kv.deserialize_page(kraw))
        g[f"page{ci}_vdeq16"] = kv.dequantize_value_page(kv.deserialize_page(vraw))
    g["num_page_cases"] = np.array([len(page_cases)])

    # -- explicit (random) selections, like test_pages.py:81-91 ---------------
    x = synth(rng, (128, 128), rng.choice(128, 16, replace=False))
    sel = np.sort(rng.choice(128, size=24, replace=False))
    kp = kv.pack_key_page(x, kv.BoostSelection(boosted=sel, d_boost=24))
    g["explicit_x"] = x
    g["explicit_sel"] = sel
    g["explicit_kbody"] = np.frombuffer(kv.serialize_page(kp)[11:], np.uint8)

    # -- cache runs: state after n inserts + one attend ----------------------
    cache_cases = [
        dict(s=4, r=8, g=8, d=8, h_kv=2, h_q=4, boost_fraction=0.25, n=61),
        dict(s=4, r=8, g=8, d=8, h_kv=2, h_q=6, boost_fraction=0.125, n=12),
        dict(s=0, r=4, g=8, d=8, h_kv=1, h_q=1, boost_fraction=0.25, n=37),
        dict(s=32, r=128, g=128, d=128, h_kv=2, h_q=8, boost_fraction=0.125, n=32 + 3 * 128 + 50),
        dict(s=32, r=128, g=128, d=128, h_kv=1, h_q=8, boost_fraction=0.25, n=32 + 2 * 128 + 128),
    ]
    for ci, c in enumerate(cache_cases):
        n = c.pop("n")
        cfg = kv.KittyConfig(**c)
        outl = rng.choice(cfg.d, size=max(1, cfg.d // 8), replace=False)
        keys = synth(rng, (cfg.h_kv, n, cfg.d), outl)
        values = synth(rng, (cfg.h_kv, n, cfg.d))
        q = synth(rng, (cfg.h_q, cfg.d))
        st = kv.KittyCacheState(cfg)
        for t in range(n):
            st.insert_token(keys[:, t], values[:, t])
        out = st.attend(q).outputs
        g[f"cache{ci}_cfg"] = np.array(
            [cfg.s, cfg.r, cfg.g, cfg.d, cfg.h_kv, cfg.h_q, cfg.d_boost, n], np.int64
        )
        g[f"cache{ci}_frac"] = np.array([cfg.boost_fraction])
        g[f"cache{ci}_keys"] = keys
        g[f"cache{ci}_values"] = values
        g[f"cache{ci}_q"] = q
        g[f"cache{ci}_out"] = out
        g[f"cache{ci}_events"] = np.array([st.key_pack_events, st.value_pack_events], np.int64)
        for h in range(cfg.h_kv):
            head = st.heads[h]
            kb = [np.frombuffer(kv.serialize_page(p)[11:], np.uint8) for p in head.key_pages]
            vb = [np.frombuffer(kv.serialize_page(p)[11:], np.uint8) for p in head.value_pages]
            g[f"cache{ci}_h{h}_kpages"] = np.stack(kb) if kb else np.zeros((0, 0), np.uint8)
            g[f"cache{ci}_h{h}_vpages"] = np.stack(vb) if vb else np.zeros((0, 0), np.uint8)
            g[f"cache{ci}_h{h}_flatk"] = st.flatten_keys(h)
            g[f"cache{ci}_h{h}_flatv"] = st.flatten_values(h)
        rep = kv.measure_cache_bytes(st)
        g[f"cache{ci}_total_bytes"] = np.array([rep.total_bytes], np.int64)
    g["num_cache_cases"] = np.array([len(cache_cases)])

    # -- memory report KAT (test_cli.py:196-206) ------------------------------
    rep = kv.memory_report(kv.KittyConfig(), 8192)
    g["mem8192"] = np.array([rep.key_page_count, rep.value_page_count, rep.total_bytes], np.int64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
