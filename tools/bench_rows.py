"""Measurements of the SURVEY 8(f) rows beside the decode path, each against the
reference (`kittykv` from baseline/_ref) on this host's CPU:

  prefill  -- kitty_prefill (bulk packer) on a C2 layer: pages/s, HBM GB/s of
              algorithmic bytes (rows read + page bodies written) vs the measured
              peak; reference: KittyCacheState.prefill (the fold of insert_token)
              on one KV head, extrapolated per page.
  pool     -- KittyBatchCache.retire + admit of one 32K-token sequence in a full
              C2 batch (slot release + bulk prefill into recycled slots).
  import   -- export_sequence / import_sequence of one 32K-token sequence
              (KTYP pages, host header rules + device copy and index checks);
              reference: serialize_page / deserialize_page of the same pages.
  sensitivity -- channel_sensitivity (4 query heads x 64 query rows, 4096 keys,
              128 channels) and boost_sweep; reference: kittykv.analysis.

One JSON line per row.  Timings use CUDA events around the device work (after
warm-up) and time.perf_counter for the host parts.  Usage:

    python tools/bench_rows.py [--rows prefill,pool,import,sensitivity]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_18643_b200 as kb  # noqa: E402


def _ref():
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        import kittykv

        return kittykv
    except Exception:
        return None


def _peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 7672.0


def _events(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def row_prefill(kv):
    cfg = kb.KittyConfig(h_kv=8, h_q=32)
    B, n = 16, 32768
    g = torch.Generator(device="cuda").manual_seed(1)
    k = torch.randn((B, 8, n, 128), generator=g, device="cuda").bfloat16()
    v = torch.randn((B, 8, n, 128), generator=g, device="cuda").bfloat16()
    cache = kb.KittyBatchCache(cfg, B, n)

    def once():
        cache.retire(0, B)
        cache.prefill(k, v)

    t = _events(once, reps=3)
    t_retire = _events(lambda: cache.retire(0, B) or cache.prefill(k[:, :, :1], v[:, :, :1]), reps=3)
    t -= t_retire  # the timed loop re-retires; subtract a retire + 1-token prefill
    c = kb.component_counts(cfg, n)
    pages = B * 8 * (c["key_pages"] + c["value_pages"])
    bytes_alg = B * 8 * (2 * n * 128 * 2) + B * 8 * (c["key_pages"] * cache.key_slot + c["value_pages"] * cache.value_slot)
    line = {"row": "f1 bulk prefill (kitty_prefill, C2 layer: 16 x 8 units x 32K tokens)", "s_per_layer": round(t, 6),
            "pages_per_s": round(pages / t), "achieved_gbs": round(bytes_alg / t / 1e9, 1), "peak_gbs": _peak(),
            "frac": round(bytes_alg / t / 1e9 / _peak(), 3)}
    if kv is not None:
        rng = np.random.default_rng(2)
        kk = rng.standard_normal((1, 32 + 128 * 16, 128)).astype(np.float32)
        st = kv.KittyCacheState(kv.KittyConfig(h_kv=1, h_q=4))
        t0 = time.perf_counter()
        st.prefill(kk, kk)
        tr = time.perf_counter() - t0
        per_page = tr / (st.key_pack_events + st.value_pack_events)
        line["reference"] = {"s_per_page": round(per_page, 6), "pages_per_s": round(1 / per_page, 1),
                             "sample": "KittyCacheState.prefill of 2 080 tokens x 1 KV head (fold of insert_token)",
                             "cores": len(os.sched_getaffinity(0))}
        line["speedup_pages_per_s"] = round(line["pages_per_s"] * per_page, 1)
    return line


def row_pool(kv):
    cfg = kb.KittyConfig(h_kv=8, h_q=32)
    B, n = 16, 32768
    g = torch.Generator(device="cuda").manual_seed(3)
    cache = kb.KittyBatchCache(cfg, B, n)
    k = torch.randn((B, 8, n, 128), generator=g, device="cuda").bfloat16()
    cache.prefill(k, k)
    one = k[0].contiguous()
    t_ret = _events(lambda: (cache.retire(3), cache.admit(3, one, one)), reps=5)
    cache.check()
    return {"row": "f2 page pool: retire + admit of one 32K-token sequence in a full C2 batch",
            "s_retire_admit": round(t_ret, 6), "slots_recycled_per_admit": 8 * (254 + 253),
            "pool_slots": cache.pool_pages, "note": "host enqueue included (a few launches)"}


def row_import(kv):
    cfg = kb.KittyConfig(h_kv=8, h_q=32)
    n = 32768
    g = torch.Generator(device="cuda").manual_seed(4)
    src = kb.KittyBatchCache(cfg, 1, n)
    k = torch.randn((1, 8, n, 128), generator=g, device="cuda").bfloat16()
    src.prefill(k, k)
    t0 = time.perf_counter()
    state = src.export_sequence(0)
    t_exp = time.perf_counter() - t0
    dst = kb.KittyBatchCache(cfg, 1, n)
    dst.import_sequence(0, state)
    dst.check()
    times = []
    for _ in range(3):
        dst.retire(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.import_sequence(0, state)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t_imp = min(times)
    pages = sum(len(h["key_pages"]) + len(h["value_pages"]) for h in state["heads"])
    nbytes = sum(len(p) for h in state["heads"] for p in h["key_pages"] + h["value_pages"])
    line = {"row": "f3 KTYP export / import of one 32K-token sequence (8 KV heads)", "pages": pages,
            "ktyp_mb": round(nbytes / 1e6, 2), "s_export": round(t_exp, 4), "s_import": round(t_imp, 4),
            "import_pages_per_s": round(pages / t_imp)}
    if kv is not None:
        from kittykv.pages import deserialize_page

        t0 = time.perf_counter()
        for h in state["heads"]:
            for p in h["key_pages"] + h["value_pages"]:
                deserialize_page(p)
        t_ref = time.perf_counter() - t0
        line["reference"] = {"s_deserialize": round(t_ref, 4), "pages_per_s": round(pages / t_ref),
                             "sample": "kittykv.deserialize_page of the same KTYP pages (no cache insertion)"}
    return line


def row_sensitivity(kv):
    spec = kb.SyntheticSpec(tokens=4096, channels=128, outlier_channels=(3, 17, 40), outlier_gain=8.0, seed=1)
    keys = kb.generate_synthetic(spec)
    q = np.random.default_rng(2).normal(0, 1, (4, 64, 128)).astype(np.float32)
    kb.channel_sensitivity(q, keys)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = kb.channel_sensitivity(q, keys)
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    rows = kb.boost_sweep(keys, q[0], [0.0, 0.0625, 0.125, 0.25], random_draws=3)
    t_sw = time.perf_counter() - t0
    exps = 4 * 64 * 4096 * 128 * 2
    line = {"row": "f4 channel_sensitivity (4 q heads x 64 rows x 4096 keys x 128 channels, fp64) and boost_sweep",
            "s_sensitivity": round(t_dev, 4), "fp64_exps_per_s": round(exps / t_dev / 1e9, 2),
            "s_boost_sweep": round(t_sw, 4), "top3": rep.top_channels(3).tolist()}
    if kv is not None:
        from kittykv import analysis as an

        t0 = time.perf_counter()
        rr = an.channel_sensitivity(q[:1, :16], keys[:1024])  # bounded sample: 1/64 of the work
        t_ref = (time.perf_counter() - t0) * (4 * 64 * 4096) / (1 * 16 * 1024)
        t0 = time.perf_counter()
        an.boost_sweep(keys, q[0], [0.0, 0.0625, 0.125, 0.25], random_draws=3)
        t_rsw = time.perf_counter() - t0
        line["reference"] = {"s_sensitivity_extrapolated": round(t_ref, 2), "s_boost_sweep": round(t_rsw, 3),
                             "sample": "kittykv.analysis.channel_sensitivity on 1 q head x 16 rows x 1024 keys, x64"}
        line["speedup_sensitivity"] = round(t_ref / t_dev, 1)
        line["speedup_boost_sweep"] = round(t_rsw / t_sw, 1)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="prefill,pool,import,sensitivity")
    args = ap.parse_args()
    kv = _ref()
    for r in args.rows.split(","):
        fn = {"prefill": row_prefill, "pool": row_pool, "import": row_import, "sensitivity": row_sensitivity}[r]
        print(json.dumps(fn(kv)), flush=True)


if __name__ == "__main__":
    main()
