"""Randomised GPU parity sweep over the shapes the reference config accepts.

Each trial draws a config (sink, local window, page size, head size, GQA
group, boost fraction, key / value bits), a ragged batch of lengths and a few
decode steps, then checks every sequence of the device cache against its own
CPU oracle cache (cache.py:83-252): page bytes bit-exact, flattened K/V
bit-exact, attention within max-abs 1e-2 (+ the bf16 rounding of outputs above
magnitude 2).  Trials alternate the product path (bf16 rows; the fused
kernels at d = g = 128) and the reference-precision path (f32 rows and f32
page metadata, generic kernels)."""

import numpy as np
import pytest
import torch

from oracle import kitty_oracle as ko

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def _close(got, want):
    return bool(np.all(np.abs(got - want) <= 1e-2 + np.abs(want) * 2.0 ** -8))


def _trial(cuda, seed):
    rng = np.random.default_rng(seed)
    fused = seed % 3 == 0
    if fused:
        g = d = 128
        s = int(rng.choice([0, 4, 32, 40]))
        r = int(rng.choice([64, 128, 200]))
    else:
        g = int(rng.choice([8, 16, 32]))
        d = int(rng.choice([8, 16, 32, 64]))
        s = int(rng.integers(0, 9))
        r = int(rng.integers(1, 40))
    group = int(rng.choice([1, 2, 4, 8]))
    h_kv = int(rng.choice([1, 2]))
    frac = float(rng.choice([0.0, 0.0625, 0.125, 0.25, 0.1]))
    cfg = cuda.KittyConfig(s=s, r=r, g=g, d=d, h_kv=h_kv, h_q=h_kv * group, boost_fraction=frac)
    b = int(rng.integers(1, 4))
    pmax = int(rng.integers(1, 6 * g + s + r))
    lens = [int(x) for x in rng.integers(0, pmax + 1, size=b)]
    lens[0] = pmax
    steps = int(rng.integers(1, 4))
    n = pmax + steps
    k = _bf16(rng.normal(0, 1, (b, h_kv, n, d)))
    k[..., rng.choice(d, max(1, d // 8), replace=False)] *= 8
    v = _bf16(rng.normal(0, 1, (b, h_kv, n, d)))
    f32 = not fused and seed % 2 == 1
    cache = cuda.KittyBatchCache(cfg, b, n + 4, row_dtype=torch.float32 if f32 else torch.bfloat16,
                                 f32_metadata=f32)
    cache.prefill(torch.from_numpy(k[:, :, :pmax]), torch.from_numpy(v[:, :, :pmax]), lengths=lens)
    ocs = []
    for bi, ln in enumerate(lens):
        oc = ko.OracleCache(s, r, g, d, h_kv, h_kv * group, frac, metadata16=not f32)
        if ln:
            oc.prefill(k[bi, :, :ln], v[bi, :, :ln])
        ocs.append(oc)
    pos = list(lens)
    for _ in range(steps):
        kn = np.stack([k[bi, :, pos[bi]] for bi in range(b)])
        vn = np.stack([v[bi, :, pos[bi]] for bi in range(b)])
        cache.append(torch.from_numpy(kn), torch.from_numpy(vn))
        for bi in range(b):
            ocs[bi].insert_token(kn[bi], vn[bi])
            pos[bi] += 1
    q = _bf16(rng.normal(0, 1, (b, h_kv * group, d)))
    out = cache.attend(torch.from_numpy(q).cuda(), out_dtype=torch.float32).cpu().numpy()
    cache.check()
    where = f"seed {seed}: s={s} r={r} g={g} d={d} group={group} h_kv={h_kv} frac={frac} lens={lens} f32={f32}"
    for bi in range(b):
        for h in range(h_kv):
            kb, vb = ocs[bi].page_bodies(h)
            ks = cache.key_page_slots(bi, h).cpu().numpy()
            vs = cache.value_page_slots(bi, h).cpu().numpy()
            assert [x.tobytes() for x in ks] == kb, where
            assert [x.tobytes() for x in vs] == vb, where
            kf, vf = cache.flatten(bi, h)
            assert np.array_equal(kf.cpu().numpy(), ocs[bi].flatten_keys(h)), where
            assert np.array_equal(vf.cpu().numpy(), ocs[bi].flatten_values(h)), where
        assert _close(out[bi], ocs[bi].attend(q[bi])), where


@pytest.mark.parametrize("seed", range(120))
def test_random_shapes_match_oracle(cuda, seed):
    _trial(cuda, seed)
