"""GPU tests of the page pool and KTYP import (row 3).

The pool: key / value slots are handed out by a device free stack as pages
are packed, recorded in non-identity block tables, returned by ``retire`` and
reused by ``admit`` (continuous batching).  Every
sequence is checked against its own oracle cache (cache.py:83-252): page bytes
bit-exact, flattened K/V bit-exact, attention within max-abs 1e-2.

Import: ``export_sequence`` -> ``import_sequence`` into another row is a
byte-identical round trip (pages.py:207-292), and damaged pages raise the
reference's exceptions (BadMagicError / TruncatedFileError / PageFormatError).
"""

import numpy as np
import pytest
import torch

from oracle import kitty_oracle as ko

pytestmark = pytest.mark.gpu

H_KV, GROUP = 2, 4


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def _rows(rng, n, d=128):
    k = rng.normal(0, 1, (H_KV, n, d)).astype(np.float32)
    k[..., rng.choice(d, 16, replace=False)] *= 8
    v = rng.normal(0, 1, (H_KV, n, d)).astype(np.float32)
    return _bf16(k), _bf16(v)


def _oracle(k, v):
    oc = ko.OracleCache(32, 128, 128, 128, H_KV, H_KV * GROUP, 0.125, metadata16=True)
    if k.shape[1]:
        oc.prefill(k, v)
    return oc


def _check_seq(cache, b, oc):
    for h in range(H_KV):
        kb, vb = oc.page_bodies(h)
        ks = cache.key_page_slots(b, h).cpu().numpy()
        vs = cache.value_page_slots(b, h).cpu().numpy()
        assert len(ks) == len(kb) and len(vs) == len(vb)
        assert all(a.tobytes() == w for a, w in zip(ks, kb))
        assert all(a.tobytes() == w for a, w in zip(vs, vb))
        kf, vf = cache.flatten(b, h)
        assert np.array_equal(kf.cpu().numpy(), oc.flatten_keys(h))
        assert np.array_equal(vf.cpu().numpy(), oc.flatten_values(h))


def _close(got, want):
    """north_star's max-abs 1e-2 on bf16 outputs, plus the bf16 rounding of the
    output itself above magnitude 2 (|ref| 2^-8)."""
    return bool(np.all(np.abs(got - want) <= 1e-2 + np.abs(want) * 2.0 ** -8))


def _device_free(cache):
    torch.cuda.synchronize()
    return cache.free_top.cpu().tolist()


def test_pool_continuous_batching(cuda):
    rng = np.random.default_rng(3)
    cfg = cuda.KittyConfig(h_kv=H_KV, h_q=H_KV * GROUP)
    lens = [280, 1100, 700, 150]  # rows 0 and 3 cross key / value page boundaries below
    B = len(lens)
    cache = cuda.KittyBatchCache(cfg, B, 2048, pool_pages=40)
    seqs = [_rows(rng, 1600) for _ in range(B)]
    ocs = []
    for b, n in enumerate(lens):
        k, v = seqs[b]
        cache.admit(b, torch.from_numpy(k[:, :n]), torch.from_numpy(v[:, :n]))
        ocs.append(_oracle(k[:, :n], v[:, :n]))
    pos = list(lens)
    assert _device_free(cache) == cache.free_pages

    def step():
        kn = np.stack([seqs[b][0][:, pos[b]] for b in range(B)])
        vn = np.stack([seqs[b][1][:, pos[b]] for b in range(B)])
        cache.append(torch.from_numpy(kn), torch.from_numpy(vn))
        for b in range(B):
            ocs[b].insert_token(kn[b], vn[b])
            pos[b] += 1
        q = _bf16(rng.normal(0, 1, (B, cfg.h_q, 128)))
        out = cache.attend(torch.from_numpy(q).cuda()).float().cpu().numpy()
        cache.check()
        for b in range(B):
            assert _close(out[b], ocs[b].attend(q[b])), b

    for _ in range(3):
        step()
    # retire sequence 1 (the longest): its slots return to the pool ...
    freed_before = list(cache.free_pages)
    cache.retire(1)
    assert cache.free_pages[0] > freed_before[0]
    assert _device_free(cache) == cache.free_pages
    assert bool((cache.key_block_table[1 * H_KV:2 * H_KV] == -1).all())
    # ... and are reused by the sequence admitted into row 1
    seqs[1] = _rows(rng, 1600)
    n1 = 900
    cache.admit(1, torch.from_numpy(seqs[1][0][:, :n1]), torch.from_numpy(seqs[1][1][:, :n1]))
    ocs[1] = _oracle(seqs[1][0][:, :n1], seqs[1][1][:, :n1])
    pos[1] = n1
    # the block tables are a real indirection now: slots are not in unit order
    kbt = cache.key_block_table.cpu().numpy()
    used = [kbt[u][kbt[u] >= 0] for u in range(cache.units)]
    flat = np.concatenate(used)
    assert len(set(flat.tolist())) == len(flat), "a slot is mapped twice"
    assert not np.array_equal(flat, np.sort(flat)), "block tables are still the identity"
    # rows 0 (n = 288: key + value page) and 3 (n = 160: key page) pack from the pool
    for _ in range(20):
        step()
    for b in range(B):
        _check_seq(cache, b, ocs[b])
    assert _device_free(cache) == cache.free_pages


def test_pool_exhaustion(cuda):
    rng = np.random.default_rng(4)
    cfg = cuda.KittyConfig(h_kv=H_KV, h_q=H_KV * GROUP)
    cache = cuda.KittyBatchCache(cfg, 1, 1024, pool_pages=6)
    k, v = _rows(rng, 600)
    with pytest.raises(cuda.KittyError, match="page pool exhausted"):
        cache.admit(0, torch.from_numpy(k[:, :544]), torch.from_numpy(v[:, :544]))  # 4 key pages x 2 heads
    assert cache.lengths == [0] and _device_free(cache) == [6, 6]
    cache.admit(0, torch.from_numpy(k[:, :288]), torch.from_numpy(v[:, :288]))  # 2 key + 1 value page per head
    assert cache.free_pages == [2, 4]
    # n = 416 packs one key + one value page per head: the last key slots
    row = lambda t: (torch.from_numpy(k[None, :, t]), torch.from_numpy(v[None, :, t]))
    for t in range(288, 543):
        cache.append(*row(t))
    cache.check()
    assert cache.free_pages == [0, 2] and _device_free(cache) == [0, 2]
    with pytest.raises(cuda.KittyError, match="page pool exhausted"):
        cache.append(*row(543))  # n = 544: the next key page has no slot; nothing launched
    assert cache.lengths == [543]
    cache.retire(0)
    assert cache.free_pages == [6, 6] and _device_free(cache) == [6, 6]


def test_empty_rows_attend_to_zero(cuda):
    rng = np.random.default_rng(5)
    cfg = cuda.KittyConfig(h_kv=H_KV, h_q=H_KV * GROUP)
    cache = cuda.KittyBatchCache(cfg, 3, 1024)
    k, v = _rows(rng, 500)
    cache.admit(1, torch.from_numpy(k), torch.from_numpy(v))
    q = _bf16(rng.normal(0, 1, (3, cfg.h_q, 128)))
    out = cache.attend(torch.from_numpy(q).cuda()).float().cpu().numpy()
    cache.check()
    assert not out[0].any() and not out[2].any()
    assert _close(out[1], _oracle(k, v).attend(q[1]))
    cache.retire(1)
    with pytest.raises(cuda.KittyError):
        cache.attend(torch.from_numpy(q).cuda())


@pytest.mark.parametrize("n", [20, 160, 545, 1337])
def test_export_import_round_trip(cuda, n):
    rng = np.random.default_rng(n)
    cfg = cuda.KittyConfig(h_kv=H_KV, h_q=H_KV * GROUP)
    src = cuda.KittyBatchCache(cfg, 2, 2048)
    k, v = _rows(rng, n)
    src.admit(0, torch.from_numpy(k), torch.from_numpy(v))
    state = src.export_sequence(0)
    dst = cuda.KittyBatchCache(cfg, 3, 512, pool_pages=64)
    other_k, other_v = _rows(rng, 400)
    dst.admit(0, torch.from_numpy(other_k), torch.from_numpy(other_v))  # occupies the first slots
    dst.import_sequence(2, state)
    dst.check()
    again = dst.export_sequence(2)
    assert again["length"] == n
    for h in range(H_KV):
        assert again["heads"][h]["key_pages"] == state["heads"][h]["key_pages"]
        assert again["heads"][h]["value_pages"] == state["heads"][h]["value_pages"]
        kf0, vf0 = src.flatten(0, h)
        kf1, vf1 = dst.flatten(2, h)
        assert torch.equal(kf0, kf1) and torch.equal(vf0, vf1)
    q = _bf16(rng.normal(0, 1, (3, cfg.h_q, 128)))
    a = src.attend(torch.from_numpy(q[:2]).cuda()).float().cpu().numpy()
    b = dst.attend(torch.from_numpy(q[[2, 1, 0]]).cuda()).float().cpu().numpy()  # row 2 gets q[0]
    want = _oracle(k, v).attend(q[0])
    assert _close(a[0], want) and _close(b[2], want)
    assert np.array_equal(a[0], b[2])  # same pages, rows and query: the same kernel result
    # decoding continues on the imported sequence exactly as on the source
    kn, vn = _rows(rng, 1)
    src.append(torch.from_numpy(np.stack([kn[:, 0]] * 2)), torch.from_numpy(np.stack([vn[:, 0]] * 2)))
    dst.append(torch.from_numpy(np.stack([kn[:, 0]] * 3)), torch.from_numpy(np.stack([vn[:, 0]] * 3)))
    for h in range(H_KV):
        assert torch.equal(src.flatten(0, h)[0], dst.flatten(2, h)[0])


def test_import_rejects_damaged_pages(cuda):
    rng = np.random.default_rng(9)
    cfg = cuda.KittyConfig(h_kv=H_KV, h_q=H_KV * GROUP)
    src = cuda.KittyBatchCache(cfg, 1, 1024)
    k, v = _rows(rng, 400)
    src.admit(0, torch.from_numpy(k), torch.from_numpy(v))
    state = src.export_sequence(0)

    def damaged(fn):
        import copy

        st = copy.deepcopy(state)
        fn(st)
        return st

    dst = cuda.KittyBatchCache(cfg, 1, 1024)
    with pytest.raises(cuda.BadMagicError):
        dst.import_sequence(0, damaged(lambda s: s["heads"][0]["key_pages"].__setitem__(0, b"XTYP" + s["heads"][0]["key_pages"][0][4:])))
    with pytest.raises(cuda.TruncatedFileError):
        dst.import_sequence(0, damaged(lambda s: s["heads"][1]["value_pages"].__setitem__(0, s["heads"][1]["value_pages"][0][:-3])))
    with pytest.raises(cuda.PageFormatError):
        dst.import_sequence(0, damaged(lambda s: s["heads"][0]["key_pages"].__setitem__(1, s["heads"][0]["key_pages"][1] + b"\0")))
    # a page of another boost fraction does not fit this cache's slots
    other = cuda.KittyBatchCache(cuda.KittyConfig(h_kv=H_KV, h_q=H_KV * GROUP, boost_fraction=0.25), 1, 1024)
    other.admit(0, torch.from_numpy(k), torch.from_numpy(v))
    with pytest.raises(cuda.PageFormatError, match="does not match"):
        dst.import_sequence(0, other.export_sequence(0))
    # a broken boost-index bijection is found on the device (pages.py:128-135)
    def break_idx(s):
        raw = bytearray(s["heads"][0]["key_pages"][0])
        off = 11 + 128 * 32 + 16 * 32  # header, dense_low, high_bits -> boost_idx
        raw[off:off + 128] = bytes([255] * 128)  # no boosted channel left
        s["heads"][0]["key_pages"][0] = bytes(raw)

    fresh = cuda.KittyBatchCache(cfg, 1, 1024)
    fresh.import_sequence(0, damaged(break_idx))
    with pytest.raises(cuda.PageFormatError):
        fresh.check()
