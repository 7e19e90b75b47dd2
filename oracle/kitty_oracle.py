"""CPU oracle for the Kitty decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``kittykv``
(``/root/reference/pkg/src/kittykv``) for the functions on the hot path:
quantize (scores, top-k boost selection, asymmetric quantizer), the page
codec (pack / dequantize / KTYP wire format), the per-sequence cache state
machine (insert / pack / segments) and decode attention.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import it, and only as the checker or the timed CPU reference.  The
product (``paper_2511_18643_b200``) never imports it.

Parity of this restatement is pinned against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``)
and against the reference's own known-answer tests (``tests/test_oracle.py``).

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/kittykv``).
"""

from __future__ import annotations

import struct

import numpy as np

SENTINEL = 255  # pages.py:32
PAGE_MAGIC = b"KTYP"  # pages.py:34
KIND_KEY, KIND_VALUE = 0, 1  # pages.py:35-36
_HDR = struct.Struct("<4sBHHH")  # pages.py:37
FP_BYTES = 2  # analysis.py:29


class OracleError(ValueError):
    """Raised where the reference raises KittyError (errors.py:4)."""


class OraclePageFormatError(OracleError):
    """Raised where the reference raises PageFormatError (errors.py:32)."""


# -- quant.py ---------------------------------------------------------------


def boost_count(fraction: float, channels: int) -> int:
    """quant.py:57-61: Python round() (half-even) of fraction * channels."""
    if not 0.0 <= fraction <= 1.0:
        raise OracleError("boost_fraction outside [0, 1]")
    return int(round(fraction * channels))


def channel_scores(x: np.ndarray) -> np.ndarray:
    """quant.py:64-72: mean |x| over tokens, float64.

    Restated as a sequential float64 sum over tokens in order, then a
    division by the token count (numpy's axis-0 reduction of a C-contiguous
    matrix adds rows in order).
    """
    x = np.asarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[0] < 1:
        raise OracleError("scores need a (tokens, channels) matrix")
    acc = np.zeros(x.shape[1], dtype=np.float64)
    for row in np.abs(x):
        acc += row.astype(np.float64)
    return acc / np.float64(x.shape[0])


def select_boost(scores: np.ndarray, fraction: float) -> np.ndarray:
    """quant.py:75-99 (magnitude heuristic): top-k by score, ties to the
    lower channel index, returned ascending (int64)."""
    scores = np.asarray(scores, dtype=np.float64)
    k = boost_count(fraction, len(scores))
    return select_boost_k(scores, k)


def select_boost_k(scores: np.ndarray, k: int) -> np.ndarray:
    """Rank formulation of quant.py:93: rank(i) = #{s_j > s_i} + #{j < i, s_j == s_i}."""
    s = np.asarray(scores, dtype=np.float64)
    d = len(s)
    rank = np.array(
        [int(np.sum(s > s[i])) + int(np.sum(s[:i] == s[i])) for i in range(d)], dtype=np.int64
    )
    return np.flatnonzero(rank < k).astype(np.int64)


def quantize_columns(x: np.ndarray, qmax) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """quant.py:102-116: per-column asymmetric quantizer in float32."""
    x = np.asarray(x, dtype=np.float32)
    mn = x.min(axis=0)
    mx = x.max(axis=0)
    qmax = np.broadcast_to(np.asarray(qmax, dtype=np.float32), mn.shape)
    with np.errstate(over="ignore", invalid="ignore"):
        scale = (mx - mn) / qmax
        safe = np.where(scale > 0, scale, np.float32(1.0)).astype(np.float32)
        codes = np.clip(np.rint((x - mn) / safe), 0, qmax).astype(np.uint8)
    codes[:, scale == 0] = 0
    return codes, scale.astype(np.float32), mn.astype(np.float32)


def dequantize_columns(codes, scale, zero) -> np.ndarray:
    """quant.py:119-120: code * scale + zero, multiply then add (no FMA)."""
    prod = codes.astype(np.float32) * np.asarray(scale, dtype=np.float32)
    return prod + np.asarray(zero, dtype=np.float32)


def fake_quantize_matrix(x: np.ndarray, axis: str, bits) -> np.ndarray:
    """quant.py:145-177."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    cols = x if axis == "per_channel" else x.T
    out = cols.copy()
    bits = np.asarray(bits)
    for b in (2, 4):
        sel = np.flatnonzero(bits == b)
        if len(sel) == 0:
            continue
        block = np.ascontiguousarray(cols[:, sel])
        c, s, z = quantize_columns(block, float(2**b - 1))
        out[:, sel] = dequantize_columns(c, s, z)
    return out if axis == "per_channel" else np.ascontiguousarray(out.T)


# -- pages.py ---------------------------------------------------------------


def pack2(codes: np.ndarray) -> np.ndarray:
    """pages.py:42-45: 4 codes per byte, element j at bits 2*(j % 4)."""
    codes = np.asarray(codes, dtype=np.uint8)
    c = codes.reshape(codes.shape[0], codes.shape[1] // 4, 4)
    return (c[..., 0] | (c[..., 1] << 2) | (c[..., 2] << 4) | (c[..., 3] << 6)).astype(np.uint8)


def unpack2(packed: np.ndarray) -> np.ndarray:
    """pages.py:48-52."""
    packed = np.asarray(packed, dtype=np.uint8)
    out = np.empty((packed.shape[0], packed.shape[1] * 4), dtype=np.uint8)
    for j in range(4):
        out[:, j::4] = (packed >> np.uint8(2 * j)) & np.uint8(3)
    return out


class KeyPage:
    """pages.py:60-69 (QuantizedKeyPage)."""

    def __init__(self, d, g, d_boost, dense_low, high_bits, boost_idx, scales, zeros):
        self.d, self.g, self.d_boost = d, g, d_boost
        self.dense_low, self.high_bits, self.boost_idx = dense_low, high_bits, boost_idx
        self.scales, self.zero_points = scales, zeros


class ValuePage:
    """pages.py:72-78 (QuantizedValuePage)."""

    def __init__(self, g, d, codes, scales, zeros):
        self.g, self.d = g, d
        self.codes, self.scales, self.zero_points = codes, scales, zeros


def pack_key_page(x: np.ndarray, boosted) -> KeyPage:
    """pages.py:81-118."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise OracleError("key page must be (G, D)")
    g, d = x.shape
    if g % 4 != 0 or g == 0:
        raise OracleError("G must be a positive multiple of 4")
    if not np.isfinite(x).all():
        raise OracleError("non-finite key page")
    boosted = np.asarray(boosted, dtype=np.int64)
    if len(boosted) and boosted[-1] >= d:
        raise OracleError("boost index outside page")
    k = len(boosted)
    mask = np.zeros(d, dtype=bool)
    mask[boosted] = True
    qmax = np.where(mask, np.float32(15.0), np.float32(3.0))
    codes, scale, zero = quantize_columns(x, qmax)
    codes = np.ascontiguousarray(codes.T)  # (D, G)
    dense_low = pack2(codes & np.uint8(3))
    high = pack2(codes[boosted] >> np.uint8(2)) if k else np.zeros((0, g // 4), np.uint8)
    idx = np.full(d, SENTINEL, dtype=np.uint8)
    idx[boosted] = np.arange(k, dtype=np.uint8)
    return KeyPage(d, g, k, dense_low, high, idx, scale, zero)


def dequantize_key_page(page: KeyPage) -> np.ndarray:
    """pages.py:121-143 (Alg. 1) -> (D, G) float32."""
    boosted = page.boost_idx != SENTINEL
    if int(boosted.sum()) != page.d_boost:
        raise OraclePageFormatError("sentinel count mismatch")
    rows = page.boost_idx[boosted]
    if not np.array_equal(np.sort(rows), np.arange(page.d_boost, dtype=np.uint8)):
        raise OraclePageFormatError("boost_idx is not a bijection")
    x = unpack2(page.dense_low)
    if page.d_boost:
        high = unpack2(page.high_bits)
        x[boosted] |= high[rows] << np.uint8(2)
    return dequantize_columns(x, page.scales[:, None], page.zero_points[:, None])


def pack_value_page(v: np.ndarray) -> ValuePage:
    """pages.py:146-162: per-token 2-bit quantization packed along channels."""
    v = np.ascontiguousarray(v, dtype=np.float32)
    g, d = v.shape
    if d % 4 != 0 or d == 0:
        raise OracleError("D must be a positive multiple of 4")
    if not np.isfinite(v).all():
        raise OracleError("non-finite value page")
    codes, scale, zero = quantize_columns(np.ascontiguousarray(v.T), np.float32(3.0))
    return ValuePage(g, d, pack2(codes.T), scale, zero)


def dequantize_value_page(page: ValuePage) -> np.ndarray:
    """pages.py:165-168 -> (G, D) float32."""
    return dequantize_columns(unpack2(page.codes), page.scales[:, None], page.zero_points[:, None])


def key_slot_bytes(d: int, g: int, d_boost: int) -> int:
    """pages.py:196-201: payload + 16-bit metadata + index."""
    return d * g // 4 + d_boost * g // 4 + 4 * d + d


def value_slot_bytes(d: int, g: int) -> int:
    """pages.py:202-203."""
    return g * d // 4 + 4 * g


def serialize_page(page) -> bytes:
    """pages.py:207-237 (KTYP)."""
    if isinstance(page, KeyPage):
        hdr = _HDR.pack(PAGE_MAGIC, KIND_KEY, page.d, page.g, page.d_boost)
        return b"".join(
            (
                hdr,
                page.dense_low.tobytes(),
                page.high_bits.tobytes(),
                page.boost_idx.tobytes(),
                np.asarray(page.scales, np.float32).astype("<f2").tobytes(),
                np.asarray(page.zero_points, np.float32).astype("<f2").tobytes(),
            )
        )
    hdr = _HDR.pack(PAGE_MAGIC, KIND_VALUE, page.d, page.g, 0)
    return b"".join(
        (
            hdr,
            page.codes.tobytes(),
            np.asarray(page.scales, np.float32).astype("<f2").tobytes(),
            np.asarray(page.zero_points, np.float32).astype("<f2").tobytes(),
        )
    )


def deserialize_page(raw: bytes):
    """pages.py:246-292 (f16 metadata promoted to f32)."""
    if len(raw) < 4 or raw[:4] != PAGE_MAGIC:
        raise OracleError("bad magic")
    if len(raw) < _HDR.size:
        raise OracleError("truncated header")
    _, kind, d, g, db = _HDR.unpack_from(raw)
    body = np.frombuffer(raw, dtype=np.uint8, offset=_HDR.size)
    if kind == KIND_KEY:
        need = key_slot_bytes(d, g, db)
        if len(body) < need:
            raise OracleError("truncated key page")
        if len(body) > need:
            raise OraclePageFormatError("trailing bytes")
        return key_page_from_body(body, d, g, db)
    if kind == KIND_VALUE:
        need = value_slot_bytes(d, g)
        if len(body) < need:
            raise OracleError("truncated value page")
        if len(body) > need:
            raise OraclePageFormatError("trailing bytes")
        return value_page_from_body(body, d, g)
    raise OraclePageFormatError("unknown kind")


def key_page_from_body(body: np.ndarray, d: int, g: int, db: int) -> KeyPage:
    """Split a KTYP key body (pages.py:215-221 component order)."""
    body = np.asarray(body, dtype=np.uint8)
    o = 0
    dense = body[o : o + d * g // 4].reshape(d, g // 4); o += d * g // 4
    high = body[o : o + db * g // 4].reshape(db, g // 4); o += db * g // 4
    idx = body[o : o + d]; o += d
    sc = body[o : o + 2 * d].view("<f2").astype(np.float32); o += 2 * d
    ze = body[o : o + 2 * d].view("<f2").astype(np.float32)
    return KeyPage(d, g, db, dense, high, idx, sc, ze)


def value_page_from_body(body: np.ndarray, d: int, g: int) -> ValuePage:
    """Split a KTYP value body (pages.py:228-235 component order)."""
    body = np.asarray(body, dtype=np.uint8)
    o = 0
    codes = body[o : o + g * d // 4].reshape(g, d // 4); o += g * d // 4
    sc = body[o : o + 2 * g].view("<f2").astype(np.float32); o += 2 * g
    ze = body[o : o + 2 * g].view("<f2").astype(np.float32)
    return ValuePage(g, d, codes, sc, ze)


def key_page_body(page: KeyPage) -> bytes:
    return serialize_page(page)[_HDR.size :]


def value_page_body(page: ValuePage) -> bytes:
    return serialize_page(page)[_HDR.size :]


def f16_roundtrip(page):
    """deserialize(serialize(page)): the page as the device sees it (f16 metadata)."""
    return deserialize_page(serialize_page(page))


# -- analysis.py: occupancy closed form and byte accounting --------------------


def component_counts(s: int, r: int, g: int, length: int) -> dict:
    """analysis.py:301-315."""
    sink = min(length, s)
    past = max(0, length - s)
    kp, kq = divmod(past, g)
    local = min(r, past)
    vp, vq = divmod(past - local, g)
    return dict(sink=sink, key_pages=kp, key_qbuf=kq, local=local, value_pages=vp, value_qbuf=vq)


def memory_total_bytes(s, r, g, d, h_kv, d_boost, length) -> int:
    """analysis.py:318-350 total_bytes for key_bits = value_bits = 2."""
    c = component_counts(s, r, g, length)
    fp_row = d * FP_BYTES * h_kv
    key = c["key_pages"] * key_slot_bytes(d, g, d_boost) * h_kv
    val = c["value_pages"] * value_slot_bytes(d, g) * h_kv
    fp = (2 * c["sink"] + c["key_qbuf"] + c["local"] + c["value_qbuf"]) * fp_row
    return key + val + fp


# -- cache.py: the state machine and attention ---------------------------------


class OracleCache:
    """cache.py:83-252 restated: one sequence, h_kv heads, key/value bits 2.

    ``metadata16`` selects what the quantized pages contribute to attention:
    False reproduces the reference (f32 scale/zero, cache.py:161,174); True
    uses the KTYP-rounded f16 metadata the device stores.
    """

    def __init__(self, s, r, g, d, h_kv, h_q, boost_fraction=0.125, metadata16=False):
        if h_q % h_kv:
            raise OracleError("h_q must be a multiple of h_kv")
        self.s, self.r, self.g, self.d = s, r, g, d
        self.h_kv, self.h_q = h_kv, h_q
        self.fraction = boost_fraction
        self.metadata16 = metadata16
        self.total = 0
        self.key_pack_events = 0
        self.value_pack_events = 0
        self.heads = [
            dict(ksink=[], vsink=[], kq=[], vq=[], local=[], kpages=[], vpages=[], kpaged=[], vpaged=[])
            for _ in range(h_kv)
        ]

    def insert_token(self, k_new, v_new):
        """cache.py:107-123 (pack runs inside insert, before any attend)."""
        k_new = np.asarray(k_new, np.float32).reshape(self.h_kv, self.d)
        v_new = np.asarray(v_new, np.float32).reshape(self.h_kv, self.d)
        in_sink = self.total < self.s
        for h, kr, vr in zip(self.heads, k_new, v_new):
            if in_sink:
                h["ksink"].append(kr.copy())
                h["vsink"].append(vr.copy())
            else:
                h["kq"].append(kr.copy())
                if len(h["local"]) == self.r:
                    h["vq"].append(h["local"].pop(0))
                h["local"].append(vr.copy())
        self.maybe_pack()
        self.total += 1

    def prefill(self, keys, values):
        """cache.py:125-142: the fold of insert_token."""
        keys = np.asarray(keys, np.float32).reshape(self.h_kv, -1, self.d)
        values = np.asarray(values, np.float32).reshape(self.h_kv, -1, self.d)
        for t in range(keys.shape[1]):
            self.insert_token(keys[:, t], values[:, t])

    def maybe_pack(self):
        """cache.py:144-178 (trigger on head 0, magnitude heuristic)."""
        if len(self.heads[0]["kq"]) == self.g:
            for h in self.heads:
                block = np.stack(h["kq"])
                sel = select_boost(channel_scores(block), self.fraction)
                page = pack_key_page(block, sel)
                h["kpages"].append(page)
                shown = f16_roundtrip(page) if self.metadata16 else page
                h["kpaged"].append(np.ascontiguousarray(dequantize_key_page(shown).T))
                h["kq"].clear()
            self.key_pack_events += 1
        if len(self.heads[0]["vq"]) == self.g:
            for h in self.heads:
                block = np.stack(h["vq"])
                page = pack_value_page(block)
                h["vpages"].append(page)
                shown = f16_roundtrip(page) if self.metadata16 else page
                h["vpaged"].append(dequantize_value_page(shown))
                h["vq"].clear()
            self.value_pack_events += 1

    def flatten_keys(self, h=0) -> np.ndarray:
        """cache.py:196-212: sink | pages | q-buffer."""
        hd = self.heads[h]
        parts = [np.zeros((0, self.d), np.float32)] + hd["ksink"] + hd["kpaged"] + hd["kq"]
        return np.concatenate([np.atleast_2d(p) for p in parts], axis=0)

    def flatten_values(self, h=0) -> np.ndarray:
        """cache.py:202-215: sink | pages | q-buffer | local."""
        hd = self.heads[h]
        parts = (
            [np.zeros((0, self.d), np.float32)] + hd["vsink"] + hd["vpaged"] + hd["vq"] + hd["local"]
        )
        return np.concatenate([np.atleast_2d(p) for p in parts], axis=0)

    def attend(self, q) -> np.ndarray:
        """cache.py:217-252: per KV head, fp32 logits / sqrt(d), stable softmax,
        probabilities times values segment by segment."""
        if self.total == 0:
            raise OracleError("attend on an empty cache")
        q = np.asarray(q, np.float32).reshape(self.h_q, self.d)
        group = self.h_q // self.h_kv
        sqrt_d = np.float32(np.sqrt(self.d))
        out = np.empty((self.h_q, self.d), np.float32)
        for h in range(self.h_kv):
            keys = self.flatten_keys(h)
            values = self.flatten_values(h)
            qg = q[h * group : (h + 1) * group]
            logits = (keys @ qg.T) / sqrt_d
            p = softmax_columns(logits)
            out[h * group : (h + 1) * group] = p.T @ values
        return out

    def page_bodies(self, h=0):
        """KTYP bodies of the pages of head h (what a device slot must equal)."""
        hd = self.heads[h]
        return [key_page_body(p) for p in hd["kpages"]], [value_page_body(p) for p in hd["vpages"]]


def bulk_unit_state(keys, values, s, r, g, boost_fraction=0.125, metadata16=True):
    """The state one KV head holds after the fold of insert_token over ``keys`` /
    ``values`` (n, d) (cache.py:107-142), built directly from the occupancy
    closed form (analysis.py:301-315) instead of token by token: key pages
    are rows [s + i g, s + (i + 1) g) packed with their own magnitude
    selection (cache.py:155-161), value pages the same rows of the values
    (cache.py:168-174: the value q-buffer receives tokens in order once they
    leave the local window).  Returns (flat_keys, flat_values, key_bodies,
    value_bodies); the flattened rows follow cache.py:196-215.  For long
    contexts (10^5 tokens) where the per-token fold is too slow; the fold's
    equality with this is checked in tests/test_oracle.py."""
    keys = np.asarray(keys, np.float32)
    values = np.asarray(values, np.float32)
    n, d = keys.shape
    c = component_counts(s, r, g, n)
    kp, vp = c["key_pages"], c["value_pages"]
    kflat, vflat, kb, vb = [keys[: c["sink"]]], [values[: c["sink"]]], [], []
    for i in range(kp):
        block = keys[s + i * g : s + (i + 1) * g]
        page = pack_key_page(block, select_boost(channel_scores(block), boost_fraction))
        kb.append(key_page_body(page))
        shown = f16_roundtrip(page) if metadata16 else page
        kflat.append(np.ascontiguousarray(dequantize_key_page(shown).T))
    kflat.append(keys[s + kp * g :])
    for i in range(vp):
        page = pack_value_page(values[s + i * g : s + (i + 1) * g])
        vb.append(value_page_body(page))
        shown = f16_roundtrip(page) if metadata16 else page
        vflat.append(dequantize_value_page(shown))
    vflat.append(values[s + vp * g :])
    return np.concatenate(kflat, axis=0), np.concatenate(vflat, axis=0), kb, vb


def attend_rows(keys, values, qg) -> np.ndarray:
    """cache.py:240-248 for one KV head: qg (group, d) against flattened rows."""
    sqrt_d = np.float32(np.sqrt(keys.shape[1]))
    logits = (np.asarray(keys, np.float32) @ np.asarray(qg, np.float32).T) / sqrt_d
    return softmax_columns(logits).T @ np.asarray(values, np.float32)


def softmax_columns(logits: np.ndarray) -> np.ndarray:
    """cache.py:255-258."""
    shifted = logits - logits.max(axis=0, keepdims=True)
    e = np.exp(shifted, dtype=np.float32)
    return e / e.sum(axis=0, keepdims=True)


def oracle_attend(keys, values, queries, kv_head_map=None) -> np.ndarray:
    """cache.py:261-301: dense fp32 attention, floor-rule GQA map."""
    keys = np.asarray(keys, np.float32)
    values = np.asarray(values, np.float32)
    queries = np.atleast_2d(np.asarray(queries, np.float32))
    if keys.ndim == 2:
        keys, values = keys[None], values[None]
    h_kv, length, d = keys.shape
    n_q = queries.shape[0]
    if kv_head_map is None:
        kv_head_map = [i * h_kv // n_q for i in range(n_q)]
    sqrt_d = np.float32(np.sqrt(d))
    out = np.empty((n_q, d), np.float32)
    for i, qv in enumerate(queries):
        logits = (keys[kv_head_map[i]] @ qv) / sqrt_d
        p = softmax_columns(logits[:, None])[:, 0]
        out[i] = p @ values[kv_head_map[i]]
    return out


def algorithmic_bytes_per_unit(s, r, g, d, d_boost, group, n) -> int:
    """SURVEY.md §8(d) byte formula for one (seq, kv-head, layer) attend at n tokens:
    pages at 16-bit metadata + fp rows at 2 B + bf16 q read and out write."""
    c = component_counts(s, r, g, n)
    key = c["key_pages"] * key_slot_bytes(d, g, d_boost)
    val = c["value_pages"] * value_slot_bytes(d, g)
    fp = 2 * d * ((c["sink"] + c["key_qbuf"]) + (c["sink"] + c["local"] + c["value_qbuf"]))
    return key + val + fp + 2 * 2 * group * d


# -- analysis.py: channel sensitivity and boost sweeps ---------------------------


def _softmax_rows64(logits: np.ndarray) -> np.ndarray:
    """analysis.py:32-35."""
    shifted = logits - logits.max(axis=-1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=-1, keepdims=True)


def channel_sensitivity(queries, keys, bits: int = 2) -> np.ndarray:
    """analysis.py:63-104 (the mse matrix only): per query head and key
    channel, the MSE between baseline and rank-1-perturbed fp64 attention
    probabilities when that channel alone is fake-quantized at ``bits``."""
    queries = np.asarray(queries, np.float32)
    keys = np.asarray(keys, np.float32)
    queries = queries[None] if queries.ndim == 2 else queries
    keys = keys[None] if keys.ndim == 2 else keys
    h_q, _, d = queries.shape
    h_kv = keys.shape[0]
    mse = np.zeros((h_q, d), np.float64)
    if bits == 16:
        return mse
    inv = 1.0 / np.sqrt(d)
    group = h_q // h_kv
    for kv in range(h_kv):
        k64 = keys[kv].astype(np.float64)
        delta = fake_quantize_matrix(keys[kv], "per_channel", np.full(d, bits)).astype(np.float64) - k64
        for j in range(group):
            qh = kv * group + j
            q64 = queries[qh].astype(np.float64)
            base = (q64 @ k64.T) * inv
            base_p = _softmax_rows64(base)
            for ch in range(d):
                p = _softmax_rows64(base + np.outer(q64[:, ch], delta[:, ch]) * inv)
                mse[qh, ch] = np.mean((p - base_p) ** 2)
    return mse


def attention_mse(keys, queries, selection) -> float:
    """analysis.py:119-142."""
    keys = np.asarray(keys, np.float32)
    queries = np.asarray(queries, np.float32)
    queries = queries[None] if queries.ndim == 2 else queries
    d = keys.shape[1]
    widths = np.full(d, 2)
    widths[np.asarray(selection, dtype=np.int64)] = 4
    quantized = fake_quantize_matrix(keys, "per_channel", widths).astype(np.float64)
    k64 = keys.astype(np.float64)
    inv = 1.0 / np.sqrt(d)
    total = 0.0
    for q in queries:
        q64 = q.astype(np.float64)
        total += np.mean((_softmax_rows64((q64 @ quantized.T) * inv) - _softmax_rows64((q64 @ k64.T) * inv)) ** 2)
    return total / len(queries)
