"""Page codec: reference names (quant.py, pages.py) backed by the sm_100a kernels.

Two layers:

* batched device entry points (``pack_key_pages``, ``pack_value_pages``,
  ``dequant_key_pages``, ``dequant_value_pages``, ``channel_scores_batch``,
  ``select_boost_batch``) taking and returning CUDA tensors, asynchronous on
  the current stream -- what a serving stack calls;
* the reference's single-page functions (``pack_key_page``,
  ``dequantize_key_page``, ... pages.py:81-168; ``channel_scores``,
  ``select_boost`` quant.py:64-99) with the same arguments, return types and
  exceptions, implemented on top of the batched kernels (synchronous, like the
  reference).

Device page slots are byte-identical to the KTYP body (pages.py:207-237).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import boost_count
from .errors import BadMagicError, KittyError, PageFormatError, TruncatedFileError

SENTINEL = 255
PAGE_MAGIC = b"KTYP"
KIND_KEY, KIND_VALUE = 0, 1
_PAGE_HEADER = struct.Struct("<4sBHHH")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _device():
    if not torch.cuda.is_available():
        raise KittyError("libkitty_b200 needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.KITTY_F32
    if t.dtype == torch.bfloat16:
        return _lib.KITTY_BF16
    raise KittyError(f"pages must be float32 or bfloat16, got {t.dtype}")


def key_slot_bytes(d: int, g: int, d_boost: int) -> int:
    return int(_lib.load_library().kitty_key_slot_bytes(d, g, d_boost))


def value_slot_bytes(d: int, g: int) -> int:
    return int(_lib.load_library().kitty_value_slot_bytes(d, g))


# -- batched device API ---------------------------------------------------------


def channel_scores_batch(x: torch.Tensor) -> torch.Tensor:
    """channel_scores (quant.py:64-72) of pages x[P, G, D] -> float64 [P, D]."""
    lib = _lib.load_library()
    x = x.contiguous()
    p, g, d = x.shape
    out = torch.empty((p, d), dtype=torch.float64, device=x.device)
    _lib.check(lib.kitty_channel_scores(x.data_ptr(), _dtype_code(x), p, g, d, out.data_ptr(), _stream()),
               "channel_scores")
    return out


def select_boost_batch(scores: torch.Tensor, k: int) -> torch.Tensor:
    """select_boost magnitude (quant.py:75-99) per row -> int64 [P, k] ascending."""
    lib = _lib.load_library()
    scores = scores.to(torch.float64).contiguous()
    p, d = scores.shape
    out = torch.empty((p, k), dtype=torch.int64, device=scores.device)
    _lib.check(lib.kitty_select_boost(scores.data_ptr(), p, d, k, out.data_ptr(), _stream()), "select_boost")
    return out


def pack_key_pages(x: torch.Tensor, d_boost: int, boosted: torch.Tensor | None = None,
                   status: torch.Tensor | None = None, with_f32_metadata: bool = False):
    """Fused channel_scores -> select_boost -> pack_key_page (cache.py:155-159) for
    pages x[P, G, D] (float32 or bfloat16, CUDA).  Returns uint8 slots [P, slot]
    (KTYP key bodies) and, if asked, (scales_f32, zeros_f32) [P, D]."""
    lib = _lib.load_library()
    x = x.contiguous()
    p, g, d = x.shape
    slot = key_slot_bytes(d, g, d_boost)
    slots = torch.empty((p, slot), dtype=torch.uint8, device=x.device)
    sc = ze = None
    if with_f32_metadata:
        sc = torch.empty((p, d), dtype=torch.float32, device=x.device)
        ze = torch.empty((p, d), dtype=torch.float32, device=x.device)
    sel_ptr = None
    if boosted is not None:
        boosted = boosted.to(device=x.device, dtype=torch.int64).contiguous()
        if boosted.shape != (p, d_boost):
            raise KittyError("boosted must be [P, d_boost]")
        sel_ptr = boosted.data_ptr()
    _lib.check(
        lib.kitty_pack_key_pages(
            x.data_ptr(), _dtype_code(x), p, g, d, d_boost, sel_ptr, slots.data_ptr(), slot,
            sc.data_ptr() if sc is not None else None, ze.data_ptr() if ze is not None else None,
            status.data_ptr() if status is not None else None, _stream(),
        ),
        "pack_key_pages",
    )
    return (slots, sc, ze) if with_f32_metadata else slots


def pack_value_pages(x: torch.Tensor, status: torch.Tensor | None = None, with_f32_metadata: bool = False):
    """pack_value_page (pages.py:146-162) for pages x[P, G, D]."""
    lib = _lib.load_library()
    x = x.contiguous()
    p, g, d = x.shape
    slot = value_slot_bytes(d, g)
    slots = torch.empty((p, slot), dtype=torch.uint8, device=x.device)
    sc = ze = None
    if with_f32_metadata:
        sc = torch.empty((p, g), dtype=torch.float32, device=x.device)
        ze = torch.empty((p, g), dtype=torch.float32, device=x.device)
    _lib.check(
        lib.kitty_pack_value_pages(
            x.data_ptr(), _dtype_code(x), p, g, d, slots.data_ptr(), slot,
            sc.data_ptr() if sc is not None else None, ze.data_ptr() if ze is not None else None,
            status.data_ptr() if status is not None else None, _stream(),
        ),
        "pack_value_pages",
    )
    return (slots, sc, ze) if with_f32_metadata else slots


def dequant_key_pages(slots: torch.Tensor, g: int, d: int, d_boost: int, scales_f32=None, zeros_f32=None,
                      status: torch.Tensor | None = None) -> torch.Tensor:
    """dequantize_key_page (pages.py:121-143) for slots[P, slot] -> float32 [P, D, G]."""
    lib = _lib.load_library()
    p = slots.shape[0]
    out = torch.empty((p, d, g), dtype=torch.float32, device=slots.device)
    _lib.check(
        lib.kitty_dequant_key_pages(
            slots.data_ptr(), slots.stride(0), p, g, d, d_boost,
            scales_f32.data_ptr() if scales_f32 is not None else None,
            zeros_f32.data_ptr() if zeros_f32 is not None else None,
            out.data_ptr(), status.data_ptr() if status is not None else None, _stream(),
        ),
        "dequantize_key_page",
    )
    return out


def dequant_value_pages(slots: torch.Tensor, g: int, d: int, scales_f32=None, zeros_f32=None) -> torch.Tensor:
    """dequantize_value_page (pages.py:165-168) for slots[P, slot] -> float32 [P, G, D]."""
    lib = _lib.load_library()
    p = slots.shape[0]
    out = torch.empty((p, g, d), dtype=torch.float32, device=slots.device)
    _lib.check(
        lib.kitty_dequant_value_pages(
            slots.data_ptr(), slots.stride(0), p, g, d,
            scales_f32.data_ptr() if scales_f32 is not None else None,
            zeros_f32.data_ptr() if zeros_f32 is not None else None,
            out.data_ptr(), _stream(),
        ),
        "dequantize_value_page",
    )
    return out


# -- the reference's single-page API ---------------------------------------------


@dataclass(frozen=True)
class BoostSelection:
    """quant.py:41-54."""

    boosted: np.ndarray
    d_boost: int

    def __post_init__(self):
        idx = np.asarray(self.boosted, dtype=np.int64)
        if idx.ndim != 1 or len(idx) != self.d_boost:
            raise KittyError("boosted index list does not match d_boost")
        if len(idx) and (np.any(np.diff(idx) <= 0) or idx[0] < 0):
            raise KittyError("boosted indices must be unique and ascending")
        object.__setattr__(self, "boosted", idx)


@dataclass(frozen=True)
class QuantizedKeyPage:
    """pages.py:60-69."""

    d: int
    g: int
    d_boost: int
    dense_low: np.ndarray
    high_bits: np.ndarray
    boost_idx: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray


@dataclass(frozen=True)
class QuantizedValuePage:
    """pages.py:72-78."""

    g: int
    d: int
    codes: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray


def _freeze(*arrays):
    for a in arrays:
        a.flags.writeable = False


def _as_matrix(x, what: str) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.dtype not in (torch.float32, torch.bfloat16):
            t = t.float()
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if t.ndim != 2:
        raise KittyError(f"{what} must be a (G, D) matrix")
    return t.to(_device()).contiguous()


def _sync_status(status: torch.Tensor, what: str):
    torch.cuda.current_stream().synchronize()
    _lib.raise_status(int(status.item()) & 0xFFFFFFFF, what)


def channel_scores(x) -> np.ndarray:
    """quant.py:64-72 on the device: float64 mean |x| over tokens."""
    t = _as_matrix(x, "scores input")
    if t.shape[0] < 1:
        raise KittyError("scores need a (tokens, channels) matrix with tokens >= 1")
    return channel_scores_batch(t[None])[0].cpu().numpy()


def select_boost(scores, boost_fraction: float, heuristic: str = "magnitude", seed=None) -> BoostSelection:
    """quant.py:75-99 (magnitude heuristic on the device).  The ``random``
    heuristic draws from numpy's PCG64 stream on the host, as the reference
    does; it is an ablation baseline, not part of the device path."""
    s = np.asarray(scores, dtype=np.float64)
    d = len(s)
    k = boost_count(boost_fraction, d)
    if heuristic == "magnitude":
        if k == 0:
            return BoostSelection(boosted=np.zeros(0, np.int64), d_boost=0)
        t = torch.from_numpy(s.copy()).to(_device())[None]
        return BoostSelection(boosted=select_boost_batch(t, k)[0].cpu().numpy(), d_boost=k)
    if heuristic == "random":
        rng = np.random.default_rng(seed)
        return BoostSelection(boosted=np.sort(rng.choice(d, size=k, replace=False)), d_boost=k)
    raise KittyError(f"unknown selection heuristic {heuristic!r}")


QUANT_BITS = (2, 4)


@dataclass(frozen=True)
class QuantParams:
    """quant.py:31-37: scale / zero-point pair of one quantization group."""

    bits: int
    scale: float
    zero_point: float


def quantize_values(xs, bits: int):
    """quant.py:123-132 on the device (kitty_quantize_lanes): one group at 2 or
    4 bits -> (codes uint8, QuantParams)."""
    if bits not in QUANT_BITS:
        raise KittyError(f"bits must be one of {QUANT_BITS}, got {bits}")
    xs = np.asarray(xs, dtype=np.float32)
    if xs.ndim != 1 or xs.size == 0:
        raise KittyError("quantize_values needs a non-empty 1-D sequence")
    if not np.isfinite(xs).all():
        raise KittyError("quantize_values input must be finite")
    lib = _lib.load_library()
    dev = _device()
    xt = torch.from_numpy(np.ascontiguousarray(xs)).to(dev)
    bt = torch.tensor([bits], dtype=torch.int32, device=dev)
    codes = torch.empty(xs.size, dtype=torch.uint8, device=dev)
    sz = torch.empty(2, dtype=torch.float32, device=dev)
    _lib.check(lib.kitty_quantize_lanes(xt.data_ptr(), xs.size, 1, 0, bt.data_ptr(), codes.data_ptr(), sz.data_ptr(),
                                        sz[1:].data_ptr(), _stream()), "quantize_values")
    scale, zero = sz.cpu().numpy()
    return codes.cpu().numpy(), QuantParams(bits=bits, scale=float(scale), zero_point=float(zero))


def dequantize_values(codes, params: QuantParams) -> np.ndarray:
    """quant.py:135-143 on the device (kitty_dequantize_lanes): code * scale + zero."""
    codes = np.asarray(codes)
    qmax = 2**params.bits - 1
    if codes.size and (codes.min() < 0 or codes.max() > qmax):
        raise KittyError(f"code outside [0, {qmax}]")
    shape = codes.shape
    flat = np.ascontiguousarray(codes.reshape(-1), dtype=np.uint8)
    if flat.size == 0:
        return np.zeros(shape, np.float32)
    lib = _lib.load_library()
    dev = _device()
    ct = torch.from_numpy(flat).to(dev)
    sz = torch.tensor([params.scale, params.zero_point], dtype=torch.float32, device=dev)
    out = torch.empty(flat.size, dtype=torch.float32, device=dev)
    _lib.check(lib.kitty_dequantize_lanes(ct.data_ptr(), flat.size, 1, 0, sz.data_ptr(), sz[1:].data_ptr(),
                                          out.data_ptr(), _stream()), "dequantize_values")
    return out.cpu().numpy().reshape(shape)


def fake_quantize_matrix(x, axis: str, bits_per_lane) -> np.ndarray:
    """quant.py:145-177 on the device (kitty_fake_quantize): quantize-then-
    dequantize every lane of ``x`` -- a column for ``per_channel``, a row for
    ``per_token`` -- at its own width in {2, 4, 16} (16 passes through)."""
    lib = _lib.load_library()
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise KittyError("fake_quantize_matrix needs a 2-D matrix")
    if axis not in ("per_channel", "per_token"):
        raise KittyError(f"axis must be per_channel or per_token, got {axis!r}")
    lanes = x.shape[1] if axis == "per_channel" else x.shape[0]
    bits = np.asarray(bits_per_lane, dtype=np.int64)
    if bits.shape != (lanes,):
        raise KittyError(f"need {lanes} lane widths, got shape {bits.shape}")
    if not np.isin(bits, (2, 4, 16)).all():
        raise KittyError("lane widths must be in {2, 4, 16}")
    dev = _device()
    xt = torch.from_numpy(x).to(dev)
    bt = torch.from_numpy(bits.astype(np.int32)).to(dev)
    out = torch.empty_like(xt)
    _lib.check(lib.kitty_fake_quantize(xt.data_ptr(), x.shape[0], x.shape[1], int(axis == "per_token"),
                                       bt.data_ptr(), out.data_ptr(), _stream()), "fake_quantize_matrix")
    return out.cpu().numpy()


def split_key_body(body: np.ndarray, d: int, g: int, d_boost: int):
    """Components of a KTYP key body in declaration order (pages.py:215-221)."""
    body = np.asarray(body, dtype=np.uint8)
    o = 0
    dense = body[o: o + d * g // 4].reshape(d, g // 4); o += d * g // 4
    high = body[o: o + d_boost * g // 4].reshape(d_boost, g // 4); o += d_boost * g // 4
    idx = body[o: o + d]; o += d
    sc = body[o: o + 2 * d].view("<f2"); o += 2 * d
    ze = body[o: o + 2 * d].view("<f2")
    return dense, high, idx, sc, ze


def split_value_body(body: np.ndarray, d: int, g: int):
    body = np.asarray(body, dtype=np.uint8)
    o = 0
    codes = body[o: o + g * d // 4].reshape(g, d // 4); o += g * d // 4
    sc = body[o: o + 2 * g].view("<f2"); o += 2 * g
    ze = body[o: o + 2 * g].view("<f2")
    return codes, sc, ze


def pack_key_page(x, sel: BoostSelection) -> QuantizedKeyPage:
    """pages.py:81-118 on the device (same validation and result)."""
    t = _as_matrix(x, "key page")
    g, d = t.shape
    if g % 4 != 0 or g == 0:
        raise KittyError(f"page token count {g} must be a positive multiple of 4")
    if len(sel.boosted) and sel.boosted[-1] >= d:
        raise KittyError("boost selection indexes a channel outside the page")
    if sel.d_boost > SENTINEL:
        raise KittyError(f"d_boost {sel.d_boost} exceeds the uint8 index space")
    status = torch.zeros(1, dtype=torch.int32, device=t.device)
    boosted = torch.from_numpy(np.asarray(sel.boosted, np.int64).reshape(1, -1))
    slots, sc, ze = pack_key_pages(t[None], sel.d_boost, boosted, status, with_f32_metadata=True)
    _sync_status(status, "key page")
    body = slots[0].cpu().numpy()
    dense, high, idx, _, _ = split_key_body(body, d, g, sel.d_boost)
    dense, high, idx = dense.copy(), high.copy(), idx.copy()
    scale, zero = sc[0].cpu().numpy(), ze[0].cpu().numpy()
    _freeze(dense, high, idx, scale, zero)
    return QuantizedKeyPage(d=d, g=g, d_boost=sel.d_boost, dense_low=dense, high_bits=high,
                            boost_idx=idx, scales=scale, zero_points=zero)


def _key_body_of(page: QuantizedKeyPage) -> np.ndarray:
    return np.concatenate([
        np.asarray(page.dense_low, np.uint8).reshape(-1),
        np.asarray(page.high_bits, np.uint8).reshape(-1),
        np.asarray(page.boost_idx, np.uint8).reshape(-1),
        np.asarray(page.scales, np.float32).astype("<f2").view(np.uint8),
        np.asarray(page.zero_points, np.float32).astype("<f2").view(np.uint8),
    ])


def _value_body_of(page: QuantizedValuePage) -> np.ndarray:
    return np.concatenate([
        np.asarray(page.codes, np.uint8).reshape(-1),
        np.asarray(page.scales, np.float32).astype("<f2").view(np.uint8),
        np.asarray(page.zero_points, np.float32).astype("<f2").view(np.uint8),
    ])


def dequantize_key_page(page: QuantizedKeyPage) -> np.ndarray:
    """pages.py:121-143 (Alg. 1) on the device -> (D, G) float32; raises
    PageFormatError on a broken sentinel pattern, like the reference."""
    dev = _device()
    body = torch.from_numpy(_key_body_of(page)).to(dev)[None]
    sc = torch.from_numpy(np.ascontiguousarray(page.scales, np.float32)).to(dev)[None]
    ze = torch.from_numpy(np.ascontiguousarray(page.zero_points, np.float32)).to(dev)[None]
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    out = dequant_key_pages(body, page.g, page.d, page.d_boost, sc, ze, status)
    _sync_status(status, "key page")
    return out[0].cpu().numpy()


def pack_value_page(v) -> QuantizedValuePage:
    """pages.py:146-162 on the device."""
    t = _as_matrix(v, "value page")
    g, d = t.shape
    if d % 4 != 0 or d == 0:
        raise KittyError(f"channel count {d} must be a positive multiple of 4")
    status = torch.zeros(1, dtype=torch.int32, device=t.device)
    slots, sc, ze = pack_value_pages(t[None], status, with_f32_metadata=True)
    _sync_status(status, "value page")
    codes, _, _ = split_value_body(slots[0].cpu().numpy(), d, g)
    codes = codes.copy()
    scale, zero = sc[0].cpu().numpy(), ze[0].cpu().numpy()
    _freeze(codes, scale, zero)
    return QuantizedValuePage(g=g, d=d, codes=codes, scales=scale, zero_points=zero)


def dequantize_value_page(page: QuantizedValuePage) -> np.ndarray:
    """pages.py:165-168 on the device -> (G, D) float32."""
    dev = _device()
    body = torch.from_numpy(_value_body_of(page)).to(dev)[None]
    sc = torch.from_numpy(np.ascontiguousarray(page.scales, np.float32)).to(dev)[None]
    ze = torch.from_numpy(np.ascontiguousarray(page.zero_points, np.float32)).to(dev)[None]
    return dequant_value_pages(body, page.g, page.d, sc, ze)[0].cpu().numpy()


# -- byte accounting and the KTYP wire format (host) -------------------------------


@dataclass(frozen=True)
class PageByteCounts:
    """pages.py:172-186."""

    payload: int
    metadata: int
    index: int

    @property
    def total(self) -> int:
        return self.payload + self.metadata + self.index


def page_byte_size(kind: str, cfg) -> PageByteCounts:
    """pages.py:189-204."""
    d, g = cfg.d, cfg.g
    if kind == "key":
        return PageByteCounts(payload=d * g // 4 + cfg.d_boost * g // 4, metadata=4 * d, index=d)
    if kind == "value":
        return PageByteCounts(payload=g * d // 4, metadata=4 * g, index=0)
    raise KittyError(f"kind must be 'key' or 'value', got {kind!r}")


def serialize_page(page) -> bytes:
    """pages.py:207-237: header + the device slot layout."""
    if isinstance(page, QuantizedKeyPage):
        hdr = _PAGE_HEADER.pack(PAGE_MAGIC, KIND_KEY, page.d, page.g, page.d_boost)
        return hdr + _key_body_of(page).tobytes()
    if isinstance(page, QuantizedValuePage):
        hdr = _PAGE_HEADER.pack(PAGE_MAGIC, KIND_VALUE, page.d, page.g, 0)
        return hdr + _value_body_of(page).tobytes()
    raise KittyError(f"cannot serialize {type(page).__name__}")


def serialize_slot(body: bytes | np.ndarray, kind: str, d: int, g: int, d_boost: int = 0) -> bytes:
    """KTYP bytes of a device slot: header + memcpy of the slot."""
    k = KIND_KEY if kind == "key" else KIND_VALUE
    return _PAGE_HEADER.pack(PAGE_MAGIC, k, d, g, d_boost if k == KIND_KEY else 0) + bytes(body)


def slot_body(raw: bytes, kind: str, d: int, g: int, d_boost: int = 0) -> bytes:
    """The body of a KTYP page (pages.py:246-292 header rules) for a device slot
    of a cache with this d / g / d_boost: BadMagicError / TruncatedFileError for
    a damaged header or body, PageFormatError for trailing bytes, another kind
    or a page shape the cache does not hold."""
    if len(raw) < len(PAGE_MAGIC) or raw[:4] != PAGE_MAGIC:
        raise BadMagicError(f"bad page magic {raw[:4]!r}")
    if len(raw) < _PAGE_HEADER.size:
        raise TruncatedFileError("page truncated in header")
    _, k, pd, pg, pb = _PAGE_HEADER.unpack_from(raw)
    want = KIND_KEY if kind == "key" else KIND_VALUE
    if k != want:
        raise PageFormatError(f"expected a {kind} page, got kind {k}")
    if (pd, pg) != (d, g) or (want == KIND_KEY and pb != d_boost):
        raise PageFormatError(f"page shape (d={pd}, g={pg}, d_boost={pb}) does not match the cache "
                              f"(d={d}, g={g}, d_boost={d_boost if want == KIND_KEY else 0})")
    need = key_slot_bytes(d, g, d_boost) if want == KIND_KEY else value_slot_bytes(d, g)
    body = raw[_PAGE_HEADER.size:]
    if len(body) < need:
        raise TruncatedFileError(f"{kind} page truncated")
    if len(body) > need:
        raise PageFormatError(f"{len(body) - need} trailing bytes after {kind} page")
    return body


def deserialize_page(raw: bytes):
    """pages.py:246-292."""
    if len(raw) < len(PAGE_MAGIC) or raw[:4] != PAGE_MAGIC:
        raise BadMagicError(f"bad page magic {raw[:4]!r}")
    if len(raw) < _PAGE_HEADER.size:
        raise TruncatedFileError("page truncated in header")
    _, kind, d, g, d_boost = _PAGE_HEADER.unpack_from(raw)
    body = np.frombuffer(raw, dtype=np.uint8, offset=_PAGE_HEADER.size)
    if kind == KIND_KEY:
        need = d * g // 4 + d_boost * g // 4 + 5 * d
        if len(body) < need:
            raise TruncatedFileError("key page truncated")
        if len(body) > need:
            raise PageFormatError(f"{len(body) - need} trailing bytes after key page")
        dense, high, idx, sc, ze = split_key_body(body, d, g, d_boost)
        scales, zeros = sc.astype(np.float32), ze.astype(np.float32)
        _freeze(scales, zeros)
        return QuantizedKeyPage(d=d, g=g, d_boost=d_boost, dense_low=dense, high_bits=high,
                                boost_idx=idx, scales=scales, zero_points=zeros)
    if kind == KIND_VALUE:
        need = g * d // 4 + 4 * g
        if len(body) < need:
            raise TruncatedFileError("value page truncated")
        if len(body) > need:
            raise PageFormatError(f"{len(body) - need} trailing bytes after value page")
        codes, sc, ze = split_value_body(body, d, g)
        scales, zeros = sc.astype(np.float32), ze.astype(np.float32)
        _freeze(scales, zeros)
        return QuantizedValuePage(g=g, d=d, codes=codes, scales=scales, zero_points=zeros)
    raise PageFormatError(f"unknown page kind {kind}")
