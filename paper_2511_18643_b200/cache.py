"""Cache runtime on the device: the batched Kitty KV store and the decode step.

``KittyBatchCache`` is the product surface: B sequences x h_kv KV heads whose
pages live in HBM (layout: include/kitty_b200.h, KittyCacheDesc).  One decode
step is ``append`` (insert_token + maybe_pack, cache.py:107-178) followed by
``attend`` (cache.py:217-252); both are single asynchronous launches on the
current stream and can be captured in a CUDA graph.

``KittyCacheState`` keeps the reference's single-sequence class name and
methods (cache.py:83-252) on top of a batch of one, so tests written against
``kittykv`` run unchanged: it keeps the reference's precision -- float32 rows
and float32 page metadata (a side table beside the f16 KTYP slots) -- on the
generic device kernels, and exposes the reference's per-head state
(``heads[h].key_sink`` ... ``value_pages``) read back from the device.  The
batched product path (``KittyBatchCache`` default) stores bf16 rows and runs
the fused decode kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import PASSTHROUGH_BITS, KittyConfig
from .errors import KittyError
from .pages import _device, _stream, key_slot_bytes, serialize_slot, value_slot_bytes


@dataclass(frozen=True)
class AttentionOutput:
    """cache.py:33-38."""

    outputs: np.ndarray
    probs: np.ndarray | None = None


def component_counts(cfg: KittyConfig, length: int) -> dict:
    """Occupancy of every component after ``length`` tokens (analysis.py:301-315)."""
    sink = min(length, cfg.s)
    past = max(0, length - cfg.s)
    kp, kq = divmod(past, cfg.g)
    local = min(cfg.r, past)
    vp, vq = divmod(past - local, cfg.g)
    return dict(sink=sink, key_pages=kp, key_qbuf=kq, local=local, value_pages=vp, value_qbuf=vq)


def _check_device_config(cfg: KittyConfig):
    if cfg.heuristic != "magnitude":
        raise KittyError("the device pack path implements the magnitude heuristic only")


class KittyBatchCache:
    """B sequences of Kitty KV cache for one attention layer, resident in HBM.

    Pages live in a shared **page pool** (PagedAttention-style,
    PAPER.md:371-374,392-396): ``key_pool`` / ``value_pool`` hold
    ``pool_pages`` KTYP slots each, a device free stack per side hands a slot
    to every page as it is packed (append / prefill / import, inside the
    kernel: no host round trip, CUDA-graph safe), and each unit's block table
    maps its page index to the slot.  ``retire`` returns a finished sequence's
    slots and ``admit`` prefills a new one into the freed row (continuous
    batching).  ``pool_pages=None`` sizes the pool for every sequence at
    ``max_tokens`` and lets it grow; an explicit budget is fixed and an append /
    prefill that would need more slots raises ``KittyError`` before launching.
    """

    def __init__(self, cfg: KittyConfig, num_seqs: int, max_tokens: int, device=None,
                 row_dtype: torch.dtype = torch.bfloat16, f32_metadata: bool = False,
                 pool_pages: int | None = None):
        """``row_dtype``: bf16 (the fused decode path) or float32 (the reference's
        precision, generic kernels); ``f32_metadata``: keep each page's float32
        scale / zero (the reference's in-memory values) beside its f16 slot;
        ``pool_pages``: slots per side (None = units x pages at max_tokens, growable)."""
        _check_device_config(cfg)
        if row_dtype not in (torch.bfloat16, torch.float32):
            raise KittyError("row_dtype must be torch.bfloat16 or torch.float32")
        self.row_dtype = row_dtype
        self.f32_metadata = bool(f32_metadata)
        self.lib = _lib.load_library()
        _lib.check(self.lib.kitty_validate_config(ctypes.byref(cfg.to_c())), "config")
        self.cfg = cfg
        self.num_seqs = int(num_seqs)
        self.device = torch.device(device) if device is not None else _device()
        self.units = self.num_seqs * cfg.h_kv
        # a 2-bit page slot is its KTYP body; a pass-through (16-bit) page slot
        # holds the block's g rows in the row dtype (cache.py:150-153,167-170)
        rows = cfg.g * cfg.d * (4 if row_dtype == torch.float32 else 2)
        self.key_slot = rows if cfg.key_bits == PASSTHROUGH_BITS else key_slot_bytes(cfg.d, cfg.g, cfg.d_boost)
        self.value_slot = rows if cfg.value_bits == PASSTHROUGH_BITS else value_slot_bytes(cfg.d, cfg.g)
        self.lengths = [0] * self.num_seqs  # host mirror of unit_len (no syncs needed)
        self.key_pack_events = [0] * self.num_seqs
        self.value_pack_events = [0] * self.num_seqs
        self.auto_pool = pool_pages is None
        if pool_pages is not None and int(pool_pages) < 0:
            raise KittyError("pool_pages must be >= 0")
        self._alloc(max_tokens, None if pool_pages is None else int(pool_pages))
        self._ws = None

    # -- storage -------------------------------------------------------------

    def _pages_for(self, max_tokens: int) -> int:
        return max(1, -(-max(0, int(max_tokens) - self.cfg.s) // self.cfg.g))

    def _alloc(self, max_tokens: int, pool_pages: int | None):
        cfg, dev, u = self.cfg, self.device, self.units
        self.max_tokens = int(max_tokens)
        self.max_pages = self._pages_for(self.max_tokens)
        slots = u * self.max_pages if pool_pages is None else pool_pages
        bf = self.row_dtype
        self.unit_len = torch.zeros(u, dtype=torch.int32, device=dev)
        self.k_sink = torch.zeros((u, cfg.s, cfg.d), dtype=bf, device=dev)
        self.v_sink = torch.zeros((u, cfg.s, cfg.d), dtype=bf, device=dev)
        self.k_qbuf = torch.zeros((u, cfg.g, cfg.d), dtype=bf, device=dev)
        self.v_ring = torch.zeros((u, cfg.r + cfg.g, cfg.d), dtype=bf, device=dev)
        self.key_block_table = torch.full((u, self.max_pages), -1, dtype=torch.int32, device=dev)
        self.value_block_table = torch.full((u, self.max_pages), -1, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self._alloc_pool(slots)

    def _alloc_pool(self, slots: int):
        cfg, dev = self.cfg, self.device
        self.pool_pages = int(slots)
        self.key_pool = torch.zeros((max(1, slots), self.key_slot), dtype=torch.uint8, device=dev)
        self.value_pool = torch.zeros((max(1, slots), self.value_slot), dtype=torch.uint8, device=dev)
        # free stacks: pops take the top, so slot 0 is handed out first
        self.key_free = torch.arange(slots - 1, -1, -1, dtype=torch.int32, device=dev)
        self.value_free = self.key_free.clone()
        self.free_top = torch.full((2,), slots, dtype=torch.int32, device=dev)
        self.free_pages = [slots, slots]  # host mirror of free_top
        if self.f32_metadata:
            self.key_meta = torch.zeros((max(1, slots), 2 * cfg.d), dtype=torch.float32, device=dev)
            self.value_meta = torch.zeros((max(1, slots), 2 * cfg.g), dtype=torch.float32, device=dev)
        else:
            self.key_meta = self.value_meta = None
        self._build_desc()

    def _build_desc(self):
        d = _lib.KittyCacheDesc()
        d.cfg = self.cfg.to_c()
        d.num_seqs = self.num_seqs
        d.max_pages = self.max_pages
        d.key_slot_bytes = self.key_slot
        d.value_slot_bytes = self.value_slot
        d.unit_len = self.unit_len.data_ptr()
        d.k_sink = self.k_sink.data_ptr()
        d.v_sink = self.v_sink.data_ptr()
        d.k_qbuf = self.k_qbuf.data_ptr()
        d.v_ring = self.v_ring.data_ptr()
        d.key_pool = self.key_pool.data_ptr()
        d.value_pool = self.value_pool.data_ptr()
        d.key_block_table = self.key_block_table.data_ptr()
        d.value_block_table = self.value_block_table.data_ptr()
        d.status = self.status.data_ptr()
        d.row_dtype = _lib.KITTY_F32 if self.row_dtype == torch.float32 else _lib.KITTY_BF16
        d.key_meta = self.key_meta.data_ptr() if self.key_meta is not None else None
        d.value_meta = self.value_meta.data_ptr() if self.value_meta is not None else None
        d.key_free = self.key_free.data_ptr()
        d.value_free = self.value_free.data_ptr()
        d.free_top = self.free_top.data_ptr()
        d.key_slots = self.pool_pages
        d.value_slots = self.pool_pages
        self.desc = d
        self._desc_ref = ctypes.byref(d)

    def _check_movable(self):
        if getattr(self, "captured", False):
            raise KittyError("this cache is referenced by a captured CUDA graph: its buffers cannot be "
                             "reallocated (size it for the whole decode before capturing)")

    def grow(self, max_tokens: int):
        """Longer sequences: widen the block tables (int32 per page; slots and
        rows stay where they are).  An auto-sized pool also gains the slots the
        new length needs -- the one path that copies page bytes."""
        self._check_movable()
        old_mp = self.max_pages
        self.max_tokens = int(max_tokens)
        self.max_pages = self._pages_for(self.max_tokens)
        if self.max_pages > old_mp:
            for name in ("key_block_table", "value_block_table"):
                t = getattr(self, name)
                nt = torch.full((self.units, self.max_pages), -1, dtype=torch.int32, device=self.device)
                nt[:, :old_mp] = t
                setattr(self, name, nt)
        if self.auto_pool and self.units * self.max_pages > self.pool_pages:
            self._grow_pool(self.units * self.max_pages)
        self._build_desc()
        self._ws = None

    def _grow_pool(self, slots: int):
        self._check_movable()
        old = dict(kp=self.key_pool, vp=self.value_pool, kf=self.key_free, vf=self.value_free,
                   km=self.key_meta, vm=self.value_meta, n=self.pool_pages, free=list(self.free_pages))
        self._alloc_pool(slots)
        n = old["n"]
        self.key_pool[:n] = old["kp"][:n]
        self.value_pool[:n] = old["vp"][:n]
        if self.f32_metadata:
            self.key_meta[:n] = old["km"][:n]
            self.value_meta[:n] = old["vm"][:n]
        added = torch.arange(slots - 1, n - 1, -1, dtype=torch.int32, device=self.device)
        for side, (stack, ostack) in enumerate(((self.key_free, old["kf"]), (self.value_free, old["vf"]))):
            top = old["free"][side]
            stack[: slots - n] = added
            stack[slots - n: slots - n + top] = ostack[:top]
            self.free_pages[side] = top + slots - n
        self.free_top.copy_(torch.tensor(self.free_pages, dtype=torch.int32))

    def _reserve(self, key_pages: int, value_pages: int):
        """Host-side admission control: the pool must hold the pages the next
        launch packs (the host mirror of the stacks is exact: page counts follow
        from the lengths)."""
        if key_pages <= self.free_pages[0] and value_pages <= self.free_pages[1]:
            return
        if self.auto_pool:
            short = max(key_pages - self.free_pages[0], value_pages - self.free_pages[1])
            self._grow_pool(self.pool_pages + max(short, self.pool_pages // 2, 1))
            self._build_desc()
            return
        raise KittyError(f"page pool exhausted: {key_pages} key / {value_pages} value pages needed, "
                         f"{self.free_pages[0]} / {self.free_pages[1]} free of {self.pool_pages}")

    def _page_pair(self, n: int):
        c = component_counts(self.cfg, n)
        return c["key_pages"], c["value_pages"]

    def workspace(self, max_tokens: int) -> torch.Tensor:
        need = int(self.lib.kitty_attention_workspace_bytes(self._desc_ref, max_tokens))
        if self._ws is None or self._ws.numel() < need:
            # zeroed: the fused kernel keeps self-resetting work counters at its head
            self._ws = torch.zeros(max(need, 16), dtype=torch.uint8, device=self.device)
        return self._ws

    # -- decode step -----------------------------------------------------------

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor):
        """Step 1 + step 3 for every sequence: k_new/v_new [B, h_kv, D] bf16.
        Every row appends (a retired row restarts from its sink)."""
        cfg = self.cfg
        if max(self.lengths) + 1 > self.max_tokens:
            self.grow(max(2 * self.max_tokens, max(self.lengths) + 1))
        need = self.append_page_need()
        self._reserve(*need)
        k_new = self._rows(k_new, (self.num_seqs, cfg.h_kv, cfg.d), "k_new")
        v_new = self._rows(v_new, (self.num_seqs, cfg.h_kv, cfg.d), "v_new")
        _lib.check(self.lib.kitty_append(self._desc_ref, k_new.data_ptr(), v_new.data_ptr(), _stream()), "append")
        self.advance_host(need)

    def append_packs(self):
        """Which sequences' next append packs a key / a value page (two lists of
        bools): the host mirror of the device's pack triggers and slot pops.
        One pass per decode step (``DecodeStep`` shares it across its layers)."""
        S, R, G = self.cfg.s, self.cfg.r, self.cfg.g
        kpk, vpk = [], []
        for n in self.lengths:
            past = n + 1 - S
            kpk.append(past > 0 and past % G == 0)
            vtot = past - R
            vpk.append(vtot > 0 and vtot % G == 0)
        return kpk, vpk

    def append_page_need(self, packs=None):
        """(key, value) pages the next append packs."""
        kpk, vpk = self.append_packs() if packs is None else packs
        return sum(kpk) * self.cfg.h_kv, sum(vpk) * self.cfg.h_kv

    def advance_host(self, need=None, packs=None):
        """Host mirror after one append launch (eager or graph replay)."""
        packs = self.append_packs() if packs is None else packs
        need = self.append_page_need(packs) if need is None else need
        self.free_pages[0] -= need[0]
        self.free_pages[1] -= need[1]
        self.lengths = [x + 1 for x in self.lengths]
        if need[0]:
            self.key_pack_events = [e + p for e, p in zip(self.key_pack_events, packs[0])]
        if need[1]:
            self.value_pack_events = [e + p for e, p in zip(self.value_pack_events, packs[1])]

    def prefill(self, keys: torch.Tensor, values: torch.Tensor, lengths=None):
        """cache.py:125-142 for an empty batch: keys/values [B, h_kv, P, D].

        ``lengths`` (optional, one per sequence, each <= P) makes the batch
        ragged: sequence b gets the first lengths[b] tokens of its rows, and
        every later append / attend works on its own length (the device reads
        the per-unit lengths; pack triggers are per sequence)."""
        if any(self.lengths):
            raise KittyError("prefill requires an empty state")
        cfg = self.cfg
        p = keys.shape[2]
        if lengths is None:
            lengths = [p] * self.num_seqs
        lengths = [int(x) for x in lengths]
        if len(lengths) != self.num_seqs or min(lengths) < 0 or max(lengths) > p:
            raise KittyError(f"lengths must be {self.num_seqs} values in [0, {p}]")
        if max(lengths) > self.max_tokens:
            self.grow(max(lengths))
        keys = self._rows(keys, (self.num_seqs, cfg.h_kv, p, cfg.d), "keys")
        values = self._rows(values, (self.num_seqs, cfg.h_kv, p, cfg.d), "values")
        if all(x == p for x in lengths):
            kp, vp = self._page_pair(p)
            self._reserve(kp * self.units, vp * self.units)
            _lib.check(self.lib.kitty_prefill(self._desc_ref, keys.data_ptr(), values.data_ptr(), p, _stream()), "prefill")
            self.free_pages[0] -= kp * self.units
            self.free_pages[1] -= vp * self.units
            for b in range(self.num_seqs):
                self._set_length(b, p)
        else:
            for b, n in enumerate(lengths):
                if n:
                    self.prefill_range(b, 1, keys[b:b + 1, :, :n], values[b:b + 1, :, :n])

    def prefill_range(self, b0: int, nb: int, keys: torch.Tensor, values: torch.Tensor):
        """kitty_prefill of the empty sequences [b0, b0 + nb) through a
        sub-descriptor that aliases this batch's buffers (keys/values
        [nb, h_kv, P, D] bf16 on the device): the host length mirror and the
        pack-event counters of those sequences become P."""
        cfg = self.cfg
        if any(self.lengths[b0:b0 + nb]):
            raise KittyError("prefill requires empty sequences")
        if keys.shape[2] > self.max_tokens:
            self.grow(keys.shape[2])
        kp, vp = self._page_pair(keys.shape[2])
        self._reserve(kp * nb * cfg.h_kv, vp * nb * cfg.h_kv)
        u0 = b0 * cfg.h_kv
        d = _lib.KittyCacheDesc()
        ctypes.memmove(ctypes.byref(d), ctypes.byref(self.desc), ctypes.sizeof(d))
        d.num_seqs = nb
        d.unit_len = self.unit_len[u0:].data_ptr()
        d.k_sink = self.k_sink[u0:].data_ptr()
        d.v_sink = self.v_sink[u0:].data_ptr()
        d.k_qbuf = self.k_qbuf[u0:].data_ptr()
        d.v_ring = self.v_ring[u0:].data_ptr()
        d.key_block_table = self.key_block_table[u0:].data_ptr()
        d.value_block_table = self.value_block_table[u0:].data_ptr()
        # both contiguous copies must be alive when the launch is enqueued: a
        # temporary freed before its consumer is enqueued can be handed to the
        # next allocation on the same stream (after the enqueue, stream order
        # makes reuse safe)
        kc, vc = keys.contiguous(), values.contiguous()
        _lib.check(self.lib.kitty_prefill(ctypes.byref(d), kc.data_ptr(), vc.data_ptr(), keys.shape[2], _stream()),
                   "prefill")
        self.free_pages[0] -= kp * nb * cfg.h_kv
        self.free_pages[1] -= vp * nb * cfg.h_kv
        for b in range(b0, b0 + nb):
            self._set_length(b, keys.shape[2])

    def _set_length(self, b: int, n: int):
        """Host mirror after a prefill of n tokens: the pack events of the fold
        of n inserts (one per full key / value page, cache.py:144-178)."""
        cfg = self.cfg
        past = max(0, n - cfg.s)
        self.lengths[b] = n
        self.key_pack_events[b] = past // cfg.g
        self.value_pack_events[b] = max(0, past - cfg.r) // cfg.g

    # -- continuous batching: retire / admit rows of the batch -----------------

    def retire(self, b: int, nb: int = 1):
        """Free sequences [b, b + nb): their slots return to the pool, the rows
        become empty (attend writes zeros for them) and can admit new ones."""
        if b < 0 or nb < 0 or b + nb > self.num_seqs:
            raise KittyError(f"sequences [{b}, {b + nb}) outside the batch of {self.num_seqs}")
        _lib.check(self.lib.kitty_release_sequences(self._desc_ref, b, nb, _stream()), "retire")
        for i in range(b, b + nb):
            kp, vp = self._page_pair(self.lengths[i])
            self.free_pages[0] += kp * self.cfg.h_kv
            self.free_pages[1] += vp * self.cfg.h_kv
            self.lengths[i] = 0
            self.key_pack_events[i] = self.value_pack_events[i] = 0

    def admit(self, b: int, keys: torch.Tensor, values: torch.Tensor):
        """Prefill a new sequence into the empty row b: keys/values [h_kv, P, D]."""
        cfg = self.cfg
        keys = self._rows(keys, (cfg.h_kv, keys.shape[1], cfg.d), "keys")[None]
        values = self._rows(values, (cfg.h_kv, keys.shape[2], cfg.d), "values")[None]
        self.prefill_range(b, 1, keys, values)

    def attend(self, q: torch.Tensor, out: torch.Tensor | None = None, out_dtype=torch.bfloat16) -> torch.Tensor:
        """Step 2 for every sequence: q [B, h_q, D] bf16 -> [B, h_q, D] (zeros
        for empty rows of the batch)."""
        cfg = self.cfg
        if max(self.lengths) == 0:
            raise KittyError("attend on an empty cache")
        q = self._rows(q, (self.num_seqs, cfg.h_q, cfg.d), "q")
        if out is None:
            out = torch.empty((self.num_seqs, cfg.h_q, cfg.d), dtype=out_dtype, device=self.device)
        code = _lib.KITTY_F32 if out.dtype == torch.float32 else _lib.KITTY_BF16
        max_tokens = max(self.lengths)
        ws = self.workspace(max_tokens)
        _lib.check(
            self.lib.kitty_decode_attention(self._desc_ref, q.data_ptr(), out.data_ptr(), code, max_tokens,
                                            ws.data_ptr(), ws.numel(), _stream()),
            "attend",
        )
        return out

    def check(self):
        """Synchronise and raise for any data-dependent error a kernel reported
        since the last check.  The status word is cleared when read, so one
        failed step does not poison later ones."""
        torch.cuda.current_stream().synchronize()
        word = int(self.status.item()) & 0xFFFFFFFF
        if word:
            self.status.zero_()
        _lib.raise_status(word, "cache")

    def _rows(self, t, shape, what):
        if not isinstance(t, torch.Tensor):
            t = torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32))
        if tuple(t.shape) != tuple(shape):
            raise KittyError(f"{what} must have shape {tuple(shape)}, got {tuple(t.shape)}")
        return t.to(device=self.device, dtype=self.row_dtype).contiguous()

    # -- readout ------------------------------------------------------------------

    def flatten(self, b: int, h: int):
        """flatten_keys / flatten_values (cache.py:210-215) -> float32 [n, D] each."""
        n = self.lengths[b]
        u = b * self.cfg.h_kv + h
        ko = torch.empty((n, self.cfg.d), dtype=torch.float32, device=self.device)
        vo = torch.empty((n, self.cfg.d), dtype=torch.float32, device=self.device)
        _lib.check(self.lib.kitty_flatten(self._desc_ref, u, n, ko.data_ptr(), vo.data_ptr(), _stream()), "flatten")
        return ko, vo

    def head_rows(self, b: int, h: int) -> dict:
        """The full-precision rows of unit (b, h) in the reference's segments
        (cache.py:65-80): key / value sink, key q-buffer, value q-buffer, value
        local window, each [rows, d] float32 read back from the device."""
        cfg, n = self.cfg, self.lengths[b]
        c = component_counts(cfg, n)
        u = b * cfg.h_kv + h
        W = cfg.r + cfg.g
        f = lambda t: t.float().cpu().numpy()
        S, kp, vp = cfg.s, c["key_pages"], c["value_pages"]
        kq_pos = [(t - S) % cfg.g for t in range(S + kp * cfg.g, S + kp * cfg.g + c["key_qbuf"])]
        vq_pos = [(t - S) % W for t in range(S + vp * cfg.g, S + vp * cfg.g + c["value_qbuf"])]
        loc_pos = [(t - S) % W for t in range(n - c["local"], n)] if n > S else []
        idx = lambda pos: torch.tensor(pos, dtype=torch.long, device=self.device)
        return dict(key_sink=f(self.k_sink[u, : c["sink"]]), value_sink=f(self.v_sink[u, : c["sink"]]),
                    key_qbuffer=f(self.k_qbuf[u][idx(kq_pos)]), value_qbuffer=f(self.v_ring[u][idx(vq_pos)]),
                    value_local=f(self.v_ring[u][idx(loc_pos)]))

    def pages(self, b: int, h: int):
        """QuantizedKeyPage / QuantizedValuePage objects of unit (b, h) in page
        order, decoded from the device slots; with f32 metadata kept, their
        scales / zero points are the float32 values (the reference's in-memory
        pages, pages.py:60-78), else the slots' f16."""
        import dataclasses

        from .pages import deserialize_page

        cfg = self.cfg
        c = self.page_counts(b)
        u = b * cfg.h_kv + h
        if cfg.key_bits == PASSTHROUGH_BITS or cfg.value_bits == PASSTHROUGH_BITS:
            def raw(pool, table, count):  # pass-through pages: the stored rows as float32 (g, d) arrays
                out = []
                for sl in table[u, :count].tolist():
                    a = pool[sl].view(self.row_dtype).view(cfg.g, cfg.d).float().cpu().numpy()
                    out.append(np.ascontiguousarray(a))
                return out
            kraw = raw(self.key_pool, self.key_block_table, c["key_pages"]) if cfg.key_bits == PASSTHROUGH_BITS else None
            vraw = raw(self.value_pool, self.value_block_table, c["value_pages"]) if cfg.value_bits == PASSTHROUGH_BITS else None
        else:
            kraw = vraw = None
        ks_ = self.key_page_slots(b, h).cpu().numpy() if kraw is None else []
        vs_ = self.value_page_slots(b, h).cpu().numpy() if vraw is None else []
        kb = [serialize_slot(x.tobytes(), "key", cfg.d, cfg.g, cfg.d_boost) for x in ks_]
        vb = [serialize_slot(x.tobytes(), "value", cfg.d, cfg.g) for x in vs_]
        kpg = kraw if kraw is not None else [deserialize_page(x) for x in kb]
        vpg = vraw if vraw is not None else [deserialize_page(x) for x in vb]
        if self.f32_metadata:
            km = self.key_meta[self.key_block_table[u, : c["key_pages"]].long()].cpu().numpy()
            vm = self.value_meta[self.value_block_table[u, : c["value_pages"]].long()].cpu().numpy()

            def frozen(a):
                a = np.ascontiguousarray(a, np.float32)
                a.flags.writeable = False
                return a

            if kraw is None:
                kpg = [dataclasses.replace(pg, scales=frozen(m[: cfg.d]), zero_points=frozen(m[cfg.d:])) for pg, m in zip(kpg, km)]
            if vraw is None:
                vpg = [dataclasses.replace(pg, scales=frozen(m[: cfg.g]), zero_points=frozen(m[cfg.g:])) for pg, m in zip(vpg, vm)]
        return kpg, vpg

    def page_counts(self, b: int) -> dict:
        return component_counts(self.cfg, self.lengths[b])

    def key_page_slots(self, b: int, h: int) -> torch.Tensor:
        """Device slots (KTYP key bodies) of (b, h) in page order."""
        c = self.page_counts(b)
        u = b * self.cfg.h_kv + h
        idx = self.key_block_table[u, : c["key_pages"]].long()
        return self.key_pool[idx]

    def value_page_slots(self, b: int, h: int) -> torch.Tensor:
        c = self.page_counts(b)
        u = b * self.cfg.h_kv + h
        idx = self.value_block_table[u, : c["value_pages"]].long()
        return self.value_pool[idx]

    def export_pages(self, b: int, h: int):
        """KTYP byte strings of all pages of (b, h): header + memcpy of each slot."""
        cfg = self.cfg
        if cfg.key_bits == PASSTHROUGH_BITS or cfg.value_bits == PASSTHROUGH_BITS:
            raise KittyError("pass-through (16-bit) pages have no KTYP encoding (pages.py:207-237)")
        ks = self.key_page_slots(b, h).cpu().numpy()
        vs = self.value_page_slots(b, h).cpu().numpy()
        return ([serialize_slot(s.tobytes(), "key", cfg.d, cfg.g, cfg.d_boost) for s in ks],
                [serialize_slot(s.tobytes(), "value", cfg.d, cfg.g) for s in vs])

    # -- offload / restore: KTYP pages + full-precision rows --------------------

    def export_sequence(self, b: int) -> dict:
        """The state of sequence b for offload: its length, and per KV head the
        KTYP pages (pages.py:207-237; header + memcpy of each slot) and the
        full-precision rows of the reference's segments (cache.py:65-80)."""
        heads = []
        for h in range(self.cfg.h_kv):
            kb, vb = self.export_pages(b, h)
            heads.append(dict(key_pages=kb, value_pages=vb, **self.head_rows(b, h)))
        return dict(length=self.lengths[b], heads=heads)

    def import_sequence(self, b: int, state: dict):
        """Restore an exported sequence into the empty row b: every page is
        decoded on the host (KTYP header rules, pages.py:246-292), copied to a
        slot the device claims from the pool and checked there (boost_idx
        bijection, pages.py:128-135); the rows go back to their sink / q-buffer
        / ring positions.  A round trip is byte-identical."""
        from .pages import slot_body

        cfg = self.cfg
        if self.lengths[b]:
            raise KittyError("import requires an empty sequence row")
        n = int(state["length"])
        c = component_counts(cfg, n)
        if len(state["heads"]) != cfg.h_kv:
            raise KittyError(f"state has {len(state['heads'])} heads, the cache {cfg.h_kv}")
        if n > self.max_tokens:
            self.grow(n)
        kp, vp = c["key_pages"], c["value_pages"]
        self._reserve(kp * cfg.h_kv, vp * cfg.h_kv)
        S, G, W = cfg.s, cfg.g, cfg.r + cfg.g
        idx = lambda pos: torch.tensor(pos, dtype=torch.long, device=self.device)
        rows = lambda a, k: torch.as_tensor(np.asarray(a, np.float32).reshape(-1, cfg.d)[:k]).to(self.device, self.row_dtype)
        keep = []
        for h, hs in enumerate(state["heads"]):
            u = b * cfg.h_kv + h
            if len(hs["key_pages"]) != kp or len(hs["value_pages"]) != vp:
                raise KittyError(f"head {h}: {len(hs['key_pages'])} / {len(hs['value_pages'])} pages, "
                                 f"length {n} needs {kp} / {vp}")
            for kind, pages, k in (("key", hs["key_pages"], 0), ("value", hs["value_pages"], 1)):
                if not pages:
                    continue
                body = b"".join(slot_body(raw, kind, cfg.d, cfg.g, cfg.d_boost) for raw in pages)
                t = torch.frombuffer(bytearray(body), dtype=torch.uint8).to(self.device)
                keep.append(t)
                _lib.check(self.lib.kitty_import_pages(self._desc_ref, u, k, t.data_ptr(), 0, len(pages), _stream()),
                           "import")
            self.k_sink[u, : c["sink"]] = rows(hs["key_sink"], c["sink"])
            self.v_sink[u, : c["sink"]] = rows(hs["value_sink"], c["sink"])
            kq_pos = [(t - S) % G for t in range(S + kp * G, S + kp * G + c["key_qbuf"])]
            vq_pos = [(t - S) % W for t in range(S + vp * G, S + vp * G + c["value_qbuf"])]
            loc_pos = [(t - S) % W for t in range(n - c["local"], n)] if n > S else []
            if kq_pos:
                self.k_qbuf[u][idx(kq_pos)] = rows(hs["key_qbuffer"], len(kq_pos))
            if vq_pos:
                self.v_ring[u][idx(vq_pos)] = rows(hs["value_qbuffer"], len(vq_pos))
            if loc_pos:
                self.v_ring[u][idx(loc_pos)] = rows(hs["value_local"], len(loc_pos))
        self.unit_len[b * cfg.h_kv:(b + 1) * cfg.h_kv] = n
        self.free_pages[0] -= kp * cfg.h_kv
        self.free_pages[1] -= vp * cfg.h_kv
        self._set_length(b, n)
        self._keep = keep  # staging buffers stay alive until the copies ran (stream order)

    def hbm_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (
            self.k_sink, self.v_sink, self.k_qbuf, self.v_ring, self.key_pool, self.value_pool))


class _RowsView:
    """The reference's _RowStore (cache.py:41-62) of rows read back from the device."""

    def __init__(self, rows: np.ndarray):
        self._rows = rows

    def __len__(self):
        return self._rows.shape[0]

    def view(self) -> np.ndarray:
        return self._rows


class _HeadView:
    """The reference's _HeadState (cache.py:65-80) of one KV head, read back
    from the device: sink row stores, q-buffer / local row lists, page lists."""

    def __init__(self, batch: "KittyBatchCache", b: int, h: int):
        rows = batch.head_rows(b, h)
        self.key_sink = _RowsView(rows["key_sink"])
        self.value_sink = _RowsView(rows["value_sink"])
        self.key_qbuffer = list(rows["key_qbuffer"])
        self.value_qbuffer = list(rows["value_qbuffer"])
        self.value_local = list(rows["value_local"])
        self.key_pages, self.value_pages = batch.pages(b, h)


class KittyCacheState:
    """The reference's per-sequence state (cache.py:83-252) on the device, at
    the reference's precision: float32 rows and float32 page metadata, the
    generic kernels (attention in f32 with expf, cache.py:241-258)."""

    def __init__(self, cfg: KittyConfig, max_tokens: int = 1024, row_dtype: torch.dtype = torch.float32):
        """``row_dtype`` float32 (default): the reference's precision; bfloat16:
        the product path (fused kernels, f16 page metadata) behind the same API."""
        _check_device_config(cfg)
        self.cfg = cfg
        self._b = KittyBatchCache(cfg, 1, max_tokens, row_dtype=row_dtype, f32_metadata=row_dtype == torch.float32)

    @property
    def total_tokens(self) -> int:
        return self._b.lengths[0]

    @property
    def key_pack_events(self) -> int:
        return self._b.key_pack_events[0]

    @property
    def value_pack_events(self) -> int:
        return self._b.value_pack_events[0]

    @property
    def batch(self) -> KittyBatchCache:
        return self._b

    @property
    def heads(self) -> list:
        """Per-KV-head state (cache.py:88), read back from the device."""
        return [_HeadView(self._b, 0, h) for h in range(self.cfg.h_kv)]

    def _coerce_rows(self, new, what):
        new = np.asarray(new.cpu() if isinstance(new, torch.Tensor) else new, dtype=np.float32)
        if new.ndim == 1:
            new = new[None, :]
        if new.shape != (self.cfg.h_kv, self.cfg.d):
            raise KittyError(f"{what} must have shape ({self.cfg.h_kv}, {self.cfg.d}), got {new.shape}")
        return torch.from_numpy(np.ascontiguousarray(new))[None]

    def insert_token(self, k_new, v_new) -> None:
        """cache.py:107-123 (pack fires inside, before any attend)."""
        self._b.append(self._coerce_rows(k_new, "k_new"), self._coerce_rows(v_new, "v_new"))
        self._b.check()

    def prefill(self, keys, values) -> None:
        """cache.py:125-142."""
        if self.total_tokens != 0:
            raise KittyError("prefill requires an empty state")
        keys = np.asarray(keys, dtype=np.float32)
        values = np.asarray(values, dtype=np.float32)
        if keys.ndim == 2:
            keys = keys[None]
        if values.ndim == 2:
            values = values[None]
        if keys.shape != values.shape or keys.shape[0] != self.cfg.h_kv:
            raise KittyError("prefill keys/values must be (h_kv, P, d) with equal shapes")
        if keys.shape[1] == 0:
            return
        self._b.prefill(torch.from_numpy(np.ascontiguousarray(keys))[None], torch.from_numpy(np.ascontiguousarray(values))[None])
        self._b.check()

    def maybe_pack(self) -> int:
        """cache.py:144-178: packing already ran inside insert; nothing is pending."""
        return 0

    def flatten_keys(self, kv_head: int = 0) -> np.ndarray:
        return self._b.flatten(0, kv_head)[0].cpu().numpy()

    def flatten_values(self, kv_head: int = 0) -> np.ndarray:
        return self._b.flatten(0, kv_head)[1].cpu().numpy()

    def attend(self, q, return_probs: bool = False) -> AttentionOutput:
        """cache.py:217-252 on the device.  With ``return_probs`` the (h_q, n)
        probabilities come from ``kitty_dense_probs`` over the flattened keys
        (the decode kernels never materialise them)."""
        if self.total_tokens == 0:
            raise KittyError("attend on an empty cache")
        q = np.asarray(q.cpu() if isinstance(q, torch.Tensor) else q, dtype=np.float32)
        if q.ndim == 1:
            q = q[None, :]
        if q.shape != (self.cfg.h_q, self.cfg.d):
            raise KittyError(f"q must have shape ({self.cfg.h_q}, {self.cfg.d}), got {q.shape}")
        qt = torch.from_numpy(np.ascontiguousarray(q))
        out = self._b.attend(qt[None], out_dtype=torch.float32)
        probs = None
        if return_probs:
            keys = torch.stack([self._b.flatten(0, h)[0] for h in range(self.cfg.h_kv)])
            probs = _dense_probs(keys, qt.to(keys.device), [i // self.cfg.group_size for i in range(self.cfg.h_q)])
        self._b.check()
        return AttentionOutput(outputs=out[0].cpu().numpy(), probs=None if probs is None else probs.cpu().numpy())

    def export_pages(self, kv_head: int = 0):
        return self._b.export_pages(0, kv_head)


def _dense_probs(keys: torch.Tensor, queries: torch.Tensor, kv_head_map) -> torch.Tensor:
    """kitty_dense_probs: keys [h_kv, L, d] f32, queries [n_q, d] f32 on the device."""
    lib = _lib.load_library()
    h_kv, length, d = keys.shape
    n_q = queries.shape[0]
    kmap = torch.tensor(list(kv_head_map), dtype=torch.int32, device=keys.device)
    probs = torch.empty((n_q, length), dtype=torch.float32, device=keys.device)
    _lib.check(lib.kitty_dense_probs(keys.contiguous().data_ptr(), h_kv, length, d, queries.contiguous().data_ptr(), n_q,
                                     kmap.data_ptr(), probs.data_ptr(), _stream()), "attention probabilities")
    return probs


def oracle_attend(keys, values, queries, kv_head_map=None) -> AttentionOutput:
    """cache.py:261-301: dense float32 attention, run on the device."""
    lib = _lib.load_library()
    dev = _device()
    keys = np.asarray(keys, dtype=np.float32)
    values = np.asarray(values, dtype=np.float32)
    queries = np.asarray(queries, dtype=np.float32)
    if queries.ndim == 1:
        queries = queries[None, :]
    if keys.ndim == 2:
        keys, values = keys[None], values[None]
    if keys.shape != values.shape:
        raise KittyError("keys and values must have matching shapes")
    h_kv, length, d = keys.shape
    if length == 0:
        raise KittyError("attention over zero tokens")
    n_q = queries.shape[0]
    if kv_head_map is None:
        kv_head_map = [i * h_kv // n_q for i in range(n_q)]
    k = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    v = torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    qs = torch.from_numpy(np.ascontiguousarray(queries)).to(dev)
    kmap = torch.tensor(list(kv_head_map), dtype=torch.int32, device=dev)
    out = torch.empty((n_q, d), dtype=torch.float32, device=dev)
    ws = torch.empty(max(16, int(lib.kitty_dense_attention_workspace_bytes(n_q, length, d))), dtype=torch.uint8, device=dev)
    _lib.check(lib.kitty_dense_attention(k.data_ptr(), v.data_ptr(), h_kv, length, d, qs.data_ptr(), n_q,
                                         kmap.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), _stream()),
               "oracle_attend")
    probs = _dense_probs(k, qs, kv_head_map)
    return AttentionOutput(outputs=out.cpu().numpy(), probs=probs.cpu().numpy())
