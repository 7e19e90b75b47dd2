"""Byte accounting of the cache (analysis.py:242-371) and the algorithmic-bytes
formula the roofline numbers use."""

from __future__ import annotations

from dataclasses import dataclass

from .cache import component_counts
from .config import PASSTHROUGH_BITS, KittyConfig
from .errors import KittyError
from .pages import page_byte_size

FP_BYTES = 2  # analysis.py:29


@dataclass(frozen=True)
class MemoryReport:
    """analysis.py:242-298."""

    length: int
    key_sink_bytes: int
    key_qbuffer_bytes: int
    key_page_count: int
    key_pages_payload: int
    key_pages_metadata: int
    key_pages_index: int
    value_sink_bytes: int
    value_local_bytes: int
    value_qbuffer_bytes: int
    value_page_count: int
    value_pages_payload: int
    value_pages_metadata: int
    baseline_bytes: int

    @property
    def total_bytes(self) -> int:
        return (self.key_sink_bytes + self.key_qbuffer_bytes + self.key_pages_payload
                + self.key_pages_metadata + self.key_pages_index + self.value_sink_bytes
                + self.value_local_bytes + self.value_qbuffer_bytes + self.value_pages_payload
                + self.value_pages_metadata)

    @property
    def kv_data_bytes(self) -> int:
        return self.total_bytes - self.key_pages_metadata - self.key_pages_index - self.value_pages_metadata

    @property
    def compression_ratio(self) -> float:
        return self.baseline_bytes / self.total_bytes if self.total_bytes else 1.0

    @property
    def kv_data_ratio(self) -> float:
        return self.baseline_bytes / self.kv_data_bytes if self.kv_data_bytes else 1.0


def _assemble(cfg: KittyConfig, length: int, c: dict) -> MemoryReport:
    """analysis.py:318-350."""
    fp_row = cfg.d * FP_BYTES * cfg.h_kv
    if cfg.key_bits == PASSTHROUGH_BITS:
        key_payload, key_meta, key_index = c["key_pages"] * cfg.g * fp_row, 0, 0
    else:
        per = page_byte_size("key", cfg)
        key_payload = c["key_pages"] * per.payload * cfg.h_kv
        key_meta = c["key_pages"] * per.metadata * cfg.h_kv
        key_index = c["key_pages"] * per.index * cfg.h_kv
    if cfg.value_bits == PASSTHROUGH_BITS:
        value_payload, value_meta = c["value_pages"] * cfg.g * fp_row, 0
    else:
        per = page_byte_size("value", cfg)
        value_payload = c["value_pages"] * per.payload * cfg.h_kv
        value_meta = c["value_pages"] * per.metadata * cfg.h_kv
    return MemoryReport(
        length=length, key_sink_bytes=c["sink"] * fp_row, key_qbuffer_bytes=c["key_qbuf"] * fp_row,
        key_page_count=c["key_pages"], key_pages_payload=key_payload, key_pages_metadata=key_meta,
        key_pages_index=key_index, value_sink_bytes=c["sink"] * fp_row,
        value_local_bytes=c["local"] * fp_row, value_qbuffer_bytes=c["value_qbuf"] * fp_row,
        value_page_count=c["value_pages"], value_pages_payload=value_payload,
        value_pages_metadata=value_meta, baseline_bytes=2 * FP_BYTES * length * cfg.d * cfg.h_kv,
    )


def memory_report(cfg: KittyConfig, length: int) -> MemoryReport:
    """analysis.py:353-357."""
    if length < 0:
        raise KittyError("length must be >= 0")
    return _assemble(cfg, length, component_counts(cfg, length))


def measure_cache_bytes(state) -> MemoryReport:
    """analysis.py:360-371: the accounting of an actually constructed state,
    counted from what the device holds for KV head 0 -- its sink / q-buffer /
    local rows and its pages, read back (KittyCacheState or (KittyBatchCache, b))."""
    if isinstance(state, tuple):
        batch, b = state
    else:
        batch, b = state.batch, 0
    rows = batch.head_rows(b, 0)
    kpages, vpages = batch.pages(b, 0)
    counts = dict(sink=len(rows["key_sink"]), key_pages=len(kpages), key_qbuf=len(rows["key_qbuffer"]),
                  local=len(rows["value_local"]), value_pages=len(vpages), value_qbuf=len(rows["value_qbuffer"]))
    return _assemble(batch.cfg, int(batch.unit_len[b * batch.cfg.h_kv].item()), counts)


def algorithmic_bytes_per_unit(cfg: KittyConfig, n: int) -> int:
    """Bytes one (seq, kv-head) attention must read/write at n tokens
    (SURVEY.md §8(d)): pages at 16-bit metadata, fp rows at 2 B, bf16 q in and
    out.  The device slots are exactly these bytes, so nothing is uncredited."""
    c = component_counts(cfg, n)
    key = c["key_pages"] * page_byte_size("key", cfg).total
    val = c["value_pages"] * page_byte_size("value", cfg).total
    fp = FP_BYTES * cfg.d * ((c["sink"] + c["key_qbuf"]) + (c["sink"] + c["local"] + c["value_qbuf"]))
    return key + val + fp + 2 * FP_BYTES * cfg.group_size * cfg.d
