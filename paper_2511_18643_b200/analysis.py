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


# -- report rendering (analysis.py:377-444: host text formatting of the results) --

PRNG_ID = "pcg64"  # tensor_io.py:37: the generator every seeded input comes from


def report_header(command: str, seed, config_mapping: dict | None = None) -> list[str]:
    """analysis.py:377-387: self-describing comment block."""
    from . import __version__

    lines = [f"# kittykv {__version__}", f"# command: {command}", f"# prng: {PRNG_ID}", f"# seed: {seed}"]
    for key in sorted(config_mapping or {}):
        lines.append(f"# {key} = {config_mapping[key]}")
    return lines


def _fmt(value) -> str:
    return format(value, ".10g") if isinstance(value, float) else str(value)


def write_csv(path, header_lines, columns, rows) -> None:
    """analysis.py:396-402."""
    with open(path, "w") as fh:
        for line in header_lines:
            fh.write(line + "\n")
        fh.write(",".join(columns) + "\n")
        for row in rows:
            fh.write(",".join(_fmt(v) for v in row) + "\n")


def sensitivity_csv_rows(report):
    """analysis.py:405-412: one row per channel, one column per query head."""
    h_q, d = report.mse.shape
    columns = ["channel"] + [f"mse_qhead_{h}" for h in range(h_q)] + ["mean_mse"]
    return columns, [[ch, *(float(report.mse[h, ch]) for h in range(h_q)), float(report.mean_mse[ch])] for ch in range(d)]


def sweep_csv_rows(rows):
    """analysis.py:415-419."""
    return ["fraction", "heuristic", "mean_mse", "max_deviation", "runs"], [
        [r.fraction, r.heuristic, r.mean_mse, r.max_deviation, r.runs] for r in rows]


def memory_summary(report: MemoryReport) -> list[str]:
    """analysis.py:422-444: ``key: value`` lines of a memory report."""
    keys = ["length", "key_sink_bytes", "key_qbuffer_bytes", "key_page_count", "key_pages_payload",
            "key_pages_metadata", "key_pages_index", "value_sink_bytes", "value_local_bytes", "value_qbuffer_bytes",
            "value_page_count", "value_pages_payload", "value_pages_metadata", "total_bytes", "kv_data_bytes",
            "baseline_bytes", "compression_ratio", "kv_data_ratio"]
    return [f"{k}: {_fmt(getattr(report, k))}" for k in keys]
