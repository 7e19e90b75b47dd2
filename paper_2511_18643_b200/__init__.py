"""paper_2511_18643_b200 -- B200-native Kitty decode hot path.

Keeps the names of the reference package ``kittykv`` (__init__.py:61-112) for
the hot path (quantize / pack / dequantize / append / attend) and adds the
batched device API (``KittyBatchCache``, ``pack_key_pages``, ...).  Compute
runs in ``libkitty_b200.so`` (hand-written sm_100a CUDA behind a C ABI,
include/kitty_b200.h); there is no CPU fallback.
"""

from ._lib import exported_symbols, load_library
from .analysis import MemoryReport, algorithmic_bytes_per_unit, measure_cache_bytes, memory_report
from .cache import AttentionOutput, KittyBatchCache, KittyCacheState, component_counts, oracle_attend
from .sensitivity import (
    SensitivityReport,
    SweepRow,
    SyntheticSpec,
    attention_mse,
    boost_sweep,
    boost_sweep_experiment,
    channel_sensitivity,
    generate_synthetic,
)
from .config import PASSTHROUGH_BITS, KittyConfig, boost_count, config_from_mapping
from .errors import (
    BadMagicError,
    ConfigError,
    DeviceError,
    KittyError,
    NonFiniteError,
    PageFormatError,
    TensorIOError,
    TruncatedFileError,
    UnknownDtypeError,
)
from .pages import (
    SENTINEL,
    BoostSelection,
    PageByteCounts,
    QuantParams,
    QuantizedKeyPage,
    QuantizedValuePage,
    channel_scores,
    channel_scores_batch,
    dequant_key_pages,
    dequant_value_pages,
    dequantize_key_page,
    dequantize_value_page,
    deserialize_page,
    dequantize_values,
    fake_quantize_matrix,
    pack_key_page,
    pack_key_pages,
    pack_value_page,
    pack_value_pages,
    page_byte_size,
    quantize_values,
    select_boost,
    select_boost_batch,
    serialize_page,
    serialize_slot,
)

__version__ = "0.1.0"

__all__ = [
    "AttentionOutput", "BadMagicError", "BoostSelection", "ConfigError", "DeviceError",
    "KittyBatchCache", "KittyCacheState", "KittyConfig", "KittyError", "MemoryReport",
    "NonFiniteError", "PASSTHROUGH_BITS", "PageByteCounts", "PageFormatError",
    "QuantizedKeyPage", "QuantizedValuePage", "SENTINEL", "TensorIOError", "TruncatedFileError",
    "UnknownDtypeError", "algorithmic_bytes_per_unit", "boost_count", "channel_scores",
    "channel_scores_batch", "component_counts", "config_from_mapping", "dequant_key_pages",
    "dequant_value_pages", "dequantize_key_page", "dequantize_value_page", "deserialize_page",
    "fake_quantize_matrix",
    "exported_symbols", "load_library", "measure_cache_bytes", "memory_report", "oracle_attend",
    "pack_key_page", "pack_key_pages", "pack_value_page", "pack_value_pages", "page_byte_size",
    "select_boost", "select_boost_batch", "serialize_page", "serialize_slot",
    "SensitivityReport", "SweepRow", "SyntheticSpec", "attention_mse", "boost_sweep", "boost_sweep_experiment",
    "channel_sensitivity", "generate_synthetic", "QuantParams", "quantize_values", "dequantize_values",
]
