"""ctypes binding of libkitty_b200.so (include/kitty_b200.h).

The library is built in-tree by ``build()`` (csrc/Makefile).  There is no
fallback: if it is missing, or no CUDA device is visible when a device entry
point is called, an exception is raised.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, DeviceError, KittyError, PageFormatError

_HERE = os.path.dirname(os.path.abspath(__file__))
# KITTY_B200_LIB points at an alternative in-tree build (kernel experiments only)
LIB_PATH = os.environ.get("KITTY_B200_LIB") or os.path.join(_HERE, "libkitty_b200.so")

KITTY_OK, KITTY_ERR_CONFIG, KITTY_ERR_INVALID, KITTY_ERR_PAGE_FORMAT, KITTY_ERR_CUDA, KITTY_ERR_UNSUPPORTED = range(6)
STATUS_NONFINITE, STATUS_PAGE_FORMAT, STATUS_OVERFLOW, STATUS_LENGTH = 1, 2, 4, 8
KITTY_F32, KITTY_BF16 = 0, 1

c_int32 = ctypes.c_int32
c_int64 = ctypes.c_int64
c_void_p = ctypes.c_void_p
c_size_t = ctypes.c_size_t


class KittyConfigC(ctypes.Structure):
    _fields_ = [
        ("s", c_int32), ("r", c_int32), ("g", c_int32), ("d", c_int32),
        ("h_kv", c_int32), ("h_q", c_int32), ("d_boost", c_int32),
        ("key_bits", c_int32), ("value_bits", c_int32),
    ]


class KittyCacheDesc(ctypes.Structure):
    _fields_ = [
        ("cfg", KittyConfigC),
        ("num_seqs", c_int32),
        ("max_pages", c_int32),
        ("key_slot_bytes", c_int64),
        ("value_slot_bytes", c_int64),
        ("unit_len", c_void_p),
        ("k_sink", c_void_p),
        ("v_sink", c_void_p),
        ("k_qbuf", c_void_p),
        ("v_ring", c_void_p),
        ("key_pool", c_void_p),
        ("value_pool", c_void_p),
        ("key_block_table", c_void_p),
        ("value_block_table", c_void_p),
        ("status", c_void_p),
        ("row_dtype", c_int32),
        ("reserved", c_int32),
        ("key_meta", c_void_p),
        ("value_meta", c_void_p),
        ("key_free", c_void_p),
        ("value_free", c_void_p),
        ("free_top", c_void_p),
        ("key_slots", c_int32),
        ("value_slots", c_int32),
    ]


# (name, restype, argtypes) -- the full exported surface of kitty_b200.h
SIGNATURES = [
    ("kitty_key_slot_bytes", c_int64, [c_int32, c_int32, c_int32]),
    ("kitty_value_slot_bytes", c_int64, [c_int32, c_int32]),
    ("kitty_validate_config", ctypes.c_int, [ctypes.POINTER(KittyConfigC)]),
    ("kitty_version", ctypes.c_char_p, []),
    ("kitty_last_error", ctypes.c_char_p, []),
    ("kitty_channel_scores", ctypes.c_int, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    ("kitty_select_boost", ctypes.c_int, [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    ("kitty_pack_key_pages", ctypes.c_int,
     [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("kitty_pack_value_pages", ctypes.c_int,
     [c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("kitty_dequant_key_pages", ctypes.c_int,
     [c_void_p, c_int64, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("kitty_dequant_value_pages", ctypes.c_int,
     [c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("kitty_quantize_lanes", ctypes.c_int,
     [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("kitty_dequantize_lanes", ctypes.c_int,
     [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("kitty_fake_quantize", ctypes.c_int, [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    ("kitty_append", ctypes.c_int, [ctypes.POINTER(KittyCacheDesc), c_void_p, c_void_p, c_void_p]),
    ("kitty_prefill", ctypes.c_int, [ctypes.POINTER(KittyCacheDesc), c_void_p, c_void_p, c_int32, c_void_p]),
    ("kitty_release_sequences", ctypes.c_int, [ctypes.POINTER(KittyCacheDesc), c_int32, c_int32, c_void_p]),
    ("kitty_import_pages", ctypes.c_int,
     [ctypes.POINTER(KittyCacheDesc), c_int32, c_int32, c_void_p, c_int32, c_int32, c_void_p]),
    ("kitty_flatten", ctypes.c_int, [ctypes.POINTER(KittyCacheDesc), c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    ("kitty_attention_workspace_bytes", c_size_t, [ctypes.POINTER(KittyCacheDesc), c_int32]),
    ("kitty_decode_attention", ctypes.c_int,
     [ctypes.POINTER(KittyCacheDesc), c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_size_t, c_void_p]),
    ("kitty_sensitivity_workspace_bytes", c_size_t, [c_int32, c_int32, c_int32, c_int32, c_int32]),
    ("kitty_channel_sensitivity", ctypes.c_int,
     [c_void_p, c_int32, c_int32, c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("kitty_attention_mse_workspace_bytes", c_size_t, [c_int32, c_int32, c_int32, c_int32]),
    ("kitty_attention_mse", ctypes.c_int,
     [c_void_p, c_int32, c_int32, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("kitty_dense_probs", ctypes.c_int,
     [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    ("kitty_dense_attention_workspace_bytes", c_size_t, [c_int32, c_int32, c_int32]),
    ("kitty_dense_attention", ctypes.c_int,
     [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
]

_lib = None


def load_library():
    """Load (once) and return the ctypes handle; raise ImportError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2511_18643_b200/csrc); there is no CPU fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load_library().kitty_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a KittyStatus to the reference exception types (errors.py:4-33)."""
    if rc == KITTY_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == KITTY_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == KITTY_ERR_PAGE_FORMAT:
        raise PageFormatError(msg)
    if rc == KITTY_ERR_CUDA:
        raise DeviceError(msg)
    raise KittyError(msg)


def raise_status(word: int, what: str = "") -> None:
    """Raise for a device status word read back after a sync."""
    if word == 0:
        return
    if word & STATUS_PAGE_FORMAT:
        raise PageFormatError(f"{what}: boost_idx sentinel count or bijection violated")
    if word & STATUS_NONFINITE:
        raise KittyError(f"{what}: page contains non-finite values")
    if word & STATUS_OVERFLOW:
        raise KittyError(f"{what}: cache capacity exceeded (block table full or page pool empty)")
    if word & STATUS_LENGTH:
        raise KittyError(f"{what}: a sequence is longer than the max_tokens bound passed to attention")
    raise KittyError(f"{what}: device status 0x{word:x}")


def exported_symbols() -> list[str]:
    return [name for name, _, _ in SIGNATURES]
