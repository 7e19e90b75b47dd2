"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/kitty_b200.h declares, and its host-only entry points agree with the
reference's byte accounting and config validation (no compute calls)."""

import ctypes
import os
import re
import subprocess

import pytest

import paper_2511_18643_b200 as kb
from paper_2511_18643_b200 import _lib
from oracle import kitty_oracle as ko

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kitty_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(kitty_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = kb.load_library()
    decl = declared_symbols()
    assert len(decl) >= 18
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == decl


def test_symbols_are_exported_from_the_so(tmp_path):
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_version_string():
    assert b"sm_100a" in kb.load_library().kitty_version()


@pytest.mark.parametrize("d,g,frac", [(128, 128, 0.0), (128, 128, 0.0625), (128, 128, 0.125),
                                      (128, 128, 0.25), (8, 8, 0.25), (64, 32, 1.0)])
def test_slot_sizes_match_reference_accounting(d, g, frac):
    lib = kb.load_library()
    db = ko.boost_count(frac, d)
    assert lib.kitty_key_slot_bytes(d, g, db) == ko.key_slot_bytes(d, g, db)
    assert lib.kitty_value_slot_bytes(d, g) == ko.value_slot_bytes(d, g)


def test_default_slot_kat():
    # test_pages.py:172-181
    lib = kb.load_library()
    assert lib.kitty_key_slot_bytes(128, 128, 16) == 5248
    assert lib.kitty_value_slot_bytes(128, 128) == 4608
    for db, size in ((0, 4736), (8, 4992), (16, 5248), (32, 5760), ):
        assert lib.kitty_key_slot_bytes(128, 128, db) == size
        assert size % 16 == 0


def _cfg(**kw):
    base = dict(s=32, r=128, g=128, d=128, h_kv=8, h_q=32, d_boost=16, key_bits=2, value_bits=2)
    base.update(kw)
    return _lib.KittyConfigC(**base)


@pytest.mark.parametrize("kw,code", [
    (dict(), _lib.KITTY_OK),
    (dict(s=-1), _lib.KITTY_ERR_CONFIG),
    (dict(r=0), _lib.KITTY_ERR_CONFIG),
    (dict(g=6), _lib.KITTY_ERR_CONFIG),
    (dict(d=10), _lib.KITTY_ERR_CONFIG),
    (dict(h_kv=2, h_q=3), _lib.KITTY_ERR_CONFIG),
    (dict(key_bits=4), _lib.KITTY_ERR_CONFIG),
    (dict(value_bits=8), _lib.KITTY_ERR_CONFIG),
    (dict(d_boost=300, d=512), _lib.KITTY_ERR_CONFIG),
    (dict(key_bits=16), _lib.KITTY_OK),  # pass-through pages: generic kernels
])
def test_validate_config_mirrors_reference(kw, code):
    # config.py:35-53 / test_cache.py:32-48
    lib = kb.load_library()
    assert lib.kitty_validate_config(ctypes.byref(_cfg(**kw))) == code


def test_status_codes_map_to_reference_exceptions():
    with pytest.raises(kb.ConfigError):
        _lib.check(_lib.KITTY_ERR_CONFIG)
    with pytest.raises(kb.PageFormatError):
        _lib.check(_lib.KITTY_ERR_PAGE_FORMAT)
    with pytest.raises(kb.KittyError):
        _lib.check(_lib.KITTY_ERR_INVALID)
    with pytest.raises(kb.DeviceError):
        _lib.check(_lib.KITTY_ERR_CUDA)
    with pytest.raises(kb.PageFormatError):
        _lib.raise_status(_lib.STATUS_PAGE_FORMAT)
    with pytest.raises(kb.KittyError):
        _lib.raise_status(_lib.STATUS_NONFINITE)
    _lib.raise_status(0)


def test_desc_struct_layout_matches_header(tmp_path):
    # offsets of the POD the C side reads (KittyCacheDesc in kitty_b200.h), as
    # the C compiler lays it out, against the ctypes mirror the shim passes
    fields = [f[0] for f in _lib.KittyCacheDesc._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "kitty_b200.h"\nint main(void) {\n'
                   + "".join(f'  printf("%zu\\n", offsetof(KittyCacheDesc, {f}));\n' for f in fields)
                   + '  printf("%zu\\n", sizeof(KittyCacheDesc));\n  return 0;\n}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [getattr(_lib.KittyCacheDesc, f).offset for f in fields] + [ctypes.sizeof(_lib.KittyCacheDesc)]
    assert got == want
    assert ctypes.sizeof(_lib.KittyConfigC) == 36


def test_invalid_args_rejected_without_gpu():
    lib = kb.load_library()
    # g not a multiple of 4 (pages.py:85-86): rejected before any launch
    rc = lib.kitty_pack_key_pages(None, 0, 1, 6, 4, 0, None, None, 64, None, None, None, None)
    assert rc == _lib.KITTY_ERR_INVALID
    rc = lib.kitty_pack_value_pages(None, 0, 1, 4, 6, None, 64, None, None, None, None)
    assert rc == _lib.KITTY_ERR_INVALID
    rc = lib.kitty_dense_attention(None, None, 1, 0, 4, None, 1, None, None, None, 0, None)
    assert rc == _lib.KITTY_ERR_INVALID
