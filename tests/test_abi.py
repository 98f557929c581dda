"""CPU tests of the C ABI boundary: the library loads, exports every symbol include/oscar.h
declares, and validates arguments on the host (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "oscar.h")
LIB = os.path.join(ROOT, "paper_2605_17757_b200", "liboscar.so")


def _ensure_built():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", ROOT], check=True, capture_output=True)


def declared_symbols():
    text = open(HEADER).read()
    return re.findall(r"OSCAR_API\s+[\w\s\*]+?\b(oscar_\w+)\s*\(", text)


def test_header_declares_the_three_calls_and_hooks():
    names = set(declared_symbols())
    for n in ["oscar_calib_accumulate", "oscar_calib_finalize", "oscar_quantize_append",
              "oscar_attend", "oscar_rotate", "oscar_quantize_rotated", "oscar_create"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    _ensure_built()
    lib = ctypes.CDLL(LIB)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    from paper_2605_17757_b200 import binding
    assert sorted(binding.EXPORTED) == sorted(declared_symbols())


def test_library_is_sm100a_only():
    _ensure_built()
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def _ctx(**kw):
    _ensure_built()
    from paper_2605_17757_b200 import binding as B
    return B, B.Oscar(B.Config(**kw))


def test_create_validation():
    _ensure_built()
    from paper_2605_17757_b200 import binding as B
    bad = [(dict(head_dim=96), B.ERR_DIM), (dict(head_dim=64), B.ERR_UNSUPPORTED),
           (dict(num_q_heads=30), B.ERR_ARG), (dict(bits=5), B.ERR_ARG),
           (dict(group_size=48), B.ERR_ARG),
           (dict(page_size=20), B.ERR_ARG), (dict(clip_ratio_k=0.0), B.ERR_ARG),
           (dict(clip_ratio_v=1.5), B.ERR_ARG)]
    for kw, st in bad:
        with pytest.raises(B.OscarError) as e:
            B.Oscar(B.Config(**kw))
        assert e.value.status == st, kw
    assert "oscar-b200" in B.version()
    # g > 8 creates (calibration, incl. the shared-rotation mode H_kv = 1) but attend refuses it
    o = B.Oscar(B.Config(num_q_heads=72, num_kv_heads=8))
    assert B.raw_call("oscar_attend", o._h, None, None, None, 1, 1, None, None, None, None, 0, None, 0,
                      None, None) == B.ERR_UNSUPPORTED
    B.Oscar(B.Config(num_q_heads=32, num_kv_heads=1))


def test_page_bytes_matches_format():
    B, o = _ctx(bits=2, group_size=64, page_size=64)
    assert o.page_bytes() == 5120                     # 2*64*32 + 64*2*8
    B, o = _ctx(bits=4, group_size=32, page_size=64, num_q_heads=1, num_kv_heads=1)
    assert o.page_bytes() == 2 * 64 * 64 + 64 * 4 * 8
    import oracle as O
    for bits, G, P in [(2, 64, 64), (4, 32, 64), (2, 128, 16), (4, 64, 32), (3, 64, 64), (3, 32, 16)]:
        B, o = _ctx(bits=bits, group_size=G, page_size=P)
        assert o.page_bytes() == O.PageFormat(128, bits, G, P).page_bytes


def test_null_and_size_validation_without_gpu():
    B, o = _ctx()
    h = o._h
    # T = 0 / N = 0 / B = 0 are no-ops; negative sizes and NULL pointers are ERR_ARG
    assert B.raw_call("oscar_quantize_append", h, None, None, None, 0, None, None, None, None) == B.OK
    assert B.raw_call("oscar_quantize_append", h, None, None, None, -1, None, None, None, None) == B.ERR_ARG
    assert B.raw_call("oscar_quantize_append", h, None, None, None, 5, None, None, None, None) == B.ERR_ARG
    assert B.raw_call("oscar_calib_accumulate", h, None, None, 0, None, None) == B.OK
    assert B.raw_call("oscar_calib_accumulate", h, None, None, -3, None, None) == B.ERR_ARG
    assert B.raw_call("oscar_calib_finalize", h, None, 0, 10, None, None, None, None, None) == B.ERR_ARG
    assert B.raw_call("oscar_rotate", h, None, None, None, 4, None) == B.ERR_ARG
    assert B.raw_call("oscar_quantize_rotated", h, None, None, None, 4, None, None) == B.ERR_ARG
    assert B.raw_call("oscar_attend", h, None, None, None, 0, 4, None, None, None, None, 0, None,
                      0, None, None) == B.OK
    assert B.raw_call("oscar_attend", h, None, None, None, 2, 4, None, None, None, None, 0, None,
                      0, None, None) == B.ERR_ARG
    assert o.attend_workspace_bytes(16, 512) > 16 * 32 * 128 * 4
    assert B.raw_call("oscar_set_variant", h, 7) == B.ERR_ARG
    assert "bad argument" in B._lib.oscar_last_error().decode()
