"""The C-ABI library: builds, loads and exports every symbol include/tsketch.h declares.
CPU only -- no compute call is made without a GPU (only argument / device checks)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tsketch.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:tsk_status|const char\*|int64_t)\s+(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2209_14637_b200 import build
    build.build()
    import paper_2209_14637_b200 as tsk
    return tsk.lib()


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("sketch_train", "sketch_apply_scw", "scw_error", "sketch_gram", "sketch_topk", "tsk_create",
              "tsk_destroy", "tsk_sync", "tsk_status_string"):
        assert f in fns


def test_every_declared_symbol_is_exported(lib):
    import paper_2209_14637_b200 as tsk
    fns = declared_functions()
    for f in fns:
        assert hasattr(lib, f), f
    assert sorted(tsk.EXPORTED) == fns
    out = subprocess.run(["nm", "-D", "--defined-only", tsk.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    assert set(fns) <= exported


def test_library_is_sm100a_tcgen05(lib):
    import paper_2209_14637_b200 as tsk
    sass = subprocess.run(["cuobjdump", "-sass", tsk.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass      # tcgen05.mma
    assert "UTMALDG" in sass                          # TMA tensor loads
    assert "LDTM" in sass                             # tcgen05.ld (TMEM -> registers)
    elf = subprocess.run(["cuobjdump", "-lelf", tsk.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


def test_status_strings(lib):
    lib.tsk_status_string.restype = ctypes.c_char_p
    for s in (0, 1, 2, -1, -2, -3, -4, -5, -6, -7, -8):
        assert lib.tsk_status_string(s)
    assert b"unknown" in lib.tsk_status_string(12345)


def test_null_and_argument_errors_without_gpu(lib):
    import paper_2209_14637_b200 as tsk
    vp = ctypes.c_void_p
    # NULL ctx is rejected synchronously by every entry point
    assert lib.tsk_sync(None) == -8
    assert lib.tsk_destroy(None) == -8
    assert lib.sketch_gram(None, vp(1), 1, 4, 4, vp(1), None, 0, None, None) == -8
    assert lib.sketch_topk(None, vp(1), 4, 2, vp(1), None, None, None) == -8
    assert lib.sketch_train(None, vp(1), 1, 4, 4, 2, vp(1), None, None, None, None) == -8
    assert lib.sketch_apply_scw(None, vp(1), 1, 4, 4, vp(1), 2, 1, None, None, None) == -8
    assert lib.scw_error(None, vp(1), 1, 4, 4, vp(1), 2, 1, vp(1)) == -8
    lib.tsk_set_scw_error_mode.argtypes = [vp, ctypes.c_int, ctypes.c_double]
    assert lib.tsk_set_scw_error_mode(None, 0, 0.0) == -8
    assert lib.tsk_create(None, 0, None) == -8
    # no sm_100 device here: tsk_create reports TSK_EDEVICE instead of falling back to the CPU
    h = ctypes.c_void_p()
    st = lib.tsk_create(ctypes.byref(h), 0, None)
    if not _has_gpu():
        assert st == -6
        with pytest.raises(RuntimeError):
            tsk.Context(0)


def _has_gpu():
    import torch
    return torch.cuda.is_available()
