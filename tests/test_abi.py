"""C-ABI library checks that need no GPU: it builds, loads, exports every declared symbol,
validates arguments synchronously, and refuses (no CPU fallback) without a device."""
import ctypes
import os
import re

import pytest

from paper_2006_13714_b200 import bm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "sc_bm.h")).read()
    return sorted(set(re.findall(r"^(?:sc_status_t|const char\*)\s+(sc_\w+)\s*\(", hdr, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2006_13714_b200 import build
    build.build()
    return bm.load_library()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(bm.EXPORTED)


def test_status_strings(lib):
    for code, name in bm.STATUS.items():
        assert bm.status_string(code) == name
    assert bm.status_string(99) == "SC_ERR_UNKNOWN"


@pytest.mark.parametrize("args", [
    (64, 64, 1, 0, 4, 21, 16, 0),     # b = 0
    (64, 64, 1, 17, 4, 21, 16, 0),    # b > 16
    (64, 64, 9, 8, 4, 21, 16, 0),     # C > 8
    (64, 64, 1, 8, 0, 21, 16, 0),     # stride 0
    (64, 64, 1, 8, 4, 0, 16, 0),      # window 0
    (64, 64, 1, 8, 4, 21, 0, 0),      # K = 0
    (64, 64, 1, 8, 4, 21, 129, 0),    # K > 128
    (7, 64, 1, 8, 4, 21, 16, 0),      # H < b
    (64, 64, 1, 8, 4, 21, 16, 7),     # bad dtype
    (70000, 70000, 1, 8, 4, 21, 16, 0),  # H*W >= 2^31
])
def test_plan_validation(lib, args):
    h = ctypes.c_void_p(123)
    rc = lib.sc_bm_plan(*args, ctypes.byref(h))
    assert rc == 1  # SC_ERR_INVALID_ARGUMENT, before any device query
    assert not h.value


def test_null_handles(lib):
    assert lib.sc_bm_plan(64, 64, 1, 8, 4, 21, 16, 0, None) == 1
    assert lib.sc_bm_run(None, None, None, None, None) == 1
    assert lib.sc_bm_plan_info(None, None) == 1
    assert lib.sc_bm_destroy(None) == 0


def test_no_cpu_fallback_without_gpu(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(bm.ScError) as e:
        bm.Plan(64, 64, 1, 8, 4, 21, 16, "u8")
    assert e.value.code in (2, 4)


def test_sm100a_code_in_library(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bm.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("args", [
    (64, 64, 1, 6, 1, 30, 0, 9, 16, 1),    # z_stride 0
    (64, 64, 1, 6, 1, 30, 1, 0, 16, 1),    # z_window 0
    (64, 64, 1, 6, 1, 30, 1, 65, 16, 1),   # z_window > 64
])
def test_plan3d_validation(lib, args):
    h = ctypes.c_void_p(123)
    assert lib.sc_bm_plan3d(*args, ctypes.byref(h)) == 1 and not h.value
    assert lib.sc_bm_run3d(None, None, 0, None, None, None) == 1


def test_plan3d_no_cpu_fallback_without_gpu(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    assert lib.sc_bm_plan3d(64, 64, 1, 6, 1, 30, 1, 9, 16, 0, ctypes.byref(h)) == 2  # uint8: unsupported
    with pytest.raises(bm.ScError) as e:
        bm.Plan3D(64, 64, 1, 6, 1, 30, 1, 9, 16)
    assert e.value.code in (2, 4)
