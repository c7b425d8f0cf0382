"""The C-ABI boundary loads and exports every entry point include/fglt.h
declares; the device code is sm_100a (no compute calls: CPU-only test)."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2007_11111_b200", "libfglt.so")
HDR = os.path.join(ROOT, "include", "fglt.h")


def declared_functions():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fglt_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for must in ("fglt_transform_csr32", "fglt_ctx_transform", "fglt_net_from_raw",
                 "fglt_stage_prepare", "fglt_stage_epilogue"):
        assert must in fns


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_python_binding_lists_all_exports():
    from paper_2007_11111_b200 import _capi
    assert sorted(_capi.EXPORTS) == declared_functions()


def test_no_device_fails_loudly_or_runs():
    """Without a GPU the boundary must refuse (code 7), never compute on CPU."""
    from paper_2007_11111_b200 import _capi
    lib = _capi.lib()
    if lib.fglt_device_count() > 0:
        pytest.skip("a CUDA device is present")
    err = _capi.FgltError()
    h = lib.fglt_ctx_create(0, None, ctypes.byref(err))
    assert not h and err.code == 7


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump absent")
def test_device_code_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_api_and_module_built():
    pkg = os.path.join(ROOT, "paper_2007_11111_b200")
    assert os.path.exists(os.path.join(pkg, "libfglt_host.so"))
    assert any(f.startswith("_core") and f.endswith(".so") for f in os.listdir(pkg))
