"""The C-ABI library loads, exports every symbol include/trigpu.h declares,
and reports errors without a GPU. No compute calls. CPU only."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2203_04774_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "trigpu.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"TL_API\s+[\w\s\*]+?\b(tl_\w+)\s*\(", src)))


def test_header_declares_the_documented_surface():
    assert declared_symbols() == sorted(_native.TRIGPU_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _native.trigpu()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
    out = subprocess.run(["nm", "-D", "--defined-only", _native.TRIGPU_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(declared_symbols()) <= exported
    # hidden visibility: no kernel / helper symbols leak
    assert all(s.startswith("tl_") for s in exported if not s.startswith("_"))


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.TRIGPU_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_size_check():
    lib = _native.trigpu()
    assert lib.tl_version() == 1
    assert lib.tl_check_sizes(5, 5) == _native.TL_OK
    # oriented_view.cpp:8-9: size mismatch is an invalid argument
    assert lib.tl_check_sizes(5, 4) == _native.TL_ERR_INVALID_ARGUMENT


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _native.trigpu()
    p = C.c_void_p()
    rc = lib.tl_create(C.byref(p), 0)
    assert rc == _native.TL_ERR_CUDA
    assert not p.value
    assert b"CUDA" in lib.tl_last_error(None) or b"device" in lib.tl_last_error(None)


def test_null_context_is_rejected():
    lib = _native.trigpu()
    assert lib.tl_list(None, 1, 0, None) == _native.TL_ERR_INVALID_ARGUMENT
    assert lib.tl_orient(None, 0, 0, None, None, None) == _native.TL_ERR_INVALID_ARGUMENT


def test_python_api_raises_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2203_04774_b200 as tg
    with pytest.raises(tg.TrigpuError):
        tg.Context(0)
