"""CPU-side checks of the C-ABI boundary (no GPU needed)."""
import ctypes
import os
import subprocess

import pytest

import paper_2402_07033_b200 as M


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(M.lib_path())
    declared = M.declared_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", M.lib_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_library_contains_tma_bulk_copies():
    """The streaming decode kernel must use TMA bulk copies (UBLKCP) and
    mbarrier waits (SYNCS) — proof it is not a plain LDG loop."""
    out = subprocess.run(["cuobjdump", "-sass", M.lib_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "UBLKCP" in sass
    assert "SYNCS" in sass


def test_shape_validation_without_gpu():
    lib = M.lib()
    ok = M.Shape(4, 8, 2, 32, 64, 2).c()
    assert lib.moe_shape_validate(ctypes.byref(ok)) == 0
    bad = M.Shape(4, 8, 9, 32, 64, 2).c()  # top_k > E  (shape.cpp:13-15)
    assert lib.moe_shape_validate(ctypes.byref(bad)) == 1
    bad = M.Shape(-1, 8, 2, 32, 64, 2).c()
    assert lib.moe_shape_validate(ctypes.byref(bad)) == 1
    bad = M.Shape(4, 8, 2, 0, 64, 2).c()
    assert lib.moe_shape_validate(ctypes.byref(bad)) == 1


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(M.MoeError) as ei:
        M.Ctx(0)
    assert ei.value.kind == "NoDevice"


def test_product_never_imports_oracle():
    pkg = os.path.dirname(M.__file__)
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".h", ".cuh", ".hpp")) or fn == "Makefile":
                txt = open(os.path.join(dirpath, fn), errors="ignore").read()
                assert "import oracle" not in txt and "moe_oracle" not in txt, fn
                assert "libmoe_ref" not in txt, fn
