"""The drop-in boundary: libpsdf.so loads without a GPU and exports every
symbol include/psdf.h declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "psdf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psdf_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header():
    from paper_2412_10084_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH), "libpsdf.so not built (run __graft_entry__.build())"
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == syms, set(_lib.EXPORTS) ^ set(syms)


def test_abi_version_and_sizes():
    from paper_2412_10084_b200 import _lib
    L = _lib.load()
    assert L.psdf_abi_version() == 1
    # decoder.hpp:17-31 sizes: in = n_s + n_a + 6
    assert L.psdf_mlp_size(4, 4, 0) == 32 * 14 + 32 + 1024 + 32 + 96 + 3
    assert L.psdf_mlp_size(2, 2, 3) == 32 * 10 + 32 + 1024 + 32 + 96 + 3 + 3 * 32
    assert ctypes.sizeof(_lib.psdf_camera) == 8 * 4 + 8 + 8 * 9 + 8 * 3 + 8
    assert ctypes.sizeof(_lib.psdf_grid_desc) == 4 * 8 + 8 * 5 + 8


def test_errors_without_gpu_are_loud():
    """No CPU fallback: with no usable device, creating a context fails."""
    import pytest
    from paper_2412_10084_b200 import api, _lib
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.PsdfError):
        api.Context(0)


def test_no_oracle_in_product():
    """The product package never imports the checkers under oracle/."""
    pkg = os.path.join(ROOT, "paper_2412_10084_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "psdf_oracle" not in txt and "sdfrecon_ref" not in txt, f
