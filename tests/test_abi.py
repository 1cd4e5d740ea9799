"""CPU-side checks of the C ABI boundary: libdinr.so builds, loads, and exports every symbol
include/dinr.h declares; host-only helpers agree with the header's formulas.  No compute
calls (there is no GPU here)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2404_19075_b200 import build, _lib

    build.build()
    return _lib


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dinr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dinr_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("dinr_set_geometry", "dinr_set_field_weights", "dinr_project", "dinr_project_and_grad",
                 "dinr_allreduce_grads"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    import ctypes

    so = ctypes.CDLL(lib.SO_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(so, name), name
    assert sorted(lib.EXPORTS) == syms


def test_param_count_and_status_strings(lib):
    L = lib.load()
    assert lib.param_count(128, 5) == 329217
    assert lib.param_count(32, 3) == 12545
    assert L.dinr_status_string(2) == b"DINR_ERANGE"


def test_no_device_is_reported_not_faked(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lib.DinrError):
        lib.create(0)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2404_19075_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "dinr_oracle" not in txt and "liboracle" not in txt, f
