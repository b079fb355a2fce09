"""CPU-side checks of the boundary (no GPU): libmvgs.so builds, loads, and
exports every symbol include/mvgs.h declares; the binding refuses to run
without the library (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mvgs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mvgs_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    import __graft_entry__
    path = __graft_entry__._load_build_module().build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 11
    for s in syms:
        assert hasattr(lib, s), s


def test_binding_symbol_list_matches_header():
    from paper_2506_12727_b200 import mvgs
    assert sorted(mvgs.SYMBOLS) == declared_symbols()


def test_camera_struct_layout_matches_synth():
    import synth
    from paper_2506_12727_b200 import mvgs
    assert synth.CAM_DTYPE.itemsize == mvgs.CAM_BYTES == 76


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2506_12727_b200 import mvgs
    with pytest.raises(mvgs.MvgsError):
        mvgs.create(0)


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2506_12727_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f
