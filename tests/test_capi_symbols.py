"""The C-ABI library builds, loads without a GPU and exports every entry
point declared in include/hpstep_b200.h (CPU only: no compute calls)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hpstep_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_ ]+\**\s*\**(hps_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_entry_points():
    names = declared()
    for must in ("hps_plan_create", "hps_ops_build", "hps_solve", "hps_leaf_eval", "hps_combine"):
        assert must in names
    assert len(names) >= 18


def test_library_exports_every_declared_symbol():
    from paper_2306_02526_b200 import _build, _lib
    if not os.path.exists(_lib.LIB_PATH):
        _build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert not [n for n in declared() if n not in _lib.SIGNATURES]


def test_library_reports_version_without_gpu():
    from paper_2306_02526_b200 import _lib
    lib = _lib.load()
    assert lib.hps_version() >= 1
    assert lib.hps_launch_count() >= 0
    assert isinstance(_lib.last_error(), str)


def test_product_refuses_to_run_without_cuda(monkeypatch):
    import torch
    import paper_2306_02526_b200 as hb
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 2, 2, 6)
    with pytest.raises(hb.HpstepError, match="CUDA"):
        hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0), sigma=1.0, dt_gamma=0.1)
