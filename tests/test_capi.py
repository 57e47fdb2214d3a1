"""The C-ABI library loads and exports every symbol include/srtt_b200.h
declares; host-only entry points behave like the reference without a GPU."""
import ctypes
import os
import re

import pytest

import paper_2603_21379_b200 as P
from paper_2603_21379_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "srtt_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srtt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 17
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_balanced_trees_match_reference_layouts():
    """test_htucker.cpp:30-60."""
    t2 = P.DimensionTree.balanced(2)
    assert [n.modes for n in t2.nodes] == [[0, 1], [0], [1]] and t2.depth() == 1
    t8 = P.DimensionTree.balanced(8)
    assert t8.num_nodes == 15 and t8.depth() == 3
    assert [t8.node(i).modes for i in range(1, 7)] == [[0, 1, 2, 3], [4, 5, 6, 7], [0, 1], [2, 3], [4, 5], [6, 7]]
    assert len(t8.leaves()) == 8
    t5 = P.DimensionTree.balanced(5)
    assert t5.node(1).modes == [0, 1, 2] and t5.node(2).modes == [3, 4] and t5.depth() == 3
    with pytest.raises(P.InvalidArgument):
        P.DimensionTree.balanced(1)


def test_no_gpu_means_a_loud_error_not_a_fallback():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(P.srtt.CudaError):
        P.Handle(0)
