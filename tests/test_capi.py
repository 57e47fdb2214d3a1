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


def test_basis_planner_picks_the_kernel_family_by_shape():
    """Host logic of K2 (no GPU): sketches with c <= 32 take the register tree
    (one CTA while the level-0 reflectors fit shared memory, else factor CTAs
    + one top CTA), 32 < c <= 64 the 8-warp teams on 256-row blocks, wider
    ones the generic kernel, and shapes whose top would not fit one CTA fall
    back to the shared-memory TSQR levels. BASELINE shapes: C1-C5."""
    lib = ctypes.CDLL(_lib.LIB_PATH)
    lib.srtt_debug_basis_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
    lib.srtt_last_error.restype = ctypes.c_char_p

    def plan(n, c, r):
        out = (ctypes.c_int64 * 5)()
        assert lib.srtt_debug_basis_plan(n, c, r, out) == 0, lib.srtt_last_error()
        return list(out)

    for n, c, r in [(128, 13, 8), (40, 11, 6), (200, 20, 12), (144, 15, 10), (12, 15, 10)]:
        kind, levels, ncta, rpc, top = plan(n, c, r)
        assert (kind, levels, ncta, top) == (1, 0, 1, n)
    kind, levels, ncta, rpc, top = plan(20736, 15, 10)          # C4 level-1 nodes
    assert (kind, levels) == (1, 1) and rpc % 128 == 0 and ncta == -(-20736 // rpc)
    assert top == (ncta - 1) * 15 + min(20736 - (ncta - 1) * rpc, 15) and top <= 4096
    kind, levels, ncta, rpc, top = plan(2048, 42, 32)           # C5 modes
    assert (kind, levels, ncta, rpc, top) == (2, 2, 8, 256, 84)
    assert plan(100, 42, 32)[:2] == [2, 0]
    assert plan(300, 80, 70)[:2] == [3, 0] and plan(60, 100, 50)[:2] == [3, 0]
    kind, levels, ncta, rpc, top = plan(5_000_000, 15, 10)      # top would not fit one CTA
    assert kind == 0 and levels >= 2
    kind, levels, ncta, rpc, top = plan(400_000, 15, 10)        # several row blocks per factor warp
    assert kind == 1 and levels == 1 and rpc > 512 and top <= 4096
    out = (ctypes.c_int64 * 5)()
    assert lib.srtt_debug_basis_plan(10, 300, 5, out) != 0      # wider than SRTT_MAX_SKETCH_COLS
