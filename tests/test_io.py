"""SRTT / SRHT containers through the C-ABI (reference test_io.cpp:13-112,
io.cpp).  Host buffers only: these run on CPU (the device-streaming read is
covered in test_gpu_io.py)."""
import os

import numpy as np
import pytest

import paper_2603_21379_b200 as P


def test_tensor_header_layout_is_exactly_as_documented(tmp_path):
    """test_io.cpp:13-29."""
    x = (np.arange(6, dtype=np.float64) + 0.5).reshape((2, 3), order="F")
    path = tmp_path / "t.srtt"
    P.write_tensor(path, x)
    b = path.read_bytes()
    assert len(b) == 4 + 4 + 8 + 2 * 8 + 6 * 8
    assert b[:4] == b"SRTT"
    assert b[4] == 1 and b[5] == 0          # version u32 LE
    assert b[8] == 2                         # order u64 LE
    assert b[16] == 2 and b[24] == 3         # dims
    assert np.frombuffer(b[32:], "<f8").tolist() == [0.5, 1.5, 2.5, 3.5, 4.5, 5.5]


def test_tensor_round_trips_bitwise(tmp_path):
    """test_io.cpp:31-38 and :105-112."""
    x = np.random.default_rng(7).standard_normal((3, 4, 5))
    path = tmp_path / "x.srtt"
    P.write_tensor(path, x)
    back = P.read_tensor(path)
    assert back.shape == x.shape
    assert np.array_equal(back, x)
    assert P.tensor_file_info(path) == ([3, 4, 5], 8 + 8 + 3 * 8)


def test_tensor_reader_rejects_corrupt_input(tmp_path):
    """test_io.cpp:40-65."""
    bad = tmp_path / "bad.srtt"
    bad.write_bytes(b"NOPE")
    with pytest.raises(P.IoError):
        P.read_tensor(bad)
    wrong = tmp_path / "ver.srtt"
    wrong.write_bytes(b"SRTT" + bytes([9, 0, 0, 0]))
    with pytest.raises(P.IoError, match="version"):
        P.read_tensor(wrong)
    full = tmp_path / "full.srtt"
    P.write_tensor(full, np.zeros((2, 2)))
    trunc = tmp_path / "trunc.srtt"
    trunc.write_bytes(full.read_bytes()[:-8])
    with pytest.raises(P.IoError):
        P.read_tensor(trunc)
    with pytest.raises(P.IoError):
        P.read_tensor(trunc, slab=(0, 1))     # the readable slab of a truncated file is still corrupt
    with pytest.raises(P.IoError):
        P.read_tensor("/nonexistent/path/tensor.srtt")
    empty = tmp_path / "empty.srtt"
    empty.write_bytes(b"")
    with pytest.raises(P.IoError):
        P.read_tensor(empty)


def test_slab_reads_match_the_full_tensor(tmp_path):
    """A last-mode slab is one contiguous byte range (what a sharded rank reads)."""
    x = np.random.default_rng(1).standard_normal((4, 3, 7))
    path = tmp_path / "s.srtt"
    P.write_tensor(path, x)
    for lo, hi in [(0, 7), (0, 1), (2, 5), (6, 7)]:
        s = P.read_tensor(path, slab=(lo, hi))
        assert s.shape == (4, 3, hi - lo)
        assert np.array_equal(s, x[..., lo:hi])
    with pytest.raises(P.InvalidArgument):
        P.read_tensor(path, slab=(5, 5))
    with pytest.raises(P.InvalidArgument):
        P.read_tensor(path, slab=(3, 8))


def _planted_ht(O, order, n, r, seed):
    tree = O.DimensionTree.balanced(order)
    rng = np.random.default_rng(seed)
    ranks = O.uniform_node_ranks(tree, r)
    leaf = [np.linalg.qr(rng.standard_normal((n, r)))[0] for _ in range(order)]
    trs = [None] * tree.num_nodes
    for i in range(tree.num_nodes):
        nd = tree.node(i)
        if not nd.is_leaf():
            trs[i] = rng.standard_normal((1 if i == 0 else ranks[i], ranks[nd.left], ranks[nd.right]))
    return O.HTuckerDecomposition(tree, leaf, trs)


def test_hierarchical_container_round_trips_bitwise(tmp_path, O):
    """test_io.cpp:67-94 and :96-103."""
    ho = _planted_ht(O, 5, 6, 3, 9)
    hp = P.HTuckerDecomposition(P.DimensionTree.balanced(5), ho.leaf_factors, ho.transfers)
    path = tmp_path / "h.srht"
    P.write_htucker(path, hp)
    assert path.read_bytes()[:4] == b"SRHT"
    back = P.read_htucker(path)
    tree = hp.tree
    assert back.tree.num_nodes == tree.num_nodes
    for i in range(tree.num_nodes):
        assert back.tree.node(i).modes == tree.node(i).modes
        assert back.tree.node(i).left == tree.node(i).left
        assert back.tree.node(i).right == tree.node(i).right
        assert back.tree.node(i).level == tree.node(i).level
    for a, b in zip(back.leaf_factors, ho.leaf_factors):
        assert np.array_equal(a, b)
    for i in range(tree.num_nodes):
        if ho.transfers[i] is not None:
            assert np.array_equal(back.transfers[i], ho.transfers[i])
    # the reloaded decomposition expands to the same tensor (oracle expansion)
    ref = O.ht_reconstruct(ho)
    got = O.ht_reconstruct(O.HTuckerDecomposition(O.DimensionTree.balanced(5), back.leaf_factors, back.transfers))
    assert O.rel_error(ref, got) <= 1e-12


def test_hierarchical_reader_rejects_corrupt_input(tmp_path, O):
    ho = _planted_ht(O, 4, 5, 2, 3)
    hp = P.HTuckerDecomposition(P.DimensionTree.balanced(4), ho.leaf_factors, ho.transfers)
    path = tmp_path / "h.srht"
    P.write_htucker(path, hp)
    raw = path.read_bytes()
    for name, blob in [("magic", b"SRTT" + raw[4:]), ("version", raw[:4] + bytes([2, 0, 0, 0]) + raw[8:]),
                       ("trunc", raw[:-8]), ("tiny", raw[:20])]:
        p = tmp_path / f"{name}.srht"
        p.write_bytes(blob)
        with pytest.raises(P.IoError):
            P.read_htucker(p)
    # implausible tree size (num_nodes > 4 * order)
    p = tmp_path / "size.srht"
    p.write_bytes(raw[:16] + (1000).to_bytes(8, "little") + raw[24:])
    with pytest.raises(P.IoError, match="implausible"):
        P.read_htucker(p)
    with pytest.raises(P.IoError):
        P.read_htucker(os.path.join(str(tmp_path), "missing.srht"))
