"""The CPU oracle restates the reference's property tests for this path
(test_tensor.cpp, test_tucker.cpp, test_htucker.cpp, test_parallel.cpp,
test_sketch.cpp). This pins the oracle's linear algebra where the reference
crosses the Eigen boundary (BDCSVD/GEMM are pinned only to tolerance)."""
import numpy as np
import pytest

import srtt_oracle as O
from planted import planted_htucker, planted_spectrum, planted_tucker, random_matrix, random_tensor


def median(v):
    return sorted(v)[len(v) // 2]


def test_index_maps_and_gathers_bitwise():
    """test_tensor.cpp:12-30, 103-143: gathers equal unfolding columns bitwise."""
    x = random_tensor((3, 4, 5), 23)
    for k in range(3):
        full = O.unfold(x, k)
        # brute-force loop unfolding (oracles.hpp:31-48)
        loop = np.zeros_like(full)
        dims = x.shape
        rest = [dims[j] for j in range(3) if j != k]
        for idx in np.ndindex(*dims):
            ridx = [idx[j] for j in range(3) if j != k]
            col = ridx[0] + rest[0] * ridx[1]
            loop[idx[k], col] = x[idx]
        assert np.array_equal(full, loop)
        cols = O.sample_indices(x.size // dims[k], 7, O.RngStream(99, k))
        assert np.array_equal(O.extract_fibers(x, k, cols), full[:, cols])
    with pytest.raises(IndexError):
        O.extract_fibers(x, 0, [20])
    y = random_tensor((2, 3, 4), 31)
    full = O.extract_group_fibers(y, [0, 2], np.arange(3))
    assert np.array_equal(O.extract_group_fibers(y, [0, 2], [2, 0]), full[:, [2, 0]])
    assert np.array_equal(O.extract_group_fibers(y, [1], [5]), O.extract_fibers(y, 1, [5]))


def test_sub_r_hosvd_recovers_planted():
    """test_tucker.cpp:105-118: 15^4, r=5, s=75, p=4, median <= 1e-8, ranks 5."""
    x, _, _ = planted_tucker((15,) * 4, (5,) * 4, 9)
    errs = []
    for seed in range(9):
        rep = O.SubsampleReport()
        t = O.sub_r_hosvd(x, [5] * 4, 4, [75] * 4, seed, report=rep)
        assert max(O.orthonormality_defect(u) for u in t.factors) <= 1e-10
        assert rep.achieved_ranks == [5] * 4
        errs.append(O.rel_error(x, O.reconstruct(t)))
    assert median(errs) <= 1e-8


def test_full_sampling_saturating_sketch_exact():
    """test_tucker.cpp:120-128."""
    x, _, _ = planted_tucker((9, 9, 9), (4, 4, 4), 13)
    t = O.sub_r_hosvd(x, [4] * 3, 5, [81] * 3, 21)
    assert O.rel_error(x, O.reconstruct(t)) <= 1e-9


def test_validation_and_determinism():
    """test_tucker.cpp:130-163."""
    x = random_tensor((6, 6, 6), 77)
    with pytest.raises(ValueError):
        O.sub_r_hosvd(x, [2] * 3, 4, [5] * 3, 1)
    with pytest.raises(ValueError):
        O.sub_r_hosvd(x, [2] * 3, 4, [37] * 3, 1)
    y, _, _ = planted_tucker((10, 10, 10), (3, 3, 3), 15)
    a = O.sub_r_hosvd(y, [3] * 3, 4, [20] * 3, 42)
    b = O.sub_r_hosvd(y, [3] * 3, 4, [20] * 3, 42)
    assert all(np.array_equal(u, v) for u, v in zip(a.factors, b.factors))
    assert np.array_equal(a.core, b.core)
    serial = O.sub_r_hosvd(y, [3] * 3, 4, [21] * 3, 5, O.ExecPolicy(workers=1, index_partitions=3))
    pooled = O.sub_r_hosvd(y, [3] * 3, 4, [21] * 3, 5, O.ExecPolicy(workers=3, index_partitions=3))
    assert all(np.array_equal(u, v) for u, v in zip(serial.factors, pooled.factors))
    assert O.rel_error(y, O.reconstruct(serial)) <= 1e-9


def test_padding_when_rank_exceeds_data_rank():
    """test_tucker.cpp:165-177."""
    x, _, _ = planted_tucker((8, 8, 8), (2, 2, 2), 19)
    rep = O.SubsampleReport()
    t = O.sub_r_hosvd(x, [4] * 3, 4, [30] * 3, 5, report=rep)
    assert rep.warnings and rep.achieved_ranks == [2, 2, 2]
    assert max(O.orthonormality_defect(u) for u in t.factors) <= 1e-10
    assert O.rel_error(x, O.reconstruct(t)) <= 1e-9


def test_projection_identity():
    """test_tucker.cpp:179-198."""
    x = random_tensor((8, 8, 8), 83)
    t = O.sub_r_hosvd(x, [3, 4, 5], 2, [30] * 3, 3)
    via_core = O.rel_error(x, O.reconstruct(t))
    via_proj = O.rel_error(x, O.multi_ttm(x, [(k, u @ u.T) for k, u in enumerate(t.factors)]))
    assert via_core == pytest.approx(via_proj, rel=1e-12)


def test_sub_r_tracks_t_hosvd():
    """test_tucker.cpp:200-213 (median within 10x of t-hosvd)."""
    x = planted_spectrum(3, 14, [0.6 ** i for i in range(10)], 23)
    us = [np.linalg.svd(O.unfold(x, k), full_matrices=False)[0][:, :4] for k in range(3)]
    det = O.rel_error(x, O.reconstruct(O.TuckerDecomposition(O.core_from_factors(x, us), us)))
    errs = [O.rel_error(x, O.reconstruct(O.sub_r_hosvd(x, [4] * 3, 4, [100] * 3, s))) for s in range(25)]
    assert median(errs) <= 10 * det


def test_sliced_core_equals_multi_ttm_and_is_worker_independent():
    """test_parallel.cpp:68-117."""
    x = random_tensor((8, 8, 8), 91)
    f = [np.linalg.qr(O.gaussian_matrix(8, 3, O.RngStream(92, k)))[0] for k in range(3)]
    ref = O.multi_ttm(x, [(k, f[k].T) for k in range(3)])
    for w in (1, 2, 4):
        assert O.rel_error(ref, O.sliced_core(x, f, O.ExecPolicy(workers=w))) <= 1e-12
    y = random_tensor((6, 7, 5, 4), 93)
    g = [np.linalg.qr(O.gaussian_matrix(n, 2, O.RngStream(94, k)))[0] for k, n in enumerate(y.shape)]
    base = O.sliced_core(y, g, O.ExecPolicy(workers=1, slice_mode=1))
    for w in (2, 3, 7):
        assert np.allclose(O.sliced_core(y, g, O.ExecPolicy(workers=w, slice_mode=1)), base, rtol=0, atol=1e-14)


def test_pick_slice_mode_rules():
    """test_parallel.cpp:119-137."""
    assert O.pick_slice_mode((8, 8, 8), 4) == 0
    assert O.pick_slice_mode((6, 8, 9), 4) == 1
    assert O.pick_slice_mode((6, 8, 9), 5) == 2
    assert O.pick_slice_mode((6, 8, 9), 3) == 0
    with pytest.raises(ValueError):
        O.pick_slice_mode((2, 2), 3)


def test_transfer_tensor_kronecker_oracles():
    """test_htucker.cpp:71-151."""
    ul = np.linalg.qr(O.gaussian_matrix(4, 2, O.RngStream(41, 0)))[0]
    ur = np.linalg.qr(O.gaussian_matrix(3, 2, O.RngStream(42, 0)))[0]
    us = np.kron(ur, ul)  # left-fastest Kronecker: column i = ul(:, i%2) (x) ur(:, i//2)
    b = O.transfer_tensor(us, ul, ur)
    for i in range(4):
        for j in range(2):
            for k in range(2):
                assert b[i, j, k] == pytest.approx(1.0 if i == j + 2 * k else 0.0, abs=1e-12)
    us = random_matrix(9, 2, 43)
    ul = random_matrix(3, 2, 44)
    ur = random_matrix(3, 2, 45)
    b = O.transfer_tensor(us, ul, ur)
    for i in range(2):
        for j in range(2):
            for k in range(2):
                dot = sum(us[a + c * 3, i] * ul[a, j] * ur[c, k] for a in range(3) for c in range(3))
                assert b[i, j, k] == pytest.approx(dot, rel=1e-13)
    xr = random_tensor((4, 3), 53)
    ul = np.linalg.qr(O.gaussian_matrix(4, 2, O.RngStream(51, 0)))[0]
    ur = np.linalg.qr(O.gaussian_matrix(3, 2, O.RngStream(52, 0)))[0]
    br = O.root_transfer(xr, ul, ur)
    for j in range(2):
        for k in range(2):
            dot = sum(xr[a, c] * ul[a, j] * ur[c, k] for a in range(4) for c in range(3))
            assert br[0, j, k] == pytest.approx(dot, rel=1e-13, abs=1e-15)


def test_sub_r_rtl_ht_recovers_planted():
    """test_htucker.cpp:221-256."""
    tree = O.DimensionTree.balanced(4)
    x, _ = planted_htucker((15,) * 4, tree, O.uniform_node_ranks(tree, 5), 11)
    budget = O.node_sample_counts(tree, x.shape, 20.0)
    errs = []
    for seed in range(5):
        rep = O.HtSubsampleReport()
        h = O.sub_r_rtl_ht(x, tree, O.uniform_node_ranks(tree, 5), budget, 4, seed, report=rep)
        errs.append(O.rel_error(x, O.ht_reconstruct(h)))
        assert rep.achieved_ranks[1:] == [5] * 6
    assert median(errs) <= 1e-7
    tree8 = O.DimensionTree.balanced(8)
    y, _ = planted_htucker((6,) * 8, tree8, O.uniform_node_ranks(tree8, 3), 29)
    budget = [1] + [min(120, tree8.node_cols(i, y.shape)) for i in range(1, 15)]
    errs = [O.rel_error(y, O.ht_reconstruct(O.sub_r_rtl_ht(y, tree8, O.uniform_node_ranks(tree8, 3), budget, 4, s)))
            for s in range(3)]
    assert median(errs) <= 1e-7


def test_ht_storage_counts():
    """test_htucker.cpp:398-431 (d=8, n=15, r=5)."""
    tree = O.DimensionTree.balanced(8)
    h = O.HTuckerDecomposition(tree, [np.zeros((15, 5))] * 8,
                               [np.zeros((1 if i == 0 else 5, 5, 5)) if not tree.node(i).is_leaf() else None
                                for i in range(15)])
    assert O.ht_storage_count(h) == 8 * 75 + 6 * 125 + 25


def test_pick_slice_mode_c_abi_matches_reference_rule():
    """srtt_pick_slice_mode (host code of the C-ABI, no GPU needed) vs the
    oracle's restatement of parallel.hpp:331-348, including the error."""
    import paper_2603_21379_b200 as P

    rng = np.random.default_rng(3)
    for _ in range(300):
        d = int(rng.integers(1, 6))
        dims = [int(v) for v in rng.integers(1, 40, size=d)]
        w = int(rng.integers(1, 20))
        try:
            want = O.pick_slice_mode(dims, w)
        except ValueError as e:
            with pytest.raises(P.InvalidArgument, match=str(e)):
                P.pick_slice_mode(dims, w)
            continue
        assert P.pick_slice_mode(dims, w) == want


def test_sliced_core_bitwise_across_workers_and_streamed():
    """sliced_core is bitwise independent of the worker count
    (acceptance.cpp:266-341 property); the slab-streamed variant used for
    C5-size parity equals it, and rel_error_streamed equals rel_error."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((9, 8, 7, 10))
    fs = [np.linalg.qr(rng.standard_normal((n, 3)))[0] for n in x.shape]
    cores = [O.sliced_core(x, fs, O.ExecPolicy(workers=w, slice_mode=sm)) for w in (1, 3, 7) for sm in (0, 3)]
    for c in cores[1:]:
        assert np.abs(c - cores[0]).max() <= 1e-13
    for w in (2, 5):
        assert np.array_equal(O.sliced_core(x, fs, O.ExecPolicy(workers=w, slice_mode=3)),
                              O.sliced_core(x, fs, O.ExecPolicy(workers=1, slice_mode=3)))
    ref = O.core_from_factors(x, fs)
    assert np.abs(cores[0] - ref).max() <= 1e-13

    def read(lo, hi):
        return x[..., lo:hi]

    st = O.sliced_core_streamed(read, x.shape, fs, slab=3)
    assert np.abs(st - ref).max() <= 1e-13
    e1 = O.rel_error_streamed(read, x.shape, ref, fs, slab=4)
    e2 = O.rel_error(x, O.reconstruct(O.TuckerDecomposition(ref, fs)))
    assert abs(e1 - e2) <= 1e-14
