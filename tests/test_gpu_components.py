"""GPU parity of each kernel through the C-ABI against the CPU oracle on
identical inputs."""
import numpy as np
import pytest

import paper_2603_21379_b200 as P
import srtt_oracle as O
from parity import projector_gap
from planted import random_tensor

pytestmark = pytest.mark.gpu
rng = np.random.default_rng(0)


def test_device_gaussian_stream_matches_reference_stream(handle):
    for seed, sid, m, s in [(0, 0, 16384, 52), (0, 7, 35831808, 60), (123, 5, 1000, 999), (9, 1, 3, 1)]:
        st = O.RngStream(seed, sid)
        O.sample_indices(m, s, st)
        ref = st.normals(301)
        _, draws = P.sample_indices(m, s, seed, sid)
        dev = P.stream_normals(seed, sid, draws, 0, 301, handle=handle)
        # same stream, same pair/cos/sin assignment; CUDA vs glibc log/sin/cos differ by ulps
        assert np.max(np.abs(dev - ref) / np.maximum(1.0, np.abs(ref))) <= 4e-16
        # odd offset continues with the cached sine (padding after an odd count)
        assert np.allclose(P.stream_normals(seed, sid, draws, 1, 10, handle=handle), ref[1:11], rtol=0, atol=1e-15)


@pytest.mark.parametrize("dims", [(12, 10, 14), (3, 4, 5), (7, 1, 9, 2), (40, 40, 40)])
def test_fiber_gathers_bitwise(handle, dims):
    """test_tensor.cpp:103-143 on the device: a pure copy, bitwise."""
    x = random_tensor(dims, 5)
    for k in range(len(dims)):
        ncols = x.size // dims[k]
        cols = O.sample_indices(ncols, min(7, ncols), O.RngStream(99, k))
        assert np.array_equal(P.extract_fibers(x, k, cols, handle=handle), O.extract_fibers(x, k, cols))
    if len(dims) >= 3:
        for modes in ([0, 2], [1, 2], [0, 1]):
            ncols = x.size // int(np.prod([dims[m] for m in modes]))
            cols = np.arange(ncols)[::-1].copy()
            assert np.array_equal(P.extract_group_fibers(x, modes, cols, handle=handle),
                                  O.extract_group_fibers(x, modes, cols))
    with pytest.raises(P.OutOfRange):
        P.extract_fibers(x, 0, [x.size // dims[0]], handle=handle)


@pytest.mark.parametrize("dims,modes,w,c", [((128, 128, 128), [0], 52, 13), ((128, 128, 128), [2], 52, 13),
                                            ((40,) * 5, [3], 44, 11), ((12,) * 6, [0, 1, 2], 60, 15),
                                            ((12,) * 6, [3, 4], 60, 15), ((9, 8, 7, 6), [1, 3], 25, 20),
                                            ((30, 20, 10), [1], 200, 42), ((30, 20, 10), [1], 250, 100),
                                            ((64, 80, 90), [0], 3000, 80),
                                            # many fibres: split over CTAs (fixed-order partial sums)
                                            ((64, 80, 90), [0], 6000, 42), ((64, 80, 90), [1], 5000, 13),
                                            ((63, 81, 90), [0], 6000, 21), ((7, 9, 5, 2000), [0, 1, 2], 1500, 15),
                                            ((12,) * 6, [0, 1, 2], 1728, 15), ((12,) * 6, [3, 4, 5], 1728, 15)])
def test_fused_sketch_matches_oracle(handle, dims, modes, w, c):
    """K1: Z = Y(cols) Omega with Omega from the reference stream; Z within 1e-13."""
    x = rng.standard_normal(dims)
    sid = 3
    ncols = x.size // int(np.prod([dims[m] for m in modes]))
    st = O.RngStream(0, sid)
    cols = O.sample_indices(ncols, w, st)
    y = O.extract_group_fibers(x, modes, cols)
    omega = O.gaussian_matrix(w, c, st)
    zo = y @ omega
    z = P.sketch(x, modes, cols, c, 0, sid, P.sample_indices(ncols, w, 0, sid)[1], handle=handle)
    assert np.linalg.norm(z - zo) / np.linalg.norm(zo) <= 1e-13
    z2 = P.sketch(x, modes, cols, c, 0, sid, 0, omega=omega, handle=handle)  # explicit Omega path
    assert np.linalg.norm(z2 - zo) / np.linalg.norm(zo) <= 1e-13


@pytest.mark.parametrize("n,c,r,decay", [(40, 11, 6, 6), (128, 13, 8, 8), (200, 20, 12, 12), (12, 15, 10, 15),
                                         (144, 15, 10, 10), (2048, 42, 32, 32), (5000, 42, 32, 14),
                                         (20736, 15, 10, 10), (3, 5, 2, 3), (1000, 24, 16, 24), (700, 32, 30, 20),
                                         (300, 80, 70, 40), (60, 100, 50, 60), (100000, 15, 10, 10),
                                         (9000, 30, 20, 12), (1500, 16, 16, 16),
                                         # edges of the kernel families
                                         (1, 1, 1, 1), (5, 1, 1, 1), (2, 2, 2, 2), (33, 32, 32, 32), (65, 33, 20, 33),
                                         (256, 64, 50, 64), (257, 64, 64, 30), (129, 16, 9, 16), (64, 17, 17, 5),
                                         # so tall that the stacked top no longer fits one CTA: shared-memory TSQR levels
                                         (1200000, 15, 10, 10)])
def test_basis_matches_oracle(handle, n, c, r, decay):
    """K2 (sketch.hpp:74-93): same numerical rank, same leading subspace,
    orthonormal to 1e-12 (test_sketch.cpp:198-204); covers the warp path,
    the multi-level TSQR path and wide sketches (n < c)."""
    k = min(n, c)
    u0 = np.linalg.qr(rng.standard_normal((n, k)))[0]
    v0 = np.linalg.qr(rng.standard_normal((c, k)))[0]
    sv = np.concatenate([np.logspace(0, -6, min(decay, k)), 1e-10 * np.ones(k - min(decay, k))])
    z = u0 @ np.diag(sv) @ v0.T
    b = P.range_basis_of_sketch(z, r, 0, 1, 0, 0, handle=handle)
    bo = O.range_basis_of_sketch(z, r, O.RngStream(0, 1))
    assert b.numerical_rank == bo.numerical_rank
    q = min(r, b.numerical_rank)
    # perturbation theory: the leading q-subspace is defined only to ~eps*sigma_1/gap
    svo = bo.singular_values
    gap = svo[q - 1] - (svo[q] if q < len(svo) else 0.0)
    tol = max(1e-12, 1e3 * np.finfo(float).eps * svo[0] / gap)
    assert projector_gap(b.q[:, :q], bo.q[:, :q]) <= tol
    assert O.orthonormality_defect(b.q) <= 1e-12
    assert np.allclose(b.singular_values, bo.singular_values[:k], rtol=0, atol=1e-13 * sv[0])


def test_basis_padding_matches_oracle(handle):
    """test_sketch.cpp:103-113: rank-1 sketch, r = 3: rank 1 reported, q has
    3 orthonormal columns, padding continues the same stream."""
    y = np.zeros((10, 6))
    y[:, 0] = 1.0
    st = O.RngStream(22, 0)
    bo = O.range_basis_of_sketch(y[:, :5], 3, st)
    b = P.range_basis_of_sketch(y[:, :5], 3, 22, 0, 0, 0, handle=handle)
    assert b.numerical_rank == 1 == bo.numerical_rank
    assert O.orthonormality_defect(b.q) <= 1e-12
    assert projector_gap(b.q, bo.q) <= 1e-12  # padded columns come from the same normals
    with pytest.raises(P.InvalidArgument):
        P.range_basis_of_sketch(y, 7, handle=handle)


@pytest.mark.parametrize("dims,ranks", [((8, 8, 8), (3, 3, 3)), ((6, 7, 5, 4), (2, 2, 2, 2)),
                                        ((40, 40, 40, 40), (6, 6, 6, 6)), ((15, 15, 15, 15), (5, 5, 5, 5)),
                                        ((128, 64, 32), (8, 9, 10)), ((300, 20, 16), (12, 7, 5)),
                                        ((9, 10, 11, 12, 13), (3, 4, 5, 6, 7)), ((17, 33), (5, 31))])
def test_core_pass_matches_multi_ttm(handle, dims, ranks):
    """K3 == core_from_factors / sliced_core (test_parallel.cpp:68-117) within
    1e-12 relative, incl. odd mode-0 extents (warp-copy loads), row blocks
    (n0 > 256), fold depths 2 and 3 with tails."""
    x = rng.standard_normal(dims)
    f = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in zip(dims, ranks)]
    ref = O.core_from_factors(x, f)
    core = P.multi_ttm_core(x, f, handle=handle)
    assert np.linalg.norm(core - ref) / np.linalg.norm(ref) <= 1e-12
    again = P.multi_ttm_core(x, f, handle=handle)
    assert np.array_equal(core, again)  # fixed-order reductions: bitwise reproducible


def test_transfer_and_root_transfer(handle):
    """K4 / K5 vs the explicit Kronecker inner products (test_htucker.cpp:87-151)."""
    for nl, nr, rs, rl, rr in [(3, 3, 2, 2, 2), (144, 144, 10, 10, 10), (12, 12, 10, 10, 10), (7, 600, 4, 3, 5)]:
        us, ul, ur = rng.standard_normal((nl * nr, rs)), rng.standard_normal((nl, rl)), rng.standard_normal((nr, rr))
        b = P.transfer_tensor(us, ul, ur, handle=handle)
        bo = O.transfer_tensor(us, ul, ur)
        assert np.max(np.abs(b - bo)) <= 1e-13 * max(1.0, np.max(np.abs(bo)))
    for nl, nr in [(4, 3), (144, 20736 // 144), (2000, 333)]:
        x = rng.standard_normal((nl, nr))
        ul = np.linalg.qr(rng.standard_normal((nl, 2)))[0]
        ur = np.linalg.qr(rng.standard_normal((nr, 3)))[0]
        b = P.root_transfer(x, ul, ur, handle=handle)
        assert np.max(np.abs(b - O.root_transfer(x, ul, ur))) <= 1e-12


@pytest.mark.parametrize("mode", ["items", "flat", "flat_swizzled"])
@pytest.mark.parametrize("dims,ranks", [((40, 40, 30, 7), (6, 6, 6, 3)), ((42, 9, 11, 13), (5, 4, 3, 2)),
                                        ((6, 70, 33), (2, 8, 5)), ((22, 17, 150), (8, 7, 9)),
                                        ((40, 40, 40, 40), (6, 6, 6, 6)), ((200, 30, 31), (12, 10, 9))])
def test_core_pass_work_decompositions(handle, monkeypatch, mode, dims, ranks):
    """The planner's core-pass variants agree with multi_ttm (1e-12) and are
    bitwise reproducible: item mode (CTA barriers per item), flat mode
    (per-warp tile ranges, in-kernel record reduction with group counters;
    groups covered by many warps and ragged last tiles) with whole-column
    boxes (n0 = 2 mod 4 pitch) or 16-row swizzled boxes."""
    monkeypatch.setenv("SRTT_FORCE_FLAT", "0" if mode == "items" else "1")
    monkeypatch.setenv("SRTT_FORCE_CB", "0" if mode == "flat_swizzled" else "1")
    x = rng.standard_normal(dims)
    f = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in zip(dims, ranks)]
    ref = O.core_from_factors(x, f)
    core = P.multi_ttm_core(x, f, handle=handle)
    assert np.linalg.norm(core - ref) / np.linalg.norm(ref) <= 1e-12
    assert np.array_equal(core, P.multi_ttm_core(x, f, handle=handle))
