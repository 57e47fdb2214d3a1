"""Sub-R-HOSVD on the B200 vs the CPU oracle and the reference's own
property tests (test_tucker.cpp), through the C-ABI."""
import numpy as np
import pytest

import paper_2603_21379_b200 as P
import srtt_oracle as O
from parity import aligned_core_error, projector_gap, tucker_rel_error
from planted import planted_tucker, random_tensor

pytestmark = pytest.mark.gpu


def median(v):
    return sorted(v)[len(v) // 2]


@pytest.mark.parametrize("dims,r,p,s,seed", [((15,) * 4, 5, 4, 75, 0), ((128, 128, 128), 8, 5, 52, 0),
                                             ((40,) * 4, 6, 5, 44, 3), ((20, 30, 25), 4, 4, 30, 11),
                                             ((9, 9, 9), 4, 5, 81, 21)])
def test_matches_oracle(handle, dims, r, p, s, seed):
    x, _, _ = planted_tucker(dims, (r,) * len(dims), 9)
    x = x + 1e-9 * np.random.default_rng(1).standard_normal(x.shape)
    rep = P.SubsampleReport()
    t = P.sub_r_hosvd(x, [r] * len(dims), p, [s] * len(dims), seed, report=rep, handle=handle)
    orep = O.SubsampleReport()
    to = O.sub_r_hosvd(x, [r] * len(dims), p, [s] * len(dims), seed, report=orep)
    assert rep.achieved_ranks == orep.achieved_ranks
    assert rep.sample_counts == [s] * len(dims)
    for ug, uc in zip(t.factors, to.factors):
        assert projector_gap(ug, uc) <= 1e-10
        assert O.orthonormality_defect(ug) <= 1e-12
    assert aligned_core_error(t.core, t.factors, to.core, to.factors) <= 1e-10
    eg, ec = tucker_rel_error(x, t.core, t.factors), O.rel_error(x, O.reconstruct(to))
    assert abs(eg - ec) <= 1e-10 * max(ec, 1.0)


def test_recovers_planted_from_few_fibers(handle):
    """test_tucker.cpp:105-118."""
    x, _, _ = planted_tucker((15,) * 4, (5,) * 4, 9)
    errs = []
    for seed in range(9):
        rep = P.SubsampleReport()
        t = P.sub_r_hosvd(x, [5] * 4, 4, [75] * 4, seed, report=rep, handle=handle)
        assert rep.achieved_ranks == [5] * 4
        errs.append(tucker_rel_error(x, t.core, t.factors))
    assert median(errs) <= 1e-8


def test_validation_messages_match_reference(handle):
    """test_tucker.cpp:130-136 (tucker.hpp:184-197 order and wording)."""
    x = random_tensor((6, 6, 6), 77)
    with pytest.raises(P.InvalidArgument, match="samples below rank \\+ oversampling in mode 0"):
        P.sub_r_hosvd(x, [2] * 3, 4, [5] * 3, 1, handle=handle)
    with pytest.raises(P.InvalidArgument, match="more samples than fibers in mode 0"):
        P.sub_r_hosvd(x, [2] * 3, 4, [37] * 3, 1, handle=handle)
    with pytest.raises(P.InvalidArgument, match="rank out of range in mode 1"):
        P.sub_r_hosvd(x, [2, 7, 2], 4, [30] * 3, 1, handle=handle)
    with pytest.raises(P.JobError) as e:  # partitioned sampling failure inside mode job 0
        P.sub_r_hosvd(x, [2] * 3, 4, [7] * 3, 1, P.ExecPolicy(index_partitions=8), handle=handle)
    assert e.value.job == 0


def test_deterministic_in_the_seed(handle):
    """test_tucker.cpp:138-163: bitwise identical reruns; partitioned too."""
    x, _, _ = planted_tucker((10, 10, 10), (3,) * 3, 15)
    a = P.sub_r_hosvd(x, [3] * 3, 4, [20] * 3, 42, handle=handle)
    b = P.sub_r_hosvd(x, [3] * 3, 4, [20] * 3, 42, handle=handle)
    assert all(np.array_equal(u, v) for u, v in zip(a.factors, b.factors)) and np.array_equal(a.core, b.core)
    pa = P.sub_r_hosvd(x, [3] * 3, 4, [21] * 3, 5, P.ExecPolicy(workers=1, index_partitions=3), handle=handle)
    pb = P.sub_r_hosvd(x, [3] * 3, 4, [21] * 3, 5, P.ExecPolicy(workers=3, index_partitions=3), handle=handle)
    assert all(np.array_equal(u, v) for u, v in zip(pa.factors, pb.factors))
    assert tucker_rel_error(x, pa.core, pa.factors) <= 1e-9
    po = O.sub_r_hosvd(x, [3] * 3, 4, [21] * 3, 5, O.ExecPolicy(workers=1, index_partitions=3))
    assert max(projector_gap(u, v) for u, v in zip(pa.factors, po.factors)) <= 1e-10


def test_pads_when_rank_exceeds_data_rank(handle):
    """test_tucker.cpp:165-177, with the padded columns equal to the oracle's."""
    x, _, _ = planted_tucker((8, 8, 8), (2, 2, 2), 19)
    rep = P.SubsampleReport()
    t = P.sub_r_hosvd(x, [4] * 3, 4, [30] * 3, 5, report=rep, handle=handle)
    assert rep.achieved_ranks == [2, 2, 2] and len(rep.warnings) == 3
    assert "sketch revealed rank 2 < target 4; basis padded" in rep.warnings[0]
    assert max(O.orthonormality_defect(u) for u in t.factors) <= 1e-10
    assert tucker_rel_error(x, t.core, t.factors) <= 1e-9
    to = O.sub_r_hosvd(x, [4] * 3, 4, [30] * 3, 5)
    assert max(projector_gap(u, v) for u, v in zip(t.factors, to.factors)) <= 1e-10


def test_projection_identity(handle):
    """test_tucker.cpp:179-198."""
    x = random_tensor((8, 8, 8), 83)
    t = P.sub_r_hosvd(x, [3, 4, 5], 2, [30] * 3, 3, handle=handle)
    via_core = tucker_rel_error(x, t.core, t.factors)
    via_proj = O.rel_error(x, O.multi_ttm(x, [(k, u @ u.T) for k, u in enumerate(t.factors)]))
    assert via_core == pytest.approx(via_proj, rel=1e-12)


def test_low_oversampling_warning_and_order1(handle):
    x = random_tensor((30,), 3)
    rep = P.SubsampleReport()
    t = P.sub_r_hosvd(x, [1], 0, [1], 3, report=rep, handle=handle)
    assert rep.warnings[0] == "oversampling below the recommended minimum of 4"
    to = O.sub_r_hosvd(x, [1], 0, [1], 3)
    assert np.allclose(np.abs(t.factors[0]), np.abs(to.factors[0]), atol=1e-14)


def test_device_resident_inputs_and_outputs(handle):
    torch = pytest.importorskip("torch")
    x, _, _ = planted_tucker((20, 20, 20), (3,) * 3, 4)
    xd = torch.from_numpy(np.ravel(x, order="F").copy()).cuda()
    td = P.sub_r_hosvd(xd, [3] * 3, 4, [28] * 3, 1, dims=[20, 20, 20], handle=handle, device_out=True)
    th = P.sub_r_hosvd(x, [3] * 3, 4, [28] * 3, 1, handle=handle)
    assert np.array_equal(td.core.cpu().numpy(), np.ravel(th.core, order="F"))
    for k in range(3):
        assert np.array_equal(td.factors[k].cpu().numpy(), np.ravel(th.factors[k], order="F"))


@pytest.mark.parametrize("use_torch_default_stream", [True, False])
def test_stream_ordered_calls_are_ordered_with_the_callers_stream(use_torch_default_stream):
    """Device-output calls without a report return once enqueued. Bound to
    the caller's stream (torch's default = the legacy stream, or a side
    stream), every call must rewrite its outputs before work the caller
    enqueues afterwards -- also the first calls after a synchronising one,
    when both parameter sets are free (this once ran unordered)."""
    import torch

    dims, r = [40, 36, 30], 5
    x_np, _, _ = planted_tucker(tuple(dims), (r,) * 3, 3)
    h = P.Handle(0, use_graphs=True)
    side = torch.cuda.Stream()
    ctx = torch.cuda.stream(side) if not use_torch_default_stream else torch.cuda.stream(torch.cuda.current_stream())
    with ctx:
        s = torch.cuda.current_stream()
        h.set_stream(s.cuda_stream)
        x = torch.from_numpy(np.ravel(x_np, order="F").copy()).cuda()
        core = torch.empty(r ** 3, dtype=torch.float64, device="cuda")
        facs = [torch.empty(n * r, dtype=torch.float64, device="cuda") for n in dims]

        def call(rep=None):
            P.sub_r_hosvd(x, [r] * 3, 4, [36] * 3, 7, dims=dims, handle=h, device_out=True, out=(core, facs),
                          report=rep)

        call(P.SubsampleReport())  # synchronous reference call
        torch.cuda.synchronize()
        ref = core.cpu().numpy().copy()
        for _ in range(4):
            core.zero_()
            call()
            got = core.cpu().numpy()  # ordered after the call on the caller's stream, no extra sync
            assert np.array_equal(got, ref)


def test_exec_policy_validated_like_the_reference(handle):
    """ExecPolicy on the GPU path: workers / slice_mode never change the
    numbers (parallel.hpp:18-21) but are validated with the reference's
    messages -- run_independent_jobs (parallel.hpp:88), pick_slice_mode
    (:331-348) and sliced_core (:369-373) -- and the resolved slice mode is
    reported."""
    x = random_tensor((6, 7, 8), 5)
    args = ([2] * 3, 4, [12] * 3, 3)
    with pytest.raises(P.InvalidArgument, match="^run_independent_jobs: workers must be >= 1$"):
        P.sub_r_hosvd(x, *args, P.ExecPolicy(workers=0), handle=handle)
    with pytest.raises(P.InvalidArgument, match="^pick_slice_mode: no mode can host 9 slices$"):
        P.sub_r_hosvd(x, *args, P.ExecPolicy(workers=9), handle=handle)
    with pytest.raises(P.InvalidArgument, match="^sliced_core: slice mode out of range$"):
        P.sub_r_hosvd(x, *args, P.ExecPolicy(workers=2, slice_mode=3), handle=handle)
    with pytest.raises(P.InvalidArgument, match="^sliced_core: more workers than slices along the slicing mode$"):
        P.sub_r_hosvd(x, *args, P.ExecPolicy(workers=7, slice_mode=0), handle=handle)
    base = P.sub_r_hosvd(x, *args, handle=handle)
    for pol in [P.ExecPolicy(workers=1), P.ExecPolicy(workers=4), P.ExecPolicy(workers=3, slice_mode=2)]:
        rep = P.SubsampleReport()
        t = P.sub_r_hosvd(x, *args, pol, report=rep, handle=handle)
        want = pol.slice_mode if pol.slice_mode is not None else O.pick_slice_mode(x.shape, pol.workers)
        assert rep.slice_mode == want
        assert np.array_equal(t.core, base.core)
        assert all(np.array_equal(u, v) for u, v in zip(t.factors, base.factors))
    rep = P.SubsampleReport()
    P.sub_r_hosvd(x, *args, report=rep, handle=handle)
    assert rep.slice_mode is None


def test_ranks_above_32_match_oracle(handle):
    """Ranks above the core kernel's 32-wide DMMA tiles (modes 0/1) run as
    rank blocks scattered into the core; parity with the oracle as usual.
    r + p above 256 is refused up front."""
    dims, ranks, p, s = (64, 56, 40), [48, 40, 20], 10, [70, 60, 40]
    x, _, _ = planted_tucker(dims, (48, 40, 20), 9)
    x = x + 1e-10 * np.random.default_rng(3).standard_normal(dims)
    rep = P.SubsampleReport()
    t = P.sub_r_hosvd(x, ranks, p, s, 4, report=rep, handle=handle)
    orep = O.SubsampleReport()
    to = O.sub_r_hosvd(x, ranks, p, s, 4, report=orep)
    assert rep.achieved_ranks == orep.achieved_ranks
    for k in range(3):
        q = rep.achieved_ranks[k]
        assert projector_gap(t.factors[k][:, :q], to.factors[k][:, :q]) <= 1e-9
    assert aligned_core_error(t.core, t.factors, to.core, to.factors) <= 1e-9
    eg, ec = tucker_rel_error(x, t.core, t.factors), tucker_rel_error(x, to.core, to.factors)
    assert abs(eg - ec) <= 1e-10 * max(ec, 1.0)
    # the component: multi_ttm with ranks (40, 36, 5)
    fs = [np.linalg.qr(np.random.default_rng(k).standard_normal((n, r)))[0] for k, (n, r) in
          enumerate(zip(dims, (40, 36, 5)))]
    g = P.multi_ttm_core(x, fs, handle=handle)
    assert np.abs(g - O.core_from_factors(x, fs)).max() <= 1e-12 * np.abs(x).max() * 64
    with pytest.raises(P.InvalidArgument, match="rank \\+ oversampling above 256"):
        P.sub_r_hosvd(np.random.default_rng(1).standard_normal((300, 300, 2)), [8, 8, 2], 250, [400, 400, 90000], 0,
                      handle=handle)


def test_wide_sketches_above_64_columns_match_oracle(handle):
    """r + p above 64 (the register basis kernels' width): the reference bounds
    ranks only by the extents (tucker.hpp:184-197), so the sketch takes
    several 64-column passes and the basis the generic global-memory kernel;
    parity with the oracle as for every other decomposition."""
    dims, ranks, p, s = (96, 90, 20), [70, 66, 12], 8, [100, 90, 30]
    x, _, _ = planted_tucker(dims, (70, 66, 12), 5)
    x = x + 1e-10 * np.random.default_rng(4).standard_normal(dims)
    rep = P.SubsampleReport()
    t = P.sub_r_hosvd(x, ranks, p, s, 7, report=rep, handle=handle)
    orep = O.SubsampleReport()
    to = O.sub_r_hosvd(x, ranks, p, s, 7, report=orep)
    assert rep.achieved_ranks == orep.achieved_ranks
    for k in range(3):
        q = rep.achieved_ranks[k]
        assert O.orthonormality_defect(t.factors[k]) <= 1e-12
        assert projector_gap(t.factors[k][:, :q], to.factors[k][:, :q]) <= 1e-9
    assert aligned_core_error(t.core, t.factors, to.core, to.factors) <= 1e-9
    eg, ec = tucker_rel_error(x, t.core, t.factors), tucker_rel_error(x, to.core, to.factors)
    assert abs(eg - ec) <= 1e-10 * max(ec, 1.0)
