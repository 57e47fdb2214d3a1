"""Sub-R-RtL-HT on the B200 vs the CPU oracle and test_htucker.cpp."""
import numpy as np
import pytest

import paper_2603_21379_b200 as P
import srtt_oracle as O
from parity import projector_gap
from planted import planted_htucker

pytestmark = pytest.mark.gpu


def median(v):
    return sorted(v)[len(v) // 2]


def as_oracle(h, otree):
    return O.HTuckerDecomposition(otree, h.leaf_factors, h.transfers)


def test_matches_oracle_d4_and_d8(handle):
    for d, n, r, w in [(4, 15, 5, None), (8, 6, 3, 120), (5, 7, 3, 40)]:
        tree, otree = P.DimensionTree.balanced(d), O.DimensionTree.balanced(d)
        x, _ = planted_htucker((n,) * d, otree, O.uniform_node_ranks(otree, r), 11)
        x = x + 1e-9 * np.random.default_rng(2).standard_normal(x.shape)
        ranks = P.uniform_node_ranks(tree, r)
        samples = P.node_sample_counts(tree, x.shape, 20.0) if w is None else \
            [1] + [min(w, tree.node_cols(i, x.shape)) for i in range(1, tree.num_nodes)]
        rep = P.HtSubsampleReport()
        h = P.sub_r_rtl_ht(x, tree, ranks, samples, 4, 3, report=rep, handle=handle)
        orep = O.HtSubsampleReport()
        ho = O.sub_r_rtl_ht(x, otree, ranks, samples, 4, 3, report=orep)
        assert rep.achieved_ranks == orep.achieved_ranks
        for ug, uc in zip(h.leaf_factors, ho.leaf_factors):
            assert projector_gap(ug, uc) <= 1e-10
        eg, ec = O.rel_error(x, O.ht_reconstruct(as_oracle(h, otree))), O.rel_error(x, O.ht_reconstruct(ho))
        assert abs(eg - ec) <= 1e-10 * max(ec, 1.0)
        assert h.transfers[0].shape == (1, r, r)


def test_recovers_planted(handle):
    """test_htucker.cpp:221-237."""
    tree, otree = P.DimensionTree.balanced(4), O.DimensionTree.balanced(4)
    x, _ = planted_htucker((15,) * 4, otree, O.uniform_node_ranks(otree, 5), 11)
    budget = P.node_sample_counts(tree, x.shape, 20.0)
    errs = []
    for seed in range(9):
        rep = P.HtSubsampleReport()
        h = P.sub_r_rtl_ht(x, tree, P.uniform_node_ranks(tree, 5), budget, 4, seed, report=rep, handle=handle)
        errs.append(O.rel_error(x, O.ht_reconstruct(as_oracle(h, otree))))
        assert rep.achieved_ranks[1:] == [5] * 6
    assert median(errs) <= 1e-7


def test_full_sampling_exact_and_determinism(handle):
    """test_htucker.cpp:258-317."""
    tree, otree = P.DimensionTree.balanced(4), O.DimensionTree.balanced(4)
    x, _ = planted_htucker((8,) * 4, otree, O.uniform_node_ranks(otree, 3), 13)
    full = [1] + [tree.node_cols(i, x.shape) for i in range(1, 7)]
    h = P.sub_r_rtl_ht(x, tree, P.uniform_node_ranks(tree, 3), full, 4, 17, handle=handle)
    assert O.rel_error(x, O.ht_reconstruct(as_oracle(h, otree))) <= 1e-9
    budget = P.node_sample_counts(tree, x.shape, 10.0)
    a = P.sub_r_rtl_ht(x, tree, P.uniform_node_ranks(tree, 3), budget, 4, 31, handle=handle)
    b = P.sub_r_rtl_ht(x, tree, P.uniform_node_ranks(tree, 3), budget, 4, 31,
                       P.ExecPolicy(workers=4, emulate_serial_root=True), handle=handle)
    assert all(np.array_equal(u, v) for u, v in zip(a.leaf_factors, b.leaf_factors))
    assert all(np.array_equal(u, v) for u, v in zip(a.transfers, b.transfers) if u is not None)


def test_validation(handle):
    tree = P.DimensionTree.balanced(4)
    x = np.random.default_rng(0).standard_normal((6,) * 4)
    ranks = P.uniform_node_ranks(tree, 2)
    with pytest.raises(P.InvalidArgument, match="samples below rank \\+ oversampling at node 1"):
        P.sub_r_rtl_ht(x, tree, ranks, [1] + [5] * 6, 4, 0, handle=handle)
    bad = list(ranks)
    bad[0] = 2
    with pytest.raises(P.InvalidArgument, match="root rank must be 1"):
        P.sub_r_rtl_ht(x, tree, bad, [1] + [30] * 6, 4, 0, handle=handle)


def test_exec_policy_workers_validated(handle):
    """tree_schedule (parallel.hpp:206) rejects workers < 1; no slice mode is
    involved on the H-Tucker path."""
    tree = P.DimensionTree.balanced(4)
    x = np.random.default_rng(0).standard_normal((6,) * 4)
    ranks = P.uniform_node_ranks(tree, 2)
    with pytest.raises(P.InvalidArgument, match="^tree_schedule: workers must be >= 1$"):
        P.sub_r_rtl_ht(x, tree, ranks, [1] + [30] * 6, 4, 0, P.ExecPolicy(workers=0), handle=handle)
    rep = P.HtSubsampleReport()
    P.sub_r_rtl_ht(x, tree, ranks, [1] + [30] * 6, 4, 0, P.ExecPolicy(workers=3), report=rep, handle=handle)
    assert rep.slice_mode is None


def test_internal_node_bases_reported(handle):
    """The report's node_bases are the bases the decomposition used: leaves
    equal the returned leaf factors bitwise, internal ones match the oracle's
    node bases."""
    tree, otree = P.DimensionTree.balanced(4), O.DimensionTree.balanced(4)
    x, _ = planted_htucker((9,) * 4, otree, O.uniform_node_ranks(otree, 3), 4)
    ranks = P.uniform_node_ranks(tree, 3)
    samples = [1] + [min(30, tree.node_cols(i, x.shape)) for i in range(1, 7)]
    rep = P.HtSubsampleReport(want_node_bases=True)
    h = P.sub_r_rtl_ht(x, tree, ranks, samples, 4, 2, report=rep, handle=handle)
    orep = O.HtSubsampleReport()
    O.sub_r_rtl_ht(x, otree, ranks, samples, 4, 2, report=orep)
    for i in range(1, 7):
        assert projector_gap(rep.node_bases[i], orep.bases[i]) <= 1e-10
        if otree.node(i).is_leaf():
            assert np.array_equal(rep.node_bases[i], h.leaf_factors[otree.node(i).modes[0]])


def test_root_children_ranks_above_32(handle):
    """H-Tucker root pass with r_left, r_right = 40 (> the 32-wide DMMA tiles):
    rank-block passes, parity with the oracle."""
    tree, otree = P.DimensionTree.balanced(4), O.DimensionTree.balanced(4)
    dims = (8, 8, 8, 8)
    ranks = [1, 40, 40, 8, 8, 8, 8]
    x = np.random.default_rng(6).standard_normal(dims)
    samples = [1] + [min(56, tree.node_cols(i, dims)) for i in range(1, 7)]
    rep = P.HtSubsampleReport()
    h = P.sub_r_rtl_ht(x, tree, ranks, samples, 6, 2, report=rep, handle=handle)
    orep = O.HtSubsampleReport()
    ho = O.sub_r_rtl_ht(x, otree, ranks, samples, 6, 2, report=orep)
    assert rep.achieved_ranks == orep.achieved_ranks
    eg, ec = O.rel_error(x, O.ht_reconstruct(as_oracle(h, otree))), O.rel_error(x, O.ht_reconstruct(ho))
    assert abs(eg - ec) <= 1e-10 * max(ec, 1.0)
    assert h.transfers[0].shape == (1, 40, 40)
