"""GPU reconstruct / ht_reconstruct / rel_error vs the oracle (SURVEY §8f
row 1; reference tucker.hpp:18-28, htucker.hpp:346-378, tensor.hpp:241-249,
experiment.cpp:248/266).  The streamed errors never materialise X-hat."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tucker(rng, dims, ranks):
    core = rng.standard_normal(ranks)
    factors = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in zip(dims, ranks)]
    return core, factors


TUCKER_CASES = [
    ((7, 5), (3, 2)),
    ((40, 33, 21), (6, 5, 4)),
    ((8, 8, 8, 8, 8), (2, 2, 2, 2, 2)),          # small leading extent -> wider leading split
    ((130, 9, 140), (12, 9, 7)),                 # r = n in one mode, ragged 128-tiles
    ((5, 6, 7, 4), (5, 6, 7, 4)),                # full ranks
    ((257, 3, 129), (17, 2, 33)),                # K > one 16-chunk, ragged K chunk
]


@pytest.mark.parametrize("dims,ranks", TUCKER_CASES)
def test_tucker_reconstruct_matches_oracle(dims, ranks, O):
    import paper_2603_21379_b200 as P

    rng = np.random.default_rng(sum(dims))
    core, factors = _tucker(rng, dims, ranks)
    ref = O.reconstruct(O.TuckerDecomposition(core, factors))
    got = P.reconstruct(P.TuckerDecomposition(core, factors))
    assert got.shape == tuple(dims)
    assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())

    x = ref + 1e-6 * rng.standard_normal(dims)
    want = O.rel_error(x, ref)
    e = P.tucker_rel_error(x, P.TuckerDecomposition(core, factors))
    assert abs(e - want) <= 1e-10 * max(want, 1.0) and abs(e - want) <= 1e-6 * want
    assert abs(P.rel_error(x, ref) - want) <= 1e-12 * want


def test_tucker_rel_error_device_inputs(O):
    import torch

    import paper_2603_21379_b200 as P

    dims, ranks = (48, 40, 36), (5, 4, 6)
    rng = np.random.default_rng(4)
    core, factors = _tucker(rng, dims, ranks)
    ref = O.reconstruct(O.TuckerDecomposition(core, factors))
    x = ref + 1e-8 * rng.standard_normal(dims)
    dev = lambda a: torch.from_numpy(np.ravel(a, order="F").copy()).cuda()  # noqa: E731
    t = P.TuckerDecomposition(dev(core), [dev(u) for u in factors])
    e = P.tucker_rel_error(dev(x), t, dims=list(dims))
    want = O.rel_error(x, ref)
    assert abs(e - want) <= 1e-6 * want
    xh = P.reconstruct(t, dims=list(dims), device_out=True)
    assert xh.is_cuda and np.abs(xh.cpu().numpy() - np.ravel(ref, order="F")).max() < 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("order,n,r", [(2, 9, 3), (3, 7, 2), (4, 6, 3), (5, 5, 2), (8, 3, 2)])
def test_ht_reconstruct_matches_oracle(order, n, r, O):
    import paper_2603_21379_b200 as P

    dims = [n] * order
    rng = np.random.default_rng(order * 10 + n)
    x = rng.standard_normal(dims)
    tree_o = O.DimensionTree.balanced(order)
    ranks = O.uniform_node_ranks(tree_o, r)
    ranks = [min(ranks[i], tree_o.node_rows(i, dims), tree_o.node_cols(i, dims)) if i else 1
             for i in range(tree_o.num_nodes)]
    samples = [1] + [min(4 * (ranks[i] + 3), tree_o.node_cols(i, dims)) for i in range(1, tree_o.num_nodes)]
    ho = O.sub_r_rtl_ht(x, tree_o, ranks, samples, 3, 5)
    ref = O.ht_reconstruct(ho)
    tree = P.DimensionTree.balanced(order)
    hp = P.HTuckerDecomposition(tree, ho.leaf_factors, ho.transfers)
    got = P.ht_reconstruct(hp)
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    want = O.rel_error(x, ref)
    e = P.ht_rel_error(x, hp)
    assert abs(e - want) <= 1e-10 * max(want, 1.0)


def test_ht_rel_error_of_gpu_decomposition(O):
    """End to end: GPU sub_r_rtl_ht -> GPU ht_rel_error vs oracle numbers."""
    import paper_2603_21379_b200 as P

    dims = [6] * 6
    rng = np.random.default_rng(2)
    terms = [[rng.standard_normal(6) for _ in dims] for _ in range(3)]
    x = sum(np.einsum("a,b,c,d,e,f->abcdef", *t) for t in terms)
    x = x + 1e-9 * np.linalg.norm(x) / np.sqrt(x.size) * rng.standard_normal(dims)
    tree = P.DimensionTree.balanced(6)
    ranks = P.uniform_node_ranks(tree, 3)
    samples = [1] + [min(4 * 8, tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
    hg = P.sub_r_rtl_ht(x, tree, ranks, samples, 5, 1)
    e = P.ht_rel_error(x, hg)
    want = O.rel_error(x, O.ht_reconstruct(O.HTuckerDecomposition(O.DimensionTree.balanced(6), hg.leaf_factors,
                                                                  hg.transfers)))
    assert abs(e - want) <= 1e-10 * max(want, 1.0)
    assert e < 1e-6


def test_rel_error_zero_norm_raises():
    import paper_2603_21379_b200 as P

    z = np.zeros((4, 5))
    with pytest.raises(P.InvalidArgument):
        P.rel_error(z, np.ones((4, 5)))
    with pytest.raises(P.InvalidArgument):
        P.rel_error(np.ones((4, 5)), np.ones((5, 4)))
    core, factors = _tucker(np.random.default_rng(0), (4, 5), (2, 2))
    with pytest.raises(P.InvalidArgument):
        P.tucker_rel_error(z, P.TuckerDecomposition(core, factors))


@pytest.mark.parametrize("cfg_name", ["c1", "c2"])
def test_config_rel_error_matches_oracle(cfg_name, O):
    """Full BASELINE configs: GPU decomposition, error streamed on the GPU vs
    the oracle's rel_error(x, reconstruct(t)) of the same decomposition."""
    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import synth

    cfg = synth.CONFIGS[cfg_name]
    xf = synth.make_tensor(cfg, seed=0, backend="numpy")
    x = O.as_tensor(xf, cfg.dims)
    t = P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0)
    e = P.tucker_rel_error(x, t)
    want = O.rel_error(x, O.reconstruct(O.TuckerDecomposition(t.core, t.factors)))
    assert abs(e - want) <= 1e-10 * max(want, 1.0)
