"""Planted test tensors restating the reference's generators.hpp (test
infrastructure): core/transfer entries and factor matrices are drawn from
the reference RNG streams (via the oracle's C restatement), factors are
orthonormalised by QR. LAPACK's QR signs may differ from Eigen's
HouseholderQR, so these are the same *distribution* as the reference's
planted tensors, not bitwise the same tensors; every test using them checks
properties (recovery, ranks, orthonormality), as the reference tests do."""
import numpy as np

import srtt_oracle as O


def orthonormalized_random(rows, cols, gaussian, rng):
    """generators.hpp:36-47 (column-major fill, then Q of a QR)."""
    vals = rng.normals(rows * cols) if gaussian else rng.uniform01(rows * cols)
    m = vals.reshape((rows, cols), order="F")
    return np.linalg.qr(m)[0]


def planted_tucker(dims, ranks, seed, kind="uniform"):
    """make_planted_tucker (generators.hpp:51-95)."""
    d = len(dims)
    crng = O.RngStream(seed, 0)
    if kind == "uniform":
        core = crng.uniform01(int(np.prod(ranks))).reshape(ranks, order="F")
    else:
        idx = np.indices(ranks).reshape(d, -1, order="F")
        pts = np.stack([idx[k] / (ranks[k] - 1) if ranks[k] > 1 else 0 * idx[k] for k in range(d)])
        core = (1.0 / (1.0 + (pts ** 2).sum(axis=0))).reshape(ranks, order="F")
    factors = [orthonormalized_random(dims[k], ranks[k], kind != "uniform", O.RngStream(seed, k + 1))
               for k in range(d)]
    x = O.reconstruct(O.TuckerDecomposition(core, factors))
    return x, core, factors


def planted_htucker(dims, tree, ranks, seed):
    """make_planted_htucker (generators.hpp:106-139)."""
    leaf = [None] * len(dims)
    for i in tree.leaves():
        m = tree.node(i).modes[0]
        leaf[m] = orthonormalized_random(dims[m], ranks[i], False, O.RngStream(seed, i))
    transfers = [None] * tree.num_nodes
    for i in range(tree.num_nodes):
        n = tree.node(i)
        if n.is_leaf():
            continue
        rng = O.RngStream(seed, i + 1000003)
        shape = (ranks[i], ranks[n.left], ranks[n.right])
        transfers[i] = rng.uniform01(int(np.prod(shape))).reshape(shape, order="F")
    h = O.HTuckerDecomposition(tree, leaf, transfers)
    return O.ht_reconstruct(h), h


def planted_spectrum(order, n, values, seed):
    """make_planted_spectrum (generators.hpp:160-183)."""
    k = len(values)
    core = np.zeros((k,) * order)
    for i, v in enumerate(values):
        core[(i,) * order] = v
    factors = [orthonormalized_random(n, k, True, O.RngStream(seed, j + 1)) for j in range(order)]
    return O.reconstruct(O.TuckerDecomposition(core, factors))


def random_tensor(dims, seed):
    """oracles.hpp:14-19: uniform in [-1, 1) from stream (seed, 0)."""
    v = O.RngStream(seed, 0).uniform01(int(np.prod(dims)))
    return O.as_tensor(2.0 * v - 1.0, dims)


def random_matrix(rows, cols, seed):
    """oracles.hpp:21-27: uniform in [-1, 1) from stream (seed, 1)."""
    v = O.RngStream(seed, 1).uniform01(rows * cols)
    return (2.0 * v - 1.0).reshape((rows, cols), order="F")
