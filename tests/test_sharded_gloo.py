"""Slab-sharded Sub-R-HOSVD orchestration (world_size 2, gloo, CPU).

Drives ``paper_2603_21379_b200.sharded.sub_r_hosvd_sharded`` -- the same
collectives the GPU path issues over NCCL -- with a CHECKER phase backend
built from the oracle (test infrastructure), and compares the sharded result
with the oracle's single-process sub_r_hosvd (tucker.hpp:177-242).  The GPU
phases behind the same orchestration are covered in test_gpu_sharded.py.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OraclePhases:
    """Phase semantics of srtt_shard_sketches / srtt_bases_from_sketches /
    srtt_shard_core restated on the oracle (CPU torch tensors in/out)."""

    def __init__(self):
        import srtt_oracle as O

        self.O = O

    def _embed(self, x_local, dims, lo, hi):
        g = np.zeros(dims, order="F")
        g[..., lo:hi] = x_local.numpy().reshape(tuple(dims[:-1]) + (hi - lo,), order="F")
        return g

    def _stream(self, dims, k, s, c, seed):
        O = self.O
        rng = O.RngStream(seed, k)
        cols = O.sample_indices(int(np.prod(dims)) // dims[k], s, rng)
        omega = O.gaussian_matrix(s, c, rng)
        return rng, cols, omega

    def shard_sketches(self, x_local, dims, lo, hi, ranks, p, samples, seed):
        O = self.O
        g = self._embed(x_local, dims, lo, hi)      # fibres of other slabs contribute zero
        out = []
        for k in range(len(dims)):
            _, cols, omega = self._stream(dims, k, samples[k], ranks[k] + p, seed)
            z = O.extract_fibers(g, k, cols) @ omega
            if k == len(dims) - 1:
                z = z[lo:hi]
            out.append(torch.from_numpy(np.ravel(z, order="F").copy()))
        return out

    def bases_from_sketches(self, dims, ranks, p, samples, seed, zs):
        O = self.O
        us, ach = [], []
        for k in range(len(dims)):
            c = ranks[k] + p
            rng, _, _ = self._stream(dims, k, samples[k], c, seed)
            z = zs[k].numpy().reshape((dims[k], c), order="F")
            b = O.range_basis_of_sketch(z, ranks[k], rng)
            us.append(torch.from_numpy(np.ravel(b.q, order="F").copy()))
            ach.append(b.numerical_rank)
        return us, ach

    def shard_core(self, x_local, dims, lo, hi, ranks, factors):
        O = self.O
        d = len(dims)
        xs = x_local.numpy().reshape(tuple(dims[:-1]) + (hi - lo,), order="F")
        for k in range(d):
            u = factors[k].numpy().reshape((dims[k], ranks[k]), order="F")
            if k == d - 1:
                u = u[lo:hi]
            xs = O.ttm(xs, u.T, k)
        return torch.from_numpy(np.ravel(xs, order="F").copy())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    try:
        for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
            if p not in sys.path:
                sys.path.insert(0, p)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2603_21379_b200 import sharded
        from test_sharded_gloo import OraclePhases

        dims, ranks, p, samples, seed = case
        x = np.random.default_rng(7).standard_normal(dims)
        lo, hi = sharded.slab_bounds(dims[-1], world, rank)
        x_local = torch.from_numpy(np.ravel(x[..., lo:hi], order="F").copy())
        t = sharded.sub_r_hosvd_sharded(x_local, dims, ranks, p, samples, seed, phases=OraclePhases())
        q.put((rank, t.core.numpy(), [u.numpy() for u in t.factors], t.achieved_ranks, t.slab))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e), None, None, None))


CASES = [
    ((6, 5, 7), [3, 2, 3], 2, [9, 8, 10], 11),       # odd last mode: ragged slabs (4 | 3)
    ((8, 6, 5, 9), [2, 3, 2, 3], 3, [10, 12, 9, 14], 3),
]


@pytest.mark.parametrize("case", CASES)
def test_sharded_matches_single_process(case, O):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=240)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r][1], str), res[r][1]

    dims, ranks, p, samples, seed = case
    x = np.random.default_rng(7).standard_normal(dims)
    ref = O.sub_r_hosvd(x, ranks, p, samples, seed)
    for r in range(world):
        _, core, factors, ach, slab = res[r]
        for k in range(len(dims)):
            u = factors[k].reshape((dims[k], ranks[k]), order="F")
            # same sketch up to summation order -> same basis to rounding
            assert np.abs(u - ref.factors[k]).max() < 1e-9
        g = core.reshape(tuple(ranks), order="F")
        assert np.linalg.norm(g - ref.core) <= 1e-10 * np.linalg.norm(ref.core)
    # every rank returns the same decomposition; slabs tile the last mode
    np.testing.assert_array_equal(res[0][1], res[1][1])
    assert res[0][4][0] == 0 and res[0][4][1] == res[1][4][0] and res[1][4][1] == dims[-1]


def test_slab_bounds_match_sliced_core():
    from paper_2603_21379_b200 import sharded

    for n in (1, 5, 7, 64):
        for w in range(1, min(n, 9) + 1):
            b = [sharded.slab_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
    with pytest.raises(ValueError):
        sharded.slab_bounds(3, 4, 0)


# ---------------------------------------------------------------------------
# H-Tucker: column ranges of the root matricization (htucker.hpp:210-341)
# ---------------------------------------------------------------------------
class OracleHtPhases:
    """srtt_ht_shard_sketches / srtt_ht_bases_from_sketches /
    srtt_ht_shard_root restated on the oracle (CPU torch tensors in/out):
    sketch entries outside this rank's flat range contribute zero."""

    def __init__(self):
        import srtt_oracle as O

        self.O = O

    def _stream(self, dims, tree, i, w, c, seed):
        O = self.O
        rng = O.RngStream(seed, i)
        cols = O.sample_indices(tree.node_cols(i, dims), w, rng)
        return rng, cols, O.gaussian_matrix(w, c, rng)

    def shard_sketches(self, x_cols, dims, tree, lo, hi, ranks, p, samples, seed):
        O = self.O
        nl = tree.node_rows(tree.node(0).left, dims)
        flo, fhi = lo * nl, hi * nl
        xl = x_cols.numpy()
        zs = {}
        for i in range(1, tree.num_nodes):
            _, cols, omega = self._stream(dims, tree, i, samples[i], ranks[i] + p, seed)
            offs = O.group_fiber_offsets(dims, tree.node(i).modes, cols)
            inside = (offs >= flo) & (offs < fhi)
            y = np.where(inside, xl[np.clip(offs - flo, 0, xl.size - 1)], 0.0)
            zs[i] = torch.from_numpy(np.ravel(y @ omega, order="F").copy())
        return zs

    def bases_from_sketches(self, dims, tree, ranks, p, samples, seed, zs):
        O = self.O
        us, ach = {}, [1] + [0] * (tree.num_nodes - 1)
        for i in range(1, tree.num_nodes):
            c = ranks[i] + p
            rng, _, _ = self._stream(dims, tree, i, samples[i], c, seed)
            z = zs[i].numpy().reshape((tree.node_rows(i, dims), c), order="F")
            b = O.range_basis_of_sketch(z, ranks[i], rng)
            us[i] = b.q
            ach[i] = b.numerical_rank
        bs = {}
        for i in range(1, tree.num_nodes):
            n = tree.node(i)
            if not n.is_leaf():
                bs[i] = torch.from_numpy(np.ravel(O.transfer_tensor(us[i], us[n.left], us[n.right]), order="F").copy())
        return {i: torch.from_numpy(np.ravel(u, order="F").copy()) for i, u in us.items()}, bs, ach

    def shard_root(self, x_cols, nl, nr, lo, hi, u_left, rl, u_right, rr):
        m = x_cols.numpy().reshape((nl, hi - lo), order="F")
        ul = u_left.numpy().reshape((nl, rl), order="F")
        ur = u_right.numpy().reshape((nr, rr), order="F")[lo:hi]
        return torch.from_numpy(np.ravel(ul.T @ m @ ur, order="F").copy())


def _ht_worker(rank, world, port, case, q):
    try:
        for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
            if p not in sys.path:
                sys.path.insert(0, p)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import srtt_oracle as O
        from paper_2603_21379_b200 import sharded
        from test_sharded_gloo import OracleHtPhases

        dims, r, p, w, seed = case
        tree = O.DimensionTree.balanced(len(dims))
        ranks = O.uniform_node_ranks(tree, r)
        samples = [1] + [min(w, tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
        x = np.random.default_rng(5).standard_normal(dims)
        lo, hi, nl, nr = sharded.column_bounds(tree, dims, world, rank)
        xc = torch.from_numpy(np.ravel(x, order="F")[lo * nl:hi * nl].copy())
        h = sharded.sub_r_rtl_ht_sharded(xc, dims, tree, ranks, samples, p, seed, phases=OracleHtPhases())
        q.put((rank, [u.numpy() for u in h.leaf_factors],
               [None if t is None else t.numpy() for t in h.transfers], h.achieved_ranks, h.columns))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put((rank, traceback.format_exc(), None, None, None))


HT_CASES = [
    ((4, 5, 3, 6), 2, 2, 12, 3),        # n_right = 18 columns -> 9 | 9
    ((3, 4, 2, 5, 3), 2, 2, 14, 8),     # order 5, n_right = 30 ... ragged tree
]


@pytest.mark.parametrize("case", HT_CASES)
def test_htucker_sharded_matches_single_process(case, O):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ht_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=240)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r][1], str), res[r][1]
    dims, rk, p, w, seed = case
    tree = O.DimensionTree.balanced(len(dims))
    ranks = O.uniform_node_ranks(tree, rk)
    samples = [1] + [min(w, tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
    x = np.random.default_rng(5).standard_normal(dims)
    orep = O.HtSubsampleReport()
    ref = O.sub_r_rtl_ht(x, tree, ranks, samples, p, seed, report=orep)
    for r in range(world):
        _, leaf, trs, ach, cols = res[r]
        assert ach == orep.achieved_ranks
        for m in range(len(dims)):
            u = leaf[m].reshape((dims[m], ranks[[i for i in tree.leaves() if tree.node(i).modes[0] == m][0]]),
                                order="F")
            assert np.linalg.norm(u @ u.T - ref.leaf_factors[m] @ ref.leaf_factors[m].T) < 1e-9
        hd = O.HTuckerDecomposition(tree, [leaf[m].reshape(ref.leaf_factors[m].shape, order="F")
                                           for m in range(len(dims))],
                                    [None if t is None else t.reshape(ref.transfers[i].shape, order="F")
                                     for i, t in enumerate(trs)])
        e1 = O.rel_error(x, O.ht_reconstruct(hd))
        e2 = O.rel_error(x, O.ht_reconstruct(ref))
        assert abs(e1 - e2) <= 1e-10 * max(e2, 1.0)
    np.testing.assert_array_equal(res[0][2][0], res[1][2][0])   # same root on both ranks
    assert res[0][4][0] == 0 and res[0][4][1] == res[1][4][0]
