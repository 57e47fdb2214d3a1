"""Slab-sharded phases on the GPU (srtt_shard_sketches / srtt_bases_from_sketches
/ srtt_shard_core).  One GPU: the W shards run one after another on the same
device and the exchanges (sum / row concatenation) are done here -- the
kernels of one shard never wait on another's, so this is a faithful
single-GPU check of what each rank computes.  A world_size-1 NCCL run covers
the orchestrator's collective calls on the device.  Checked against the
oracle's single-process sub_r_hosvd (tucker.hpp:177-242)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    ((6, 5, 7), [3, 2, 3], 2, [9, 8, 10], 11, 2),
    ((8, 6, 5, 9), [2, 3, 2, 3], 3, [10, 12, 9, 14], 3, 3),
    ((40, 36, 64), [6, 5, 8], 5, [30, 28, 40], 5, 8),
    ((120, 100, 96), [10, 10, 10], 6, [44, 44, 44], 0, 4),
]


@pytest.mark.parametrize("case", CASES)
def test_sharded_phases_match_oracle(case, O):
    import torch

    from paper_2603_21379_b200 import sharded

    dims, ranks, p, samples, seed, W = case
    d = len(dims)
    x = np.random.default_rng(7).standard_normal(dims)
    ph = sharded.GpuShardPhases()
    bounds = [sharded.slab_bounds(dims[-1], W, w) for w in range(W)]
    locs = [torch.from_numpy(np.ravel(x[..., lo:hi], order="F").copy()).cuda() for lo, hi in bounds]
    parts = [ph.shard_sketches(xl, dims, lo, hi, ranks, p, samples, seed) for xl, (lo, hi) in zip(locs, bounds)]
    zs = [sum(pp[k] for pp in parts) for k in range(d - 1)]
    c = ranks[-1] + p
    zs.append(torch.cat([pp[d - 1].view(c, hi - lo) for pp, (lo, hi) in zip(parts, bounds)], dim=1).reshape(-1))

    ref = O.sub_r_hosvd(x, ranks, p, samples, seed)
    # partial sketches sum to the oracle's Z_k; the row blocks stack to Z_{d-1}
    for k in range(d):
        rng = O.RngStream(seed, k)
        cols = O.sample_indices(x.size // dims[k], samples[k], rng)
        zr = np.ravel(O.extract_fibers(x, k, cols) @ O.gaussian_matrix(samples[k], ranks[k] + p, rng), order="F")
        assert np.abs(zs[k].cpu().numpy() - zr).max() <= 1e-12 * max(1.0, np.abs(zr).max()) * samples[k]

    us, ach = ph.bases_from_sketches(dims, ranks, p, samples, seed, zs)
    assert ach == [int(a) for a in ref_ach(O, x, ranks, p, samples, seed)]
    for k in range(d):
        u = us[k].cpu().numpy().reshape((dims[k], ranks[k]), order="F")
        assert np.linalg.norm(u @ u.T - ref.factors[k] @ ref.factors[k].T) < 1e-9
    core = sum(ph.shard_core(xl, dims, lo, hi, ranks, us) for xl, (lo, hi) in zip(locs, bounds))
    # align to the oracle's factors (sign/rotation-free comparison)
    from parity import aligned_core_error

    g = core.cpu().numpy().reshape(tuple(ranks), order="F")
    fac = [u.cpu().numpy().reshape((dims[k], ranks[k]), order="F") for k, u in enumerate(us)]
    assert aligned_core_error(g, fac, ref.core, ref.factors) < 1e-10


def ref_ach(O, x, ranks, p, samples, seed):
    rep = O.SubsampleReport()
    O.sub_r_hosvd(x, ranks, p, samples, seed, report=rep)
    return rep.achieved_ranks


def test_sharded_equals_single_gpu():
    """Sharded result vs the single-GPU sub_r_hosvd on the same input."""
    import torch

    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import sharded

    dims, ranks, p, samples, seed, W = (64, 48, 80), [8, 6, 8], 4, [40, 36, 44], 9, 4
    x = np.random.default_rng(3).standard_normal(dims)
    single = P.sub_r_hosvd(x, ranks, p, samples, seed)
    ph = sharded.GpuShardPhases()
    bounds = [sharded.slab_bounds(dims[-1], W, w) for w in range(W)]
    locs = [torch.from_numpy(np.ravel(x[..., lo:hi], order="F").copy()).cuda() for lo, hi in bounds]
    parts = [ph.shard_sketches(xl, dims, lo, hi, ranks, p, samples, seed) for xl, (lo, hi) in zip(locs, bounds)]
    zs = [sum(pp[k] for pp in parts) for k in range(2)]
    zs.append(torch.cat([pp[2].view(ranks[2] + p, hi - lo) for pp, (lo, hi) in zip(parts, bounds)], 1).reshape(-1))
    us, _ = ph.bases_from_sketches(dims, ranks, p, samples, seed, zs)
    for k in range(3):
        u = us[k].cpu().numpy().reshape((dims[k], ranks[k]), order="F")
        assert np.abs(np.abs(u) - np.abs(single.factors[k])).max() < 1e-9
    core = sum(ph.shard_core(xl, dims, lo, hi, ranks, us) for xl, (lo, hi) in zip(locs, bounds))
    g = core.cpu().numpy().reshape(tuple(ranks), order="F")
    assert np.linalg.norm(np.abs(g) - np.abs(single.core)) <= 1e-10 * np.linalg.norm(single.core)


def test_shard_argument_errors():
    import torch

    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import sharded

    ph = sharded.GpuShardPhases()
    x = torch.zeros(6 * 5 * 3, dtype=torch.float64, device="cuda")
    with pytest.raises(P.InvalidArgument):
        ph.shard_sketches(x, [6, 5, 7], 5, 8, [2, 2, 2], 2, [8, 8, 8], 0)   # hi > n
    with pytest.raises(P.InvalidArgument):
        ph.shard_sketches(x, [6, 5, 7], 3, 3, [2, 2, 2], 2, [8, 8, 8], 0)   # empty slab


_NCCL_SCRIPT = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path[:0] = [os.environ["ROOT"], os.path.join(os.environ["ROOT"], "oracle"), os.path.join(os.environ["ROOT"], "tests")]
from paper_2603_21379_b200 import sharded
import srtt_oracle as O
from parity import aligned_core_error
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
dims, ranks, p, samples, seed = (30, 24, 20), [5, 4, 5], 4, [24, 22, 26], 13
x = np.random.default_rng(1).standard_normal(dims)
xl = torch.from_numpy(np.ravel(x, order="F").copy()).cuda()
t = sharded.sub_r_hosvd_sharded(xl, dims, ranks, p, samples, seed)
ref = O.sub_r_hosvd(x, ranks, p, samples, seed)
fac = [u.cpu().numpy().reshape((dims[k], ranks[k]), order="F") for k, u in enumerate(t.factors)]
err = aligned_core_error(t.core.cpu().numpy().reshape(tuple(ranks), order="F"), fac, ref.core, ref.factors)
assert err < 1e-10, err
dist.destroy_process_group()
print("OK")
"""


def test_orchestrator_nccl_world1():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    r = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


# ---------------------------------------------------------------------------
# H-Tucker column-range sharding: phases emulated rank by rank on one GPU
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dims,r,p,w,seed,W", [((6, 5, 7, 4), 3, 4, 24, 1, 3), ((5, 4, 6, 3, 4, 5), 3, 4, 30, 2, 4),
                                                ((12,) * 6, 4, 5, 40, 0, 5)])
def test_ht_sharded_phases_match_oracle(dims, r, p, w, seed, W, O):
    """Each rank's srtt_ht_shard_sketches / srtt_ht_shard_root on its column
    range of M, the exchanges (sums) done here: the reduced sketches equal the
    oracle's node sketches, and the bases / transfers / root give the
    oracle's decomposition (htucker.hpp:210-341)."""
    import torch

    from paper_2603_21379_b200 import sharded
    from parity import aligned_core_error

    import paper_2603_21379_b200 as P

    tree = O.DimensionTree.balanced(len(dims))
    ptree = P.DimensionTree.balanced(len(dims))
    ranks = O.uniform_node_ranks(tree, r)
    samples = [1] + [min(w, tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(dims)
    xf = torch.from_numpy(np.ravel(x, order="F").copy()).cuda()
    ph = sharded.GpuHtShardPhases()
    bounds = [sharded.column_bounds(ptree, dims, W, g) for g in range(W)]
    nl, nr = bounds[0][2], bounds[0][3]
    parts = [ph.shard_sketches(xf[lo * nl:hi * nl].contiguous(), dims, ptree, lo, hi, ranks, p, samples, seed)
             for lo, hi, _, _ in bounds]
    zs = {i: sum(pp[i] for pp in parts) for i in range(1, tree.num_nodes)}
    orep = O.HtSubsampleReport()
    ref = O.sub_r_rtl_ht(x, tree, ranks, samples, p, seed, report=orep)
    for i in range(1, tree.num_nodes):
        zr = orep.sketches[i]
        zg = zs[i].cpu().numpy().reshape(zr.shape, order="F")
        assert np.linalg.norm(zg - zr) <= 1e-13 * np.linalg.norm(zr), i
    us, bs, ach = ph.bases_from_sketches(dims, ptree, ranks, p, samples, seed, zs)
    assert ach == orep.achieved_ranks
    ub = {i: us[i].cpu().numpy().reshape(orep.bases[i].shape, order="F") for i in us}
    for i in ub:
        assert np.linalg.norm(ub[i] @ ub[i].T - orep.bases[i] @ orep.bases[i].T) <= 1e-10
    root = tree.node(0)
    b0 = sum(ph.shard_root(xf[lo * nl:hi * nl].contiguous(), nl, nr, lo, hi, us[root.left], r, us[root.right], r)
             for lo, hi, _, _ in bounds)
    b0 = b0.cpu().numpy().reshape((1, r, r), order="F")
    one = np.ones((1, 1))
    assert aligned_core_error(b0, [one, ub[root.left], ub[root.right]], ref.transfers[0],
                              [one, orep.bases[root.left], orep.bases[root.right]]) <= 1e-10
    for i, b in bs.items():
        n = tree.node(i)
        bt = b.cpu().numpy().reshape(ref.transfers[i].shape, order="F")
        assert aligned_core_error(bt, [ub[i], ub[n.left], ub[n.right]], ref.transfers[i],
                                  [orep.bases[i], orep.bases[n.left], orep.bases[n.right]]) <= 1e-10


# ---------------------------------------------------------------------------
# Fused NCCL entries (srtt_sub_r_hosvd_sharded / srtt_sub_r_rtl_ht_sharded)
# ---------------------------------------------------------------------------
def test_fused_nccl_world1_equals_single_gpu(O):
    """World 1: the slab is the whole tensor and the allreduces are copies,
    so the fused sharded decompositions (kernels + NCCL captured in one CUDA
    graph) return BITWISE the single-GPU results; replays too."""
    import torch

    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import sharded

    h = P.Handle(0, use_graphs=True)
    sharded.comm_init_local(h)
    assert sharded.comm_info(h) == (1, 0)
    h.set_stream(torch.cuda.current_stream().cuda_stream)
    dims, ranks, p, samples, seed = [40, 36, 30], [6, 5, 6], 5, [44, 40, 44], 3
    x = torch.from_numpy(np.ravel(np.random.default_rng(2).standard_normal(dims), order="F").copy()).cuda()
    single = P.sub_r_hosvd(x, ranks, p, samples, seed, dims=dims, device_out=True, handle=P.Handle(0))
    rep = P.SubsampleReport()
    t = sharded.sub_r_hosvd_nccl(x, dims, ranks, p, samples, seed, handle=h, report=rep)
    assert rep.achieved_ranks == ranks and rep.timings["gather"] > 0
    for _ in range(3):  # graph replays (stream-ordered)
        t = sharded.sub_r_hosvd_nccl(x, dims, ranks, p, samples, seed, handle=h)
    torch.cuda.synchronize()
    assert torch.equal(t.core, single.core)
    assert all(torch.equal(a, b) for a, b in zip(t.factors, single.factors))

    tree = P.DimensionTree.balanced(4)
    hd = [9, 8, 7, 6]
    hr = P.uniform_node_ranks(tree, 3)
    hs = [1] + [min(24, tree.node_cols(i, hd)) for i in range(1, tree.num_nodes)]
    y = torch.from_numpy(np.ravel(np.random.default_rng(4).standard_normal(hd), order="F").copy()).cuda()
    hs1 = P.sub_r_rtl_ht(y, tree, hr, hs, 4, 6, dims=hd, device_out=True, handle=P.Handle(0))
    rep = P.HtSubsampleReport()
    hs2 = sharded.sub_r_rtl_ht_nccl(y, hd, tree, hr, hs, 4, 6, handle=h, report=rep)
    hs2 = sharded.sub_r_rtl_ht_nccl(y, hd, tree, hr, hs, 4, 6, handle=h)
    torch.cuda.synchronize()
    assert rep.achieved_ranks == [1] + [3] * 6
    assert all(torch.equal(a, b) for a, b in zip(hs1.leaf_factors, hs2.leaf_factors))
    assert all(torch.equal(a.reshape(-1), b) for a, b in zip(hs1.transfers, hs2.transfers) if a is not None)


def test_replicated_world1_equals_single_gpu():
    """Replicated regime (all of X on every rank, modes / nodes assigned to
    ranks, factor pack allreduced): at world 1 every target is this rank's
    and the split full pass is the whole pass, so the outputs equal the
    single-GPU ones bitwise."""
    import torch

    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import sharded

    h = P.Handle(0, use_graphs=True)
    sharded.comm_init_local(h)
    h.set_stream(torch.cuda.current_stream().cuda_stream)
    dims, ranks, p, samples, seed = [40, 36, 30, 8], [6, 5, 6, 3], 5, [44, 40, 44, 30], 8
    x = torch.from_numpy(np.ravel(np.random.default_rng(5).standard_normal(dims), order="F").copy()).cuda()
    single = P.sub_r_hosvd(x, ranks, p, samples, seed, dims=dims, device_out=True, handle=P.Handle(0))
    rep = P.SubsampleReport()
    t = sharded.sub_r_hosvd_nccl(x, dims, ranks, p, samples, seed, handle=h, report=rep, replicated=True)
    t = sharded.sub_r_hosvd_nccl(x, dims, ranks, p, samples, seed, handle=h, replicated=True)
    torch.cuda.synchronize()
    assert rep.achieved_ranks == ranks
    assert torch.equal(t.core, single.core)
    assert all(torch.equal(a, b) for a, b in zip(t.factors, single.factors))
    tree = P.DimensionTree.balanced(4)
    hd = [9, 8, 7, 6]
    hr = P.uniform_node_ranks(tree, 3)
    hs = [1] + [min(24, tree.node_cols(i, hd)) for i in range(1, tree.num_nodes)]
    y = torch.from_numpy(np.ravel(np.random.default_rng(4).standard_normal(hd), order="F").copy()).cuda()
    h1 = P.sub_r_rtl_ht(y, tree, hr, hs, 4, 6, dims=hd, device_out=True, handle=P.Handle(0))
    rep = P.HtSubsampleReport()
    h2 = sharded.sub_r_rtl_ht_nccl(y, hd, tree, hr, hs, 4, 6, handle=h, report=rep, replicated=True)
    torch.cuda.synchronize()
    assert rep.achieved_ranks == [1] + [3] * 6
    assert all(torch.equal(a, b) for a, b in zip(h1.leaf_factors, h2.leaf_factors))
    assert all(torch.equal(a.reshape(-1), b) for a, b in zip(h1.transfers, h2.transfers) if a is not None)


def test_target_assignment_is_balanced_and_identical_on_every_rank(O):
    """The LPT assignment the replicated regime uses, restated: every target
    goes to exactly one rank and the heaviest rank carries at most the
    optimum plus the largest target (the greedy bound)."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        n, world = int(rng.integers(1, 15)), int(rng.integers(1, 9))
        cost = rng.integers(1, 100, size=n).astype(float)
        order = sorted(range(n), key=lambda t: -cost[t])
        load, owner = [0.0] * world, [0] * n
        for t in order:
            w = min(range(world), key=lambda r: (load[r], r))
            load[w] += cost[t]
            owner[t] = w
        assert max(load) <= cost.sum() / world + cost.max() + 1e-9


def test_fused_nccl_errors():
    import torch

    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import sharded

    h = P.Handle(0)
    x = torch.zeros(6 * 5 * 7, dtype=torch.float64, device="cuda")
    with pytest.raises(P.InvalidArgument, match="no communicator"):
        sharded.sub_r_hosvd_nccl(x, [6, 5, 7], [2, 2, 2], 2, [8, 8, 8], 0, handle=h)
    sharded.comm_init_local(h)
    with pytest.raises(P.InvalidArgument, match="more samples than fibers"):
        sharded.sub_r_hosvd_nccl(x, [6, 5, 7], [2, 2, 2], 2, [99, 8, 8], 0, handle=h)
