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
