"""Device-side container IO: SRTT payload streamed through pinned staging
into HBM (whole tensor or a last-mode slab) and written back from HBM
(reference io.cpp:92-121)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_read_and_write_round_trip(tmp_path):
    import torch

    import paper_2603_21379_b200 as P

    x = np.random.default_rng(3).standard_normal((33, 17, 29))
    path = tmp_path / "x.srtt"
    P.write_tensor(path, x)
    d = P.read_tensor(path, device=True)
    assert d.is_cuda and np.array_equal(d.cpu().numpy(), np.ravel(x, order="F"))
    for lo, hi in [(0, 29), (5, 6), (10, 29)]:
        s = P.read_tensor(path, slab=(lo, hi), device=True)
        assert np.array_equal(s.cpu().numpy(), np.ravel(x[..., lo:hi], order="F"))
    back = tmp_path / "back.srtt"
    P.write_tensor(back, d, dims=[33, 17, 29])
    assert back.read_bytes() == path.read_bytes()


def test_large_read_crosses_staging_chunks(tmp_path):
    """> 64 MiB payload: several pinned chunks, both staging buffers reused."""
    import torch

    import paper_2603_21379_b200 as P

    dims = (256, 256, 160)   # 80 MiB
    x = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda")
    path = tmp_path / "big.srtt"
    P.write_tensor(path, x, dims=list(dims))
    y = P.read_tensor(path, device=True)
    assert torch.equal(x, y)
    s = P.read_tensor(path, slab=(37, 151), device=True)
    assert torch.equal(s, x.view(dims[2], -1)[37:151].reshape(-1))


def test_sharded_decomposition_from_file(tmp_path, O):
    """Each emulated rank reads only its slab from the file, then runs the
    shard phases; the result matches the oracle on the full tensor."""
    import torch

    from paper_2603_21379_b200 import sharded
    from parity import aligned_core_error

    import paper_2603_21379_b200 as P

    dims, ranks, p, samples, seed, W = (24, 20, 30), [4, 3, 5], 4, [20, 18, 24], 2, 3
    x = np.random.default_rng(5).standard_normal(dims)
    path = tmp_path / "x.srtt"
    P.write_tensor(path, x)
    ph = sharded.GpuShardPhases()
    bounds = [sharded.slab_bounds(dims[-1], W, w) for w in range(W)]
    locs = [P.read_tensor(path, slab=b, device=True) for b in bounds]
    parts = [ph.shard_sketches(xl, list(dims), lo, hi, ranks, p, samples, seed) for xl, (lo, hi) in zip(locs, bounds)]
    zs = [sum(pp[k] for pp in parts) for k in range(2)]
    zs.append(torch.cat([pp[2].view(ranks[2] + p, hi - lo) for pp, (lo, hi) in zip(parts, bounds)], 1).reshape(-1))
    us, _ = ph.bases_from_sketches(list(dims), ranks, p, samples, seed, zs)
    core = sum(ph.shard_core(xl, list(dims), lo, hi, ranks, us) for xl, (lo, hi) in zip(locs, bounds))
    ref = O.sub_r_hosvd(x, ranks, p, samples, seed)
    fac = [u.cpu().numpy().reshape((dims[k], ranks[k]), order="F") for k, u in enumerate(us)]
    g = core.cpu().numpy().reshape(tuple(ranks), order="F")
    assert aligned_core_error(g, fac, ref.core, ref.factors) < 1e-10
