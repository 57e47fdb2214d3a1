"""Seeded synthetic stand-ins for the BASELINE.json configs (C1-C5).

The reference ships no fixtures for these configs (its generators.hpp makes
different tensors), so these generators define them, following SURVEY.md
§8(d) and BASELINE.json `configs`.  Every tensor is returned FLAT with the
first index fastest (reference tensor.hpp:17-20).  Two backends:
``backend="torch"`` generates on a CUDA device (bench), ``"numpy"`` on the
host (CPU tests / the reference arm).  Bits differ between backends (libm,
RNG); parity tests always hand the same bits to both sides by copying.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    kind: str            # "tucker" | "htucker"
    dims: tuple
    rank: int
    p: int
    description: str
    base: str = ""       # tensor family (added variants reuse a BASELINE config's generator)
    fibres: int = 0      # Tucker: fibres per mode (0: the 4 (r + p) rule)
    alpha: float = 0.0   # H-Tucker: node budgets w_S = min(ceil(alpha n_S), n_notS) (0: 4 (r + p))

    @property
    def order(self):
        return len(self.dims)

    @property
    def entries(self):
        return int(np.prod(self.dims))

    @property
    def family(self):
        return self.base or self.name

    def samples(self):
        """s = 4 (r + p) per mode (explicit for C1, assumed for the rest)."""
        return [self.fibres or 4 * (self.rank + self.p)] * self.order

    def node_samples(self, tree, dims=None):
        """H-Tucker node budgets: min(4 (r + p), n_notS), or the alpha rule
        of node_sample_counts (dimension_tree.hpp:174-183); root entry 1."""
        import math

        dims = list(dims or self.dims)
        out = [1]
        for i in range(1, tree.num_nodes):
            cols = tree.node_cols(i, dims)
            want = math.ceil(self.alpha * tree.node_rows(i, dims)) if self.alpha else 4 * (self.rank + self.p)
            out.append(min(want, cols))
        return out


CONFIGS = {
    "c1": Config("c1", "tucker", (128, 128, 128), 8, 5,
                 "order-3 Tucker 128^3, planted rank 8 + 1e-8 relative noise, r=8 p=5 s=52"),
    "c2": Config("c2", "tucker", (40, 40, 40, 40, 40), 6, 5,
                 "order-5 Tucker 40^5, decaying 6^5 core, Gaussian-QR factors, N(0,1e-20) noise, r=6 p=5 s=44"),
    "c3": Config("c3", "tucker", (200, 200, 200, 200), 12, 8,
                 "order-4 function tensor 1/(x1+x2+x3+x4) on [0.1,1]^4 grid, r=12 p=8 s=80"),
    "c4": Config("c4", "htucker", (12,) * 8, 10, 5,
                 "order-8 H-Tucker 12^8, sum of 10 rank-1 Gaussian terms + 1e-8 relative noise, r=10 p=5 w=60"),
    "c5": Config("c5", "tucker", (2048, 2048, 2048), 32, 10,
                 "order-3 Tucker 2048^3, rank-32 N(0,1) core + Gaussian-QR factors + 1e-6 relative noise, r=32 p=10 s=168"),
    # ---- sketch-heavy variants ADDED for the K1 bandwidth measurement
    # (SURVEY §8d); NOT BASELINE configs
    "c4a20": Config("c4a20", "htucker", (12,) * 8, 10, 5,
                    "ADDED variant of c4: node budgets by alpha = 20 (dimension_tree.hpp:174-183), so both "
                    "level-1 nodes sample all 20736 columns", base="c4", alpha=20.0),
    "c5s64k": Config("c5s64k", "tucker", (2048, 2048, 2048), 32, 10,
                     "ADDED variant of c5: s = 65536 fibres per mode (1.07 GB gathered per mode)", base="c5",
                     fibres=65536),
}


# ---------------------------------------------------------------------------
# backend helpers
# ---------------------------------------------------------------------------
class _NP:
    def __init__(self, seed):
        self.rng = np.random.default_rng(seed)

    def randn(self, *shape):
        return self.rng.standard_normal(shape)

    def qr_q(self, a):
        return np.linalg.qr(a)[0]

    def expand(self, core, factors):
        """first-index-fastest flat X = core x_1 U_1 ... x_d U_d."""
        x = core
        for k, u in enumerate(factors):
            x = np.moveaxis(np.tensordot(u, x, axes=([1], [k])), 0, k)
        return np.ravel(x, order="F")

    def norm(self, v):
        return float(np.linalg.norm(v))


class _Torch:
    def __init__(self, seed, device):
        import torch

        self.t = torch
        self.dev = torch.device(device)
        self.g = torch.Generator(device=self.dev)
        self.g.manual_seed(int(seed))

    def randn(self, *shape):
        return self.t.randn(*shape, dtype=self.t.float64, device=self.dev, generator=self.g)

    def qr_q(self, a):
        return self.t.linalg.qr(a)[0]

    def expand(self, core, factors):
        # build the reversed-axes row-major tensor == first-index-fastest X
        t = self.t
        x = core.permute(*reversed(range(core.dim()))).contiguous()  # axes (d-1 .. 0)
        d = core.dim()
        for k, u in enumerate(factors):
            ax = d - 1 - k
            x = t.tensordot(x, u, dims=([ax], [1]))          # new axis appended last
            x = x.movedim(-1, ax).contiguous()
        return x.reshape(-1)

    def norm(self, v):
        return float(self.t.linalg.vector_norm(v))


def _backend(backend, seed, device):
    return _NP(seed) if backend == "numpy" else _Torch(seed, device)


def _add_relative_noise(B, x, rel, chunk=1 << 26):
    """x += rel * ||x|| * E / ||E|| with E iid N(0,1), chunked so the noise
    never needs a second full-size buffer (SURVEY §8d noise rule)."""
    n = x.shape[0]
    nx = B.norm(x)
    if isinstance(B, _NP):
        state = B.rng.bit_generator.state
        e2 = 0.0
        for lo in range(0, n, chunk):
            e = B.rng.standard_normal(min(chunk, n - lo))
            e2 += float(e @ e)
        B.rng.bit_generator.state = state
        scale = rel * nx / np.sqrt(e2)
        for lo in range(0, n, chunk):
            x[lo:lo + chunk] += scale * B.rng.standard_normal(min(chunk, n - lo))
    else:
        st = B.g.get_state()
        e2 = 0.0
        for lo in range(0, n, chunk):
            e = B.randn(min(chunk, n - lo))
            e2 += float((e * e).sum())
        B.g.set_state(st)
        scale = rel * nx / np.sqrt(e2)
        for lo in range(0, n, chunk):
            x[lo:lo + chunk].add_(B.randn(min(chunk, n - lo)), alpha=scale)
    return x


def _function_tensor(dims, backend, device):
    """C3: X(i) = 1/(x_i1 + x_i2 + x_i3 + x_i4), x = 0.1 + i*0.9/(n-1),
    evaluated as (((a+b)+c)+d) then one division (no FMA) -> identical bits
    on every backend."""
    n = dims[0]
    if backend == "numpy":
        g = 0.1 + np.arange(n) * (0.9 / (n - 1))
        a = g[:, None, None, None]
        b = g[None, :, None, None]
        c = g[None, None, :, None]
        dd = g[None, None, None, :]
        x = 1.0 / (((a + b) + c) + dd)
        return np.ravel(x, order="F")
    import torch

    g = 0.1 + torch.arange(n, dtype=torch.float64, device=device) * (0.9 / (n - 1))
    # reversed-axes row-major (i4, i3, i2, i1)
    s = ((g.view(1, 1, 1, n) + g.view(1, 1, n, 1)) + g.view(1, n, 1, 1)) + g.view(n, 1, 1, 1)
    return (1.0 / s).reshape(-1)


def make_tensor(cfg: Config, seed: int = 0, backend: str = "torch", device: str = "cuda", dims=None):
    """Flat, first-index-fastest float64 tensor for config `cfg` (optionally
    with smaller `dims` of the same family for tests)."""
    dims = tuple(dims or cfg.dims)
    d = len(dims)
    fam = cfg.family
    if fam == "c3":
        return _function_tensor(dims, backend, device)
    B = _backend(backend, seed, device)
    r = cfg.rank
    if fam in ("c1", "c5"):
        core = B.randn(*([r] * d))
        factors = [B.qr_q(B.randn(n, r)) for n in dims]
        x = B.expand(core, factors)
        return _add_relative_noise(B, x, 1e-8 if fam == "c1" else 1e-6)
    if fam == "c2":
        core = B.randn(*([r] * d))
        idx = np.indices([r] * d).sum(axis=0)
        scale = 10.0 ** (-idx / d)
        if backend == "numpy":
            core = core * scale
        else:
            core = core * B.t.from_numpy(scale).to(B.dev)
        factors = [B.qr_q(B.randn(n, r)) for n in dims]
        x = B.expand(core, factors)
        if backend == "numpy":
            x += 1e-10 * B.rng.standard_normal(x.shape[0])
        else:
            x.add_(B.randn(x.shape[0]), alpha=1e-10)
        return x
    if fam == "c4":
        # sum of 10 rank-1 terms: core = superdiagonal of ones (10^d), factors a_t^(k)
        terms = 10
        vecs = [B.randn(n, terms) for n in dims]
        if backend == "numpy":
            x = np.zeros(int(np.prod(dims)))
            for t in range(terms):
                v = vecs[0][:, t]
                for k in range(1, d):
                    v = np.multiply.outer(vecs[k][:, t], v).reshape(-1)  # first index fastest
                x += v
        else:
            t_ = B.t
            x = t_.zeros(int(np.prod(dims)), dtype=t_.float64, device=B.dev)
            for t in range(terms):
                v = vecs[0][:, t]
                for k in range(1, d):
                    v = t_.outer(vecs[k][:, t], v).reshape(-1)
                x += v
        return _add_relative_noise(B, x, 1e-8)
    raise ValueError(cfg.name)
