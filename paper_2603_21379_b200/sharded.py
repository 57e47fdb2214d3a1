"""Slab-sharded Sub-R-HOSVD: one process per GPU, X split along its last mode.

The reference parallelises one Tucker job inside a process: mode jobs run
concurrently (tucker.hpp:196-214) and the core is reduced slab by slab along
a slice mode (``sliced_core``, parallel.hpp:355-445).  Across GPUs the same
slab algebra holds with the slabs living on different devices:

  rank w owns X[..., lo_w:hi_w)  (slab bounds of parallel.hpp:400-404)

  1. sketches   Z_k = Y_k Omega_k.  Every rank samples the same fibres and
                generates the same Omega (same seed, counter-based stream).
                For k < d-1 a sampled fibre lies in exactly one slab, so the
                per-rank partial sketches SUM to Z_k           -> all_reduce
                For k = d-1 the fibres run along the sliced mode, so each
                rank owns rows [lo_w, hi_w) of Z_{d-1}         -> all_gather
  2. bases      U_k = range_basis_of_sketch(Z_k): identical on every rank
                (same Z, same deterministic kernel, same padding stream).
  3. core       G = sum_w X_w x_{k<d-1} U_k^T x_{d-1} U_{d-1}[lo_w:hi_w]^T
                                                               -> all_reduce

Only the sketches (sum n_k (r_k+p) doubles) and the core (prod r_k doubles)
cross the interconnect; X never moves.  Work per rank is the slab, so the
scaling is weak in the slab size.  The phase calls go through the C-ABI
(``srtt_shard_sketches`` / ``srtt_bases_from_sketches`` / ``srtt_shard_core``)
and the collectives through ``torch.distributed`` (NCCL on GPUs; any backend
works because the phases are pluggable -- the CPU tests drive the same
orchestration with gloo and a checker backend).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import srtt as _s


def slab_bounds(n: int, world: int, rank: int):
    """[lo, hi) of slab ``rank`` -- the split of parallel.hpp:400-404."""
    if world > n:
        raise _s.InvalidArgument("sharded sub_r_hosvd: more ranks than slices along the last mode")
    lo = rank * (n // world) + min(rank, n % world)
    hi = lo + n // world + (1 if rank < n % world else 0)
    return lo, hi


class GpuShardPhases:
    """The three phases on this process's GPU through the C-ABI.  Inputs and
    outputs are flat CUDA float64 torch tensors (first index fastest,
    matrices column-major)."""

    def __init__(self, handle: _s.Handle | None = None):
        self.h = handle or _s.default_handle()
        lib = _s._L()
        vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        lib.srtt_shard_sketches.argtypes = [vp, vp, i32, i32, vp, i64, i64, vp, i64, vp, u64, vp, vp, i32]
        lib.srtt_bases_from_sketches.argtypes = [vp, i32, vp, vp, i64, vp, u64, vp, vp, i32, vp, i32, vp]
        lib.srtt_shard_core.argtypes = [vp, vp, i32, i32, vp, i64, i64, vp, vp, i32, vp, i32]
        self.lib = lib

    def _bind(self):
        """Run every phase on torch's CURRENT stream: the collectives between
        the phases (torch.distributed / NCCL) and the torch ops that produce
        x_local are ordered on that stream, so a phase bound to the handle's
        own non-blocking stream could read sketches that are not reduced yet."""
        import torch

        self.h.set_stream(torch.cuda.current_stream().cuda_stream)

    def shard_sketches(self, x_local, dims, lo, hi, ranks, p, samples, seed):
        import torch

        self._bind()

        d = len(dims)
        rows = [dims[k] if k < d - 1 else hi - lo for k in range(d)]
        sizes = [rows[k] * (ranks[k] + p) for k in range(d)]
        # the summed sketches (k < d-1) are views of ONE buffer, so a single
        # all_reduce exchanges them (self.partial_sums)
        flat = torch.empty(sum(sizes[:-1]), dtype=torch.float64, device=x_local.device)
        offs = np.cumsum([0] + sizes[:-1])
        zs = [flat[offs[k]:offs[k + 1]] for k in range(d - 1)]
        zs.append(torch.empty(sizes[-1], dtype=torch.float64, device=x_local.device))
        self.partial_sums = flat
        zp = (C.c_void_p * d)(*[z.data_ptr() for z in zs])
        dims_a, ranks_a, samp_a = _s._i64(dims), _s._i64(ranks), _s._i64(samples)
        _s._check(self.lib.srtt_shard_sketches(self.h._h, x_local.data_ptr(), 1, d, dims_a.ctypes.data, lo, hi,
                                               ranks_a.ctypes.data, p, samp_a.ctypes.data, seed, None, zp, 1))
        return zs

    def bases_from_sketches(self, dims, ranks, p, samples, seed, zs):
        import torch

        self._bind()
        d = len(dims)
        us = [torch.empty(dims[k] * ranks[k], dtype=torch.float64, device=zs[0].device) for k in range(d)]
        zp = (C.c_void_p * d)(*[z.data_ptr() for z in zs])
        up = (C.c_void_p * d)(*[u.data_ptr() for u in us])
        ach = np.zeros(d, dtype=np.int64)
        dims_a, ranks_a, samp_a = _s._i64(dims), _s._i64(ranks), _s._i64(samples)
        _s._check(self.lib.srtt_bases_from_sketches(self.h._h, d, dims_a.ctypes.data, ranks_a.ctypes.data, p,
                                                    samp_a.ctypes.data, seed, None, zp, 1, up, 1, ach.ctypes.data))
        return us, [int(a) for a in ach]

    def shard_core(self, x_local, dims, lo, hi, ranks, factors):
        import torch

        self._bind()
        d = len(dims)
        g = torch.empty(int(np.prod(ranks)), dtype=torch.float64, device=x_local.device)
        fp = (C.c_void_p * d)(*[u.data_ptr() for u in factors])
        dims_a, ranks_a = _s._i64(dims), _s._i64(ranks)
        _s._check(self.lib.srtt_shard_core(self.h._h, x_local.data_ptr(), 1, d, dims_a.ctypes.data, lo, hi,
                                           ranks_a.ctypes.data, fp, 1, g.data_ptr(), 1))
        return g


def load_slab(path, *, group=None, handle=None):
    """This rank's slab of an SRTT file, read straight into its GPU: the
    last-mode slab is one contiguous byte range of the file (io.cpp:106-117),
    so no rank touches another's bytes. Returns (x_local, dims, (lo, hi))."""
    import torch.distributed as dist

    dims, _ = _s.tensor_file_info(path)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    me = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = slab_bounds(dims[-1], world, me)
    return _s.read_tensor(path, slab=(lo, hi), device=True, handle=handle), dims, (lo, hi)


@dataclass
class ShardedTucker:
    core: object          # flat tensor, prod(ranks), first index fastest (identical on every rank)
    factors: list         # flat tensors, n_k * r_k column-major (identical on every rank)
    achieved_ranks: list
    slab: tuple           # this rank's [lo, hi) along the last mode


def _gather_rows(z_local, n_local, c, counts, group):
    """All-gather row blocks of a column-major matrix with ragged row counts."""
    import torch
    import torch.distributed as dist

    mx = max(counts)
    padded = torch.zeros((c, mx), dtype=z_local.dtype, device=z_local.device)
    padded[:, :n_local] = z_local.view(c, n_local)      # column-major n_local x c == row-major c x n_local
    parts = [torch.empty_like(padded) for _ in counts]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:, :cnt] for p, cnt in zip(parts, counts)], dim=1).reshape(-1)


def sub_r_hosvd_sharded(x_local, dims, target, oversampling, samples, seed, *, group=None, phases=None):
    """Sub-R-HOSVD of a tensor whose last mode is sharded over the process
    group (tucker.hpp:177-242 with parallel.hpp:355-445's slab reduction
    across ranks).  ``x_local`` is this rank's slab ``X[..., lo:hi)`` as a
    flat float64 tensor (first index fastest) on this rank's device;
    ``dims`` are the global extents.  Returns identical factors and core on
    every rank."""
    import torch.distributed as dist

    d = len(dims)
    if len(target) != d or len(samples) != d:
        raise _s.InvalidArgument("sub_r_hosvd: rank/sample vector order mismatch")
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    L = d - 1
    bounds = [slab_bounds(dims[L], world, w) for w in range(world)]
    lo, hi = bounds[me]
    counts = [b - a for a, b in bounds]
    if min(counts) < target[L]:
        raise _s.InvalidArgument("sharded sub_r_hosvd: every slab must hold at least r_{d-1} slices")
    if x_local.numel() != int(np.prod(dims[:L])) * (hi - lo):
        raise _s.InvalidArgument("sharded sub_r_hosvd: local slab size mismatch")
    ph = phases or GpuShardPhases()
    zs = ph.shard_sketches(x_local, dims, lo, hi, target, oversampling, samples, seed)
    partial = getattr(ph, "partial_sums", None)
    if partial is not None:  # one collective for all summed sketches
        dist.all_reduce(partial, group=group)
    else:
        for k in range(L):
            dist.all_reduce(zs[k], group=group)
    zs[L] = _gather_rows(zs[L], hi - lo, target[L] + oversampling, counts, group)
    factors, achieved = ph.bases_from_sketches(dims, target, oversampling, samples, seed, zs)
    core = ph.shard_core(x_local, dims, lo, hi, target, factors)
    dist.all_reduce(core, group=group)
    return ShardedTucker(core=core, factors=factors, achieved_ranks=achieved, slab=(lo, hi))
