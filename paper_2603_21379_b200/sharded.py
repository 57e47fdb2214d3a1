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
cross the interconnect; X never moves.

Two ways to run it:

* ``sub_r_hosvd_nccl`` / ``sub_r_rtl_ht_nccl`` (the product path): ONE C-ABI
  call per rank (``srtt_sub_r_hosvd_sharded`` / ``srtt_sub_r_rtl_ht_sharded``)
  whose handle owns an NCCL communicator (``comm_init``); kernels and
  collectives are captured in one CUDA graph per call signature.
* ``sub_r_hosvd_sharded`` / ``sub_r_rtl_ht_sharded``: the same algebra as
  separate synchronous phases (``srtt_shard_*`` / ``srtt_ht_shard_*``) with
  the exchanges issued here through ``torch.distributed`` (any backend: the
  CPU tests drive this orchestration with gloo and a checker backend).

H-Tucker (htucker.hpp:210-341) splits X into column ranges of the root
matricization M = n_left x n_right (a contiguous byte range of X): every
node's sketch is a sum over its sampled fibre entries, so each rank forms
PARTIAL sketches of every node from its range (allreduce), the bases and
transfers follow identically on every rank, and the root transfer
B_0 = sum_w U_l^T M_w U_r[c_lo:c_hi] is one more allreduce (htucker.hpp:67-85).
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


def _dist():
    import torch.distributed as dist

    return dist


def comm_init(handle: _s.Handle, group=None):
    """Give ``handle`` an NCCL communicator spanning the torch.distributed
    group: rank 0 creates the NCCL unique id, the group broadcasts it, every
    rank calls ``srtt_comm_init`` (the handle owns the communicator)."""
    dist = _dist()
    lib = _s._L()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    uid = C.create_string_buffer(128)
    if me == 0:
        _s._check(lib.srtt_comm_unique_id(uid))
    obj = [bytes(uid.raw) if me == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    uid = C.create_string_buffer(obj[0], 128)
    _s._check(lib.srtt_comm_init(handle._h, world, me, uid))
    return world, me


def comm_init_local(handle: _s.Handle, world: int = 1, rank: int = 0, unique_id: bytes | None = None):
    """``srtt_comm_init`` without torch.distributed: ``unique_id`` from
    ``new_unique_id()`` distributed by any means (world 1 needs none)."""
    lib = _s._L()
    if unique_id is None:
        unique_id = new_unique_id()
    uid = C.create_string_buffer(bytes(unique_id), 128)
    _s._check(lib.srtt_comm_init(handle._h, int(world), int(rank), uid))


def new_unique_id() -> bytes:
    uid = C.create_string_buffer(128)
    _s._check(_s._L().srtt_comm_unique_id(uid))
    return bytes(uid.raw)


def comm_destroy(handle: _s.Handle):
    _s._check(_s._L().srtt_comm_destroy(handle._h))


def comm_info(handle: _s.Handle):
    w, r = C.c_int32(), C.c_int32()
    _s._check(_s._L().srtt_comm_info(handle._h, C.byref(w), C.byref(r)))
    return int(w.value), int(r.value)


def column_bounds(tree, dims, world: int, rank: int):
    """[c_lo, c_hi) of rank's columns of the root matricization
    M = n_left x n_right, and (n_left, n_right)."""
    nl = tree.node_rows(tree.node(0).left, dims)
    nr = tree.node_rows(tree.node(0).right, dims)
    lo, hi = slab_bounds(nr, world, rank)
    return lo, hi, nl, nr


def sub_r_hosvd_nccl(x_slab, dims, target, oversampling, samples, seed, *, handle, exec_policy=None,
                     report=None, out=None, device_out=True, replicated=False):
    """Fused slab-sharded sub_r_hosvd through ``srtt_sub_r_hosvd_sharded``
    (the handle must own a communicator, see ``comm_init``). ``x_slab`` is
    this rank's X[..., lo:hi) (flat, first index fastest: a CUDA float64
    tensor, or a host numpy array staged by the library) with the bounds of
    ``slab_bounds``; returns identical outputs on every rank (device tensors,
    or numpy arrays with ``device_out=False``). Stream-ordered when the
    outputs stay on the device and no report is requested."""
    import torch

    world, me = comm_info(handle)
    if world < 1:
        raise _s.InvalidArgument("sharded: the handle has no communicator (comm_init)")
    d = len(dims)
    lo, hi = slab_bounds(dims[-1], world, me)
    call = _s._CALLS.get(("sh",) + (tuple(dims), tuple(target), tuple(samples)))
    if call is None:
        call = _s._CALLS.setdefault(("sh",) + (tuple(dims), tuple(target), tuple(samples)),
                                    _s._TuckerCall(dims, target, samples))
    xf = _s._flat_f64(x_slab)
    xp, xdev = _s._ptr(xf)
    if out is None:
        if device_out:
            dev = torch.device("cuda", handle.device)
            out = (torch.empty(int(np.prod(target)), dtype=torch.float64, device=dev),
                   [torch.empty(dims[k] * target[k], dtype=torch.float64, device=dev) for k in range(d)])
        else:
            out = (np.zeros(int(np.prod(target))), [np.zeros(dims[k] * target[k]) for k in range(d)])
    for k in range(d):
        call.fptrs[k] = _s._ptr(out[1][k])[0]
    ex = exec_policy._c() if exec_policy is not None else None
    rep_arg = C.byref(call.rep) if (report is not None or not device_out) else None
    if replicated:  # x_slab is ALL of X; modes assigned to ranks, core split by slabs of the replica
        _s._check(_s._L().srtt_sub_r_hosvd_replicated(
            handle._h, xp, xdev, d, call.dims_a.ctypes.data, call.ranks_a.ctypes.data, int(oversampling),
            call.samp_a.ctypes.data, int(seed) & (2**64 - 1), C.byref(ex) if ex is not None else None,
            _s._ptr(out[0])[0], call.fptrs, int(device_out), rep_arg))
    else:
        _s._check(_s._L().srtt_sub_r_hosvd_sharded(
            handle._h, xp, xdev, d, call.dims_a.ctypes.data, lo, hi, call.ranks_a.ctypes.data,
            int(oversampling), call.samp_a.ctypes.data, int(seed) & (2**64 - 1),
            C.byref(ex) if ex is not None else None, _s._ptr(out[0])[0], call.fptrs, int(device_out), rep_arg))
    if report is not None:
        _s._report_from(call.rep, d, call.ach, call.sc, report, handle)
    return ShardedTucker(core=out[0], factors=list(out[1]), achieved_ranks=list(getattr(report, "achieved_ranks", [])),
                         slab=(lo, hi))


def sub_r_rtl_ht_nccl(x_cols, dims, tree, ranks, samples, oversampling, seed, *, handle, exec_policy=None,
                      report=None, device_out=True, replicated=False):
    """Fused column-range-sharded sub_r_rtl_ht through
    ``srtt_sub_r_rtl_ht_sharded``; ``x_cols`` holds this rank's columns
    [c_lo, c_hi) of M = n_left x n_right (``column_bounds``). Returns device
    leaf factors (by mode) and transfers (by node id), identical on every
    rank."""
    import torch

    world, me = comm_info(handle)
    if world < 1:
        raise _s.InvalidArgument("sharded: the handle has no communicator (comm_init)")
    d = len(dims)
    lo, hi, nl, nr = column_bounds(tree, dims, world, me)
    nn = tree.num_nodes
    dev = torch.device("cuda", handle.device)

    def alloc(n):
        return torch.empty(n, dtype=torch.float64, device=dev) if device_out else np.zeros(n)

    leaf = [None] * d
    for i in tree.leaves():
        m = tree.node(i).modes[0]
        leaf[m] = alloc(dims[m] * ranks[i])
    trs = [None] * nn
    for i in range(nn):
        n = tree.node(i)
        if not n.is_leaf():
            trs[i] = alloc((1 if i == 0 else ranks[i]) * ranks[n.left] * ranks[n.right])
    lp = (C.c_void_p * d)(*[_s._ptr(u)[0] for u in leaf])
    tp = (C.c_void_p * nn)(*[None if t is None else _s._ptr(t)[0] for t in trs])
    xf = _s._flat_f64(x_cols)
    xp, xdev = _s._ptr(xf)
    ranks_a, samp_a, dims_a = _s._i64(ranks), _s._i64(samples), _s._i64(dims)
    ach, sc = np.zeros(nn, np.int64), np.zeros(nn, np.int64)
    wbuf = C.create_string_buffer(8192)
    crep = _s._Report(sc.ctypes.data_as(C.POINTER(C.c_int64)), ach.ctypes.data_as(C.POINTER(C.c_int64)),
                      C.cast(wbuf, C.c_char_p), 8192, 0)
    ct = tree._c()
    ex = exec_policy._c() if exec_policy is not None else None
    rarg = C.byref(crep) if (report is not None or not device_out) else None
    if replicated:  # x_cols is ALL of X; nodes assigned to ranks, root split by column ranges
        _s._check(_s._L().srtt_sub_r_rtl_ht_replicated(
            handle._h, xp, xdev, d, dims_a.ctypes.data, C.byref(ct), ranks_a.ctypes.data, samp_a.ctypes.data,
            int(oversampling), int(seed) & (2**64 - 1), C.byref(ex) if ex is not None else None, lp, tp,
            int(device_out), rarg))
    else:
        _s._check(_s._L().srtt_sub_r_rtl_ht_sharded(
            handle._h, xp, xdev, d, dims_a.ctypes.data, lo, hi, C.byref(ct), ranks_a.ctypes.data,
            samp_a.ctypes.data, int(oversampling), int(seed) & (2**64 - 1), C.byref(ex) if ex is not None else None,
            lp, tp, int(device_out), rarg))
    if report is not None:
        _s._report_from(crep, nn, ach, sc, report, handle)
    return _s.HTuckerDecomposition(tree, leaf, trs)


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


# ---------------------------------------------------------------------------
# H-Tucker: column-range sharding, phases + torch.distributed orchestration
# ---------------------------------------------------------------------------
class GpuHtShardPhases:
    """srtt_ht_shard_sketches / srtt_ht_bases_from_sketches / srtt_ht_shard_root
    on this process's GPU (run on torch's current stream)."""

    def __init__(self, handle: _s.Handle | None = None):
        self.h = handle or _s.default_handle()
        lib = _s._L()
        vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        lib.srtt_ht_shard_sketches.argtypes = [vp, vp, i32, i32, vp, i64, i64, vp, vp, vp, i64, u64, vp, vp, i32]
        lib.srtt_ht_bases_from_sketches.argtypes = [vp, i32, vp, vp, vp, vp, i64, u64, vp, vp, i32, vp, vp, i32, vp]
        lib.srtt_ht_shard_root.argtypes = [vp, vp, i32, i64, i64, i64, i64, vp, i32, vp, i32, i32, vp, i32]
        self.lib = lib

    def _bind(self):
        import torch

        self.h.set_stream(torch.cuda.current_stream().cuda_stream)

    def shard_sketches(self, x_cols, dims, tree, lo, hi, ranks, p, samples, seed):
        """Partial sketch of every node (id -> flat n_S x (r_S+p) tensor)."""
        import torch

        self._bind()
        nn = tree.num_nodes
        zs = {i: torch.empty(tree.node_rows(i, dims) * (ranks[i] + p), dtype=torch.float64, device=x_cols.device)
              for i in range(1, nn)}
        zp = (C.c_void_p * nn)(*([None] + [zs[i].data_ptr() for i in range(1, nn)]))
        ct = tree._c()
        dims_a, ranks_a, samp_a = _s._i64(dims), _s._i64(ranks), _s._i64(samples)  # alive across the call
        _s._check(self.lib.srtt_ht_shard_sketches(self.h._h, x_cols.data_ptr(), 1, len(dims), dims_a.ctypes.data,
                                                  lo, hi, C.byref(ct), ranks_a.ctypes.data, samp_a.ctypes.data, p,
                                                  seed, None, zp, 1))
        return zs

    def bases_from_sketches(self, dims, tree, ranks, p, samples, seed, zs):
        """(node bases by id, transfers by id, achieved ranks)."""
        import torch

        self._bind()
        nn = tree.num_nodes
        dev = zs[1].device
        us = {i: torch.empty(tree.node_rows(i, dims) * ranks[i], dtype=torch.float64, device=dev)
              for i in range(1, nn)}
        bs = {}
        for i in range(1, nn):
            n = tree.node(i)
            if not n.is_leaf():
                bs[i] = torch.empty(ranks[i] * ranks[n.left] * ranks[n.right], dtype=torch.float64, device=dev)
        zp = (C.c_void_p * nn)(*([None] + [zs[i].data_ptr() for i in range(1, nn)]))
        up = (C.c_void_p * nn)(*([None] + [us[i].data_ptr() for i in range(1, nn)]))
        bp = (C.c_void_p * nn)(*[bs[i].data_ptr() if i in bs else None for i in range(nn)])
        ach = np.zeros(nn, np.int64)
        ct = tree._c()
        dims_a, ranks_a, samp_a = _s._i64(dims), _s._i64(ranks), _s._i64(samples)  # alive across the call
        _s._check(self.lib.srtt_ht_bases_from_sketches(self.h._h, len(dims), dims_a.ctypes.data, C.byref(ct),
                                                       ranks_a.ctypes.data, samp_a.ctypes.data, p, seed, None, zp, 1,
                                                       up, bp, 1, ach.ctypes.data))
        return us, bs, [int(a) for a in ach]

    def shard_root(self, x_cols, nl, nr, lo, hi, u_left, rl, u_right, rr):
        import torch

        self._bind()
        b = torch.empty(rl * rr, dtype=torch.float64, device=x_cols.device)
        _s._check(self.lib.srtt_ht_shard_root(self.h._h, x_cols.data_ptr(), 1, nl, nr, lo, hi, u_left.data_ptr(), rl,
                                              u_right.data_ptr(), rr, 1, b.data_ptr(), 1))
        return b


@dataclass
class ShardedHTucker:
    leaf_factors: list    # by mode, flat n_m x r (identical on every rank)
    transfers: list       # by node id (root: 1 x r_l x r_r), None for leaves
    node_bases: dict      # id -> flat basis (identical on every rank)
    achieved_ranks: list
    columns: tuple        # this rank's [c_lo, c_hi) of the root matricization


def sub_r_rtl_ht_sharded(x_cols, dims, tree, ranks, samples, oversampling, seed, *, group=None, phases=None):
    """Sub-R-RtL-HT (htucker.hpp:210-341) of a tensor split into column
    ranges of the root matricization over the process group, as three phases
    with the exchanges issued here: allreduce of every node's partial sketch,
    identical bases / transfers on every rank, allreduce of the partial root
    transfer."""
    dist = _dist()
    nn = tree.num_nodes
    d = len(dims)
    if tree.order != d:
        raise _s.InvalidArgument("sub_r_rtl_ht: tree and tensor order mismatch")
    if len(ranks) != nn or len(samples) != nn:
        raise _s.InvalidArgument("sub_r_rtl_ht: rank/sample vector must have one entry per node")
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    lo, hi, nl, nr = column_bounds(tree, dims, world, me)
    if x_cols.numel() != (hi - lo) * nl:
        raise _s.InvalidArgument("sharded sub_r_rtl_ht: local column range size mismatch")
    ph = phases or GpuHtShardPhases()
    zs = ph.shard_sketches(x_cols, dims, tree, lo, hi, ranks, oversampling, samples, seed)
    import torch

    flat = torch.cat([zs[i].reshape(-1) for i in range(1, nn)])   # ONE collective for all nodes
    dist.all_reduce(flat, group=group)
    off = 0
    for i in range(1, nn):
        n = zs[i].numel()
        zs[i] = flat[off:off + n]
        off += n
    us, bs, ach = ph.bases_from_sketches(dims, tree, ranks, oversampling, samples, seed, zs)
    root = tree.node(0)
    b0 = ph.shard_root(x_cols, nl, nr, lo, hi, us[root.left], ranks[root.left], us[root.right], ranks[root.right])
    dist.all_reduce(b0, group=group)
    leaf = [None] * d
    for i in tree.leaves():
        leaf[tree.node(i).modes[0]] = us[i]
    trs = [None] * nn
    trs[0] = b0
    for i, b in bs.items():
        trs[i] = b
    return ShardedHTucker(leaf_factors=leaf, transfers=trs, node_bases=us, achieved_ranks=ach, columns=(lo, hi))
