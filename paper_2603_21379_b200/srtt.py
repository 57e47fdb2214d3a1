"""Python mirror of the reference's hot-path API over the C-ABI.

Names, argument meaning, validation and error behaviour follow the
reference's C++ API (proj/include/srtt/*.hpp); every compute call goes
through ``libsrtt_b200.so`` (hand-written sm_100a kernels).  There is no
CPU fallback: if the shared library is missing or no B200 is visible, the
calls raise.

Layout conventions (reference tensor.hpp:17-20, common.hpp:21-24): tensors
are flat with the FIRST index fastest -- a numpy array ``x`` of shape dims is
passed as ``np.ravel(x, order="F")``; factors are column-major ``n x r``.

Reference exceptions map to Python ones:
  std::invalid_argument -> InvalidArgument (ValueError)
  std::out_of_range     -> OutOfRange (IndexError)
  JobError(job)         -> JobError (RuntimeError, ``.job`` holds the index)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import load_library

# ---------------------------------------------------------------------------
# errors
# ---------------------------------------------------------------------------
SRTT_OK = 0
SRTT_ERR_INVALID_ARGUMENT = 1
SRTT_ERR_OUT_OF_RANGE = 2
SRTT_ERR_CUDA = 3
SRTT_ERR_NCCL = 4
SRTT_ERR_OUT_OF_MEMORY = 5
SRTT_ERR_INTERNAL = 6
SRTT_ERR_JOB = 7
SRTT_ERR_IO = 8

STAGES = ["sampling", "extract", "sketch", "svd", "transfer", "ttm", "gather", "serial_tail",
          "factor_wall", "h2d", "d2h"]


class SrttError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    pass


class OutOfRange(IndexError):
    pass


class JobError(RuntimeError):
    """parallel.hpp:79-129: first failing job's index + message."""

    def __init__(self, msg):
        super().__init__(msg)
        try:
            self.job = int(msg.split(":", 1)[0].split()[1])
        except Exception:  # pragma: no cover
            self.job = -1


class CudaError(SrttError):
    pass


class IoError(RuntimeError):
    """io.hpp:10-13."""


def _check(rc):
    if rc == SRTT_OK:
        return
    msg = _L().srtt_last_error().decode()
    if rc == SRTT_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == SRTT_ERR_OUT_OF_RANGE:
        raise OutOfRange(msg)
    if rc == SRTT_ERR_JOB:
        raise JobError(msg)
    if rc == SRTT_ERR_IO:
        raise IoError(msg)
    if rc in (SRTT_ERR_CUDA, SRTT_ERR_OUT_OF_MEMORY):
        raise CudaError(msg)
    raise SrttError(f"srtt error {rc}: {msg}")


# ---------------------------------------------------------------------------
# C structs
# ---------------------------------------------------------------------------
class _Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("use_graphs", C.c_int32), ("reserved", C.c_int32 * 6)]


class _Exec(C.Structure):
    _fields_ = [("workers", C.c_int64), ("slice_mode", C.c_int64), ("index_partitions", C.c_int64),
                ("emulate_serial_root", C.c_int32), ("reserved", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("sample_counts", C.POINTER(C.c_int64)), ("achieved_ranks", C.POINTER(C.c_int64)),
                ("warnings", C.c_char_p), ("warnings_capacity", C.c_int64), ("num_warnings", C.c_int64),
                ("stage_seconds", C.c_double * len(STAGES)), ("flags", C.c_int32), ("reserved", C.c_int32),
                ("kernel_seconds", C.c_double * 4), ("launches", C.c_int64), ("slice_mode", C.c_int64),
                ("node_bases", C.c_void_p)]


class _Tree(C.Structure):
    _fields_ = [("num_nodes", C.c_int32), ("mode_begin", C.POINTER(C.c_int32)), ("modes", C.POINTER(C.c_int32)),
                ("left", C.POINTER(C.c_int32)), ("right", C.POINTER(C.c_int32))]


_LIB = None


def _L():
    global _LIB
    if _LIB is None:
        lib = load_library()
        vp = C.c_void_p
        i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
        lib.srtt_last_error.restype = C.c_char_p
        lib.srtt_create.argtypes = [C.POINTER(_Options), C.POINTER(vp)]
        lib.srtt_destroy.argtypes = [vp]
        lib.srtt_last_launch_count.argtypes = [vp]
        lib.srtt_last_launch_count.restype = i64
        lib.srtt_set_stream.argtypes = [vp, vp]
        lib.srtt_sample_indices.argtypes = [u64, u64, i64, i64, i64, vp, vp]
        lib.srtt_stream_normals.argtypes = [vp, u64, u64, u64, u64, i64, vp]
        lib.srtt_tree_balanced.argtypes = [i32] + [vp] * 7
        lib.srtt_pick_slice_mode.argtypes = [i32, vp, i64, vp]
        lib.srtt_sub_r_hosvd.argtypes = [vp, vp, i32, i32, vp, vp, i64, vp, u64, vp, vp, vp, i32, vp]
        lib.srtt_sub_r_rtl_ht.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, i64, u64, vp, vp, vp, i32, vp]
        lib.srtt_extract_fibers.argtypes = [vp, vp, i32, i32, vp, i32, vp, i64, vp, vp, i32]
        lib.srtt_sketch.argtypes = [vp, vp, i32, i32, vp, i32, vp, i64, vp, i32, u64, u64, u64, vp, vp, i32]
        lib.srtt_range_basis_of_sketch.argtypes = [vp, vp, i32, i64, i32, i32, u64, u64, u64, i64, vp, vp, vp,
                                                   i32]
        lib.srtt_multi_ttm_core.argtypes = [vp, vp, i32, i32, vp, vp, vp, i32, vp, i32]
        lib.srtt_transfer_tensor.argtypes = [vp, vp, vp, vp, i64, i64, i32, i32, i32, i32, vp]
        lib.srtt_root_transfer.argtypes = [vp, vp, i32, i64, i64, vp, i32, vp, i32, i32, vp, i32]
        lib.srtt_rel_error.argtypes = [vp, vp, vp, i32, i64, vp]
        lib.srtt_tensor_file_info.argtypes = [C.c_char_p, vp, vp, i32, vp]
        lib.srtt_read_tensor.argtypes = [vp, C.c_char_p, i64, i64, vp, i32, i64]
        lib.srtt_write_tensor.argtypes = [vp, C.c_char_p, i32, vp, vp, i32]
        lib.srtt_write_htucker.argtypes = [C.c_char_p, i32, vp, vp, vp, vp, vp]
        lib.srtt_read_htucker.argtypes = [C.c_char_p] + [vp] * 11
        lib.srtt_tucker_reconstruct.argtypes = [vp, i32, vp, vp, vp, vp, i32, vp, i32]
        lib.srtt_tucker_rel_error.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, i32, vp]
        lib.srtt_ht_reconstruct.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32, vp, i32]
        lib.srtt_ht_rel_error.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, vp, i32, vp]
        lib.srtt_comm_unique_id.argtypes = [vp]
        lib.srtt_comm_init.argtypes = [vp, i32, i32, vp]
        lib.srtt_comm_destroy.argtypes = [vp]
        lib.srtt_comm_info.argtypes = [vp, vp, vp]
        lib.srtt_split_bounds.argtypes = [i64, i32, i32, vp, vp]
        lib.srtt_sub_r_hosvd_sharded.argtypes = [vp, vp, i32, i32, vp, i64, i64, vp, i64, vp, u64, vp, vp, vp, i32,
                                                 vp]
        lib.srtt_sub_r_rtl_ht_sharded.argtypes = [vp, vp, i32, i32, vp, i64, i64, vp, vp, vp, i64, u64, vp, vp, vp,
                                                  i32, vp]
        lib.srtt_sub_r_hosvd_replicated.argtypes = [vp, vp, i32, i32, vp, vp, i64, vp, u64, vp, vp, vp, i32, vp]
        lib.srtt_sub_r_rtl_ht_replicated.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, i64, u64, vp, vp, vp, i32,
                                                     vp]
        _LIB = lib
    return _LIB


def _ptr(a):
    """(pointer, on_device) of a numpy array or a CUDA torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data, 0
    if hasattr(a, "data_ptr") and getattr(a, "is_cuda", False):
        return a.data_ptr(), 1
    raise TypeError(f"unsupported buffer type {type(a)}")


def _i64(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64))


def _flat_f64(x):
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(np.ravel(x, order="F"), dtype=np.float64)
    if hasattr(x, "is_cuda") and x.is_cuda:
        import torch

        if x.dtype != torch.float64 or not x.is_contiguous():
            raise TypeError("device tensors must be contiguous float64 (first index fastest)")
        return x
    return np.ascontiguousarray(np.ravel(np.asarray(x, dtype=np.float64), order="F"))


# ---------------------------------------------------------------------------
# handle
# ---------------------------------------------------------------------------
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


class Handle:
    """Owns a device, a stream, the workspace arena and pinned staging."""

    def __init__(self, device: int = 0, use_graphs: bool = True):
        self._h = C.c_void_p()
        opts = _Options(device=device, use_graphs=int(use_graphs))
        _check(_L().srtt_create(C.byref(opts), C.byref(self._h)))
        self.device = device

    def close(self):
        if getattr(self, "_h", None) and self._h.value and _LIB is not None:
            _LIB.srtt_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()

    def set_stream(self, stream_ptr):
        """Run on an external cudaStream_t (int handle, e.g. torch's
        ``torch.cuda.current_stream().cuda_stream``); None = the handle's own
        stream. ``0`` is torch's default stream, i.e. the legacy default
        stream (``cudaStreamLegacy``): the engine's work is then ordered with
        it (graphs are captured on the own stream and launched into it)."""
        if stream_ptr is None:
            ptr = None
        elif stream_ptr == 0:
            ptr = C.c_void_p(CUDA_STREAM_LEGACY)
        else:
            ptr = C.c_void_p(stream_ptr)
        _check(_L().srtt_set_stream(self._h, ptr))

    @property
    def last_launch_count(self) -> int:
        return int(_L().srtt_last_launch_count(self._h))


_DEFAULT = {}


def default_handle(device: int = 0) -> Handle:
    if device not in _DEFAULT:
        _DEFAULT[device] = Handle(device)
    return _DEFAULT[device]


# ---------------------------------------------------------------------------
# reference-shaped types
# ---------------------------------------------------------------------------
@dataclass
class ExecPolicy:
    """parallel.hpp:23-28."""
    workers: int = 1
    slice_mode: int | None = None
    index_partitions: int = 1
    emulate_serial_root: bool = False

    def _c(self):
        return _Exec(self.workers, -1 if self.slice_mode is None else self.slice_mode, self.index_partitions,
                     int(self.emulate_serial_root), 0)


@dataclass
class SubsampleReport:
    """tucker.hpp:129-134 / htucker.hpp:196-201, plus device stage times."""
    sample_counts: list = field(default_factory=list)
    achieved_ranks: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    timings: dict = field(default_factory=dict)
    flags: int = 0
    launches: int = 0
    kernel_seconds: dict = field(default_factory=dict)
    slice_mode: int | None = None
    # H-Tucker: set want_node_bases to get every node's basis (id -> U_S)
    want_node_bases: bool = False
    node_bases: dict = field(default_factory=dict)


HtSubsampleReport = SubsampleReport


@dataclass
class TuckerDecomposition:
    core: object      # numpy nd-array of shape ranks (or a flat device tensor)
    factors: list     # U_k, n_k x r_k


@dataclass
class HTuckerDecomposition:
    tree: "DimensionTree"
    leaf_factors: list
    transfers: list


class TreeNode:
    def __init__(self, modes, left, right, parent, level):
        self.modes = [int(m) for m in modes]
        self.left, self.right, self.parent, self.level = left, right, parent, level

    def is_leaf(self):
        return self.left < 0


class DimensionTree:
    """dimension_tree.hpp:27-152 (balanced() is computed by the library)."""

    def __init__(self, nodes):
        self.nodes = nodes

    @staticmethod
    def balanced(order: int) -> "DimensionTree":
        n = max(2 * order - 1, 1)
        nn = C.c_int32()
        mb = np.zeros(n + 1, np.int32)
        modes = np.zeros(max(order * order, 1), np.int32)
        left, right, parent, level = (np.zeros(n, np.int32) for _ in range(4))
        _check(_L().srtt_tree_balanced(order, C.byref(nn), mb.ctypes.data, modes.ctypes.data, left.ctypes.data,
                                       right.ctypes.data, parent.ctypes.data, level.ctypes.data))
        nodes = [TreeNode(modes[mb[i]:mb[i + 1]], int(left[i]), int(right[i]), int(parent[i]), int(level[i]))
                 for i in range(nn.value)]
        return DimensionTree(nodes)

    @property
    def num_nodes(self):
        return len(self.nodes)

    @property
    def order(self):
        return len(self.nodes[0].modes)

    def node(self, i):
        return self.nodes[i]

    def leaves(self):
        return [i for i, n in enumerate(self.nodes) if n.is_leaf()]

    def depth(self):
        return max(n.level for n in self.nodes)

    def internal_nodes_bottom_up(self):
        out = []
        for lvl in range(self.depth(), 0, -1):
            out += [i for i in range(1, self.num_nodes) if not self.nodes[i].is_leaf() and self.nodes[i].level == lvl]
        return out

    def node_rows(self, i, dims):
        return int(np.prod([dims[m] for m in self.nodes[i].modes]))

    def node_cols(self, i, dims):
        return int(np.prod(dims)) // self.node_rows(i, dims)

    def _c(self):
        mb, modes = [0], []
        for n in self.nodes:
            modes += [int(m) for m in n.modes]
            mb.append(len(modes))
        self._keep = [np.asarray(mb, np.int32), np.asarray(modes or [0], np.int32),
                      np.asarray([n.left for n in self.nodes], np.int32),
                      np.asarray([n.right for n in self.nodes], np.int32)]
        P = C.POINTER(C.c_int32)
        return _Tree(len(self.nodes), *(k.ctypes.data_as(P) for k in self._keep))


def uniform_node_ranks(tree, rank):
    """dimension_tree.hpp:159-163."""
    out = [rank] * tree.num_nodes
    out[0] = 1
    return out


def node_sample_counts(tree, dims, alpha):
    """dimension_tree.hpp:174-183."""
    import math

    out = [1] * tree.num_nodes
    for i in range(1, tree.num_nodes):
        out[i] = min(int(math.ceil(alpha * tree.node_rows(i, dims))), tree.node_cols(i, dims))
    return out
    return out


# ---------------------------------------------------------------------------
# sampling (host, bit-exact)
# ---------------------------------------------------------------------------
def sample_indices(m: int, s: int, seed: int, stream_id: int, partitions: int = 1):
    """RngStream(seed, stream_id) + sample_indices[_partitioned]; returns
    (indices, u64 draws consumed by the parent stream)."""
    out = np.zeros(max(int(s), 1), np.int64)
    draws = C.c_uint64()
    _check(_L().srtt_sample_indices(seed & (2**64 - 1), stream_id & (2**64 - 1), m, s, partitions,
                                    out.ctypes.data, C.byref(draws)))
    return out[:s], int(draws.value)


def stream_normals(seed, stream_id, draw_offset, t0, n, handle=None):
    """Device generator of the stream's normals (K1's Omega source)."""
    h = handle or default_handle()
    out = np.zeros(n)
    _check(_L().srtt_stream_normals(h._h, seed, stream_id, draw_offset, t0, n, out.ctypes.data))
    return out


# ---------------------------------------------------------------------------
# decompositions
# ---------------------------------------------------------------------------
def _report_from(crep, n, ach, samp, report, handle):
    if report is None:
        return
    report.sample_counts = [int(v) for v in samp[:n]]
    report.achieved_ranks = [int(v) for v in ach[:n]]
    txt = crep.warnings.decode() if crep.warnings else ""
    report.warnings = [w for w in txt.split("\n") if w]
    report.timings = {name: float(crep.stage_seconds[i]) for i, name in enumerate(STAGES)}
    report.flags = int(crep.flags)
    report.launches = int(crep.launches)
    report.jacobi_sweeps = int(crep.reserved)
    report.slice_mode = None if int(crep.slice_mode) < 0 else int(crep.slice_mode)
    report.kernel_seconds = {"sketch": float(crep.kernel_seconds[0]), "basis": float(crep.kernel_seconds[1]),
                             "core": float(crep.kernel_seconds[2]), "transfer": float(crep.kernel_seconds[3])}


def _alloc_out(shape_list, device_out, like):
    if device_out:
        import torch

        dev = like.device if hasattr(like, "device") else torch.device("cuda")
        return [torch.empty(int(np.prod(s)), dtype=torch.float64, device=dev) for s in shape_list]
    return [np.zeros(int(np.prod(s))) for s in shape_list]


class _TuckerCall:
    """Per-signature cache of the ctypes argument blocks of one Tucker call
    (keeps the per-call Python overhead to a handful of microseconds)."""

    def __init__(self, dims, target, samples):
        d = len(dims)
        self.d = d
        self.dims_a, self.ranks_a, self.samp_a = _i64(dims), _i64(target), _i64(samples)
        self.ach, self.sc = np.zeros(d, np.int64), np.zeros(d, np.int64)
        self.wbuf = C.create_string_buffer(8192)
        self.rep = _Report(self.sc.ctypes.data_as(C.POINTER(C.c_int64)),
                           self.ach.ctypes.data_as(C.POINTER(C.c_int64)), C.cast(self.wbuf, C.c_char_p), 8192, 0)
        self.fptrs = (C.c_void_p * d)()


_CALLS = {}


def sub_r_hosvd(x, target, oversampling, samples, seed, exec_policy=None, report=None, *, dims=None,
                handle=None, device_out=False, out=None):
    """tucker.hpp:177-242.  ``x``: numpy nd-array (dims taken from its shape)
    or a flat float64 array / CUDA tensor together with ``dims``.
    ``out=(core, [factors])`` reuses caller-allocated outputs (flat, device
    tensors when ``device_out``)."""
    h = handle or default_handle()
    if dims is None:
        dims = list(np.shape(x))
    d = len(dims)
    xf = _flat_f64(x)
    xp, xdev = _ptr(xf)
    if len(target) != d:
        raise InvalidArgument("sub_r_hosvd: rank vector order mismatch")
    if len(samples) != len(target):
        raise InvalidArgument("sub_r_hosvd: samples vector order mismatch")
    key = (tuple(dims), tuple(target), tuple(samples))
    call = _CALLS.get(key)
    if call is None:
        call = _CALLS.setdefault(key, _TuckerCall(dims, target, samples))
    if out is None:
        outs = _alloc_out([call.ranks_a] + [(dims[k], target[k]) for k in range(d)], device_out, xf)
    else:
        outs = [out[0]] + list(out[1])
    for k in range(d):
        call.fptrs[k] = _ptr(outs[k + 1])[0]
    ex = exec_policy._c() if exec_policy is not None else None
    # device outputs without a report: stream-ordered (asynchronous) call
    rep_arg = C.byref(call.rep) if (report is not None or not device_out) else None
    _check(_L().srtt_sub_r_hosvd(h._h, xp, xdev, d, call.dims_a.ctypes.data, call.ranks_a.ctypes.data,
                                 int(oversampling), call.samp_a.ctypes.data, int(seed) & (2**64 - 1),
                                 C.byref(ex) if ex is not None else None, _ptr(outs[0])[0], call.fptrs,
                                 int(device_out), rep_arg))
    if report is not None:
        _report_from(call.rep, d, call.ach, call.sc, report, h)
    if device_out:
        return TuckerDecomposition(core=outs[0], factors=outs[1:])
    core = outs[0].reshape(tuple(int(r) for r in target), order="F")
    factors = [outs[k + 1].reshape((dims[k], target[k]), order="F") for k in range(d)]
    return TuckerDecomposition(core=core, factors=factors)


def sub_r_rtl_ht(x, tree, ranks, samples, oversampling, seed, exec_policy=None, report=None, *, dims=None,
                 handle=None, device_out=False):
    """htucker.hpp:210-341."""
    h = handle or default_handle()
    if dims is None:
        dims = list(np.shape(x))
    d = len(dims)
    xf = _flat_f64(x)
    xp, xdev = _ptr(xf)
    if tree.order != d:
        raise InvalidArgument("sub_r_rtl_ht: tree and tensor order mismatch")
    nn = tree.num_nodes
    if len(ranks) != nn:
        raise InvalidArgument("sub_r_rtl_ht: rank vector must have one entry per node")
    if len(samples) != nn:
        raise InvalidArgument("sub_r_rtl_ht: samples vector must have one entry per node")
    ranks_a, samp_a, dims_a = _i64(ranks), _i64(samples), _i64(dims)
    leaf_shape = [None] * d
    for i in tree.leaves():
        m = tree.node(i).modes[0]
        leaf_shape[m] = (dims[m], ranks[i])
    tshape = {}
    for i in range(nn):
        n = tree.node(i)
        if not n.is_leaf():
            tshape[i] = (1 if i == 0 else ranks[i], ranks[n.left], ranks[n.right])
    leaf = _alloc_out(leaf_shape, device_out, xf)
    trs = {i: _alloc_out([s], device_out, xf)[0] for i, s in tshape.items()}
    lp = (C.c_void_p * d)(*[_ptr(o)[0] for o in leaf])
    tp = (C.c_void_p * nn)(*[_ptr(trs[i])[0] if i in trs else None for i in range(nn)])
    ach, sc = np.zeros(nn, np.int64), np.zeros(nn, np.int64)
    wbuf = C.create_string_buffer(8192)
    crep = _Report(sc.ctypes.data_as(C.POINTER(C.c_int64)), ach.ctypes.data_as(C.POINTER(C.c_int64)),
                   C.cast(wbuf, C.c_char_p), 8192, 0)
    nb = None
    if report is not None and getattr(report, "want_node_bases", False):
        # every node's basis as used by the decomposition (internal nodes too)
        nshape = {i: (tree.node_rows(i, dims), ranks[i]) for i in range(1, nn)}
        nb = {i: _alloc_out([nshape[i]], device_out, xf)[0] for i in range(1, nn)}
        nbp = (C.c_void_p * nn)(*([None] + [_ptr(nb[i])[0] for i in range(1, nn)]))
        crep.node_bases = C.cast(nbp, C.c_void_p)
    ct = tree._c()
    ex = exec_policy._c() if exec_policy is not None else None
    # device outputs and no report: the call is stream-ordered (returns
    # before the kernels finish, like sub_r_hosvd)
    rep_arg = None if (device_out and report is None) else C.byref(crep)
    _check(_L().srtt_sub_r_rtl_ht(h._h, xp, xdev, d, dims_a.ctypes.data, C.byref(ct), ranks_a.ctypes.data,
                                  samp_a.ctypes.data, int(oversampling), int(seed) & (2**64 - 1),
                                  C.byref(ex) if ex is not None else None, lp, tp, int(device_out), rep_arg))
    if rep_arg is not None:
        _report_from(crep, nn, ach, sc, report, h)
        if nb is not None:
            report.node_bases = {i: (b if device_out else b.reshape(nshape[i], order="F")) for i, b in nb.items()}
    if device_out:
        return HTuckerDecomposition(tree, leaf, [trs.get(i) for i in range(nn)])
    leaf_np = [leaf[m].reshape(leaf_shape[m], order="F") for m in range(d)]
    tr_np = [trs[i].reshape(tshape[i], order="F") if i in trs else None for i in range(nn)]
    return HTuckerDecomposition(tree, leaf_np, tr_np)


# ---------------------------------------------------------------------------
# components (reference test-facing functions)
# ---------------------------------------------------------------------------
def extract_group_fibers(x, modes, cols, *, handle=None):
    """unfolding.hpp:57-111 (a single mode == extract_fibers)."""
    h = handle or default_handle()
    dims = list(x.shape)
    xf = _flat_f64(x)
    modes_a = np.ascontiguousarray(np.asarray(modes, np.int32))
    cols_a = _i64(cols)
    rows = int(np.prod([dims[m] for m in modes])) if len(modes) else 0
    y = np.zeros(max(rows * len(cols_a), 1))
    dims_a = _i64(dims)  # keep alive across the call
    _check(_L().srtt_extract_fibers(h._h, xf.ctypes.data, 0, len(dims), dims_a.ctypes.data, len(modes_a),
                                    modes_a.ctypes.data, len(cols_a), cols_a.ctypes.data, y.ctypes.data, 0))
    return y[:rows * len(cols_a)].reshape((rows, len(cols_a)), order="F")


def extract_fibers(x, mode, cols, *, handle=None):
    """unfolding.hpp:32-52."""
    return extract_group_fibers(x, [mode], cols, handle=handle)


def sketch(x, modes, cols, c, seed, stream_id, draw_offset, omega=None, *, dims=None, handle=None):
    """K1 alone: Z = Y(cols) * Omega, Omega from stream (seed, stream_id).
    ``x``: numpy nd-array, or a flat CUDA float64 tensor with ``dims``."""
    h = handle or default_handle()
    dims = list(x.shape) if dims is None else list(dims)
    xf = _flat_f64(x)
    xp, xdev = _ptr(xf)
    modes_a = np.ascontiguousarray(np.asarray(modes, np.int32))
    cols_a = _i64(cols)
    rows = int(np.prod([dims[m] for m in modes]))
    z = np.zeros(rows * c)
    om = None if omega is None else np.ascontiguousarray(np.ravel(omega, order="F"), dtype=np.float64)
    dims_a = _i64(dims)
    _check(_L().srtt_sketch(h._h, xp, xdev, len(dims), dims_a.ctypes.data, len(modes_a),
                            modes_a.ctypes.data, len(cols_a), cols_a.ctypes.data, c, seed, stream_id, draw_offset,
                            om.ctypes.data if om is not None else None, z.ctypes.data, 0))
    return z.reshape((rows, c), order="F")


@dataclass
class RangeBasis:
    q: np.ndarray
    numerical_rank: int
    singular_values: np.ndarray


def range_basis_of_sketch(z, rank, seed=0, stream_id=0, draw_offset=0, normal_base=0, *, handle=None):
    """sketch.hpp:74-93 (padding continues stream (seed, stream_id))."""
    h = handle or default_handle()
    z = np.asarray(z, dtype=np.float64)
    n, c = z.shape
    zf = np.ascontiguousarray(np.ravel(z, order="F"))
    q = np.zeros(n * max(rank, 1))
    nr = C.c_int64()
    sv = np.zeros(min(n, c))
    _check(_L().srtt_range_basis_of_sketch(h._h, zf.ctypes.data, 0, n, c, rank, seed, stream_id, draw_offset,
                                           normal_base, q.ctypes.data, C.byref(nr), sv.ctypes.data, 0))
    return RangeBasis(q.reshape((n, rank), order="F"), int(nr.value), sv)


def multi_ttm_core(x, factors, *, handle=None):
    """core_from_factors (tucker.hpp:43-50) / sliced_core (parallel.hpp:355-445)."""
    h = handle or default_handle()
    dims = list(x.shape)
    ranks = [f.shape[1] for f in factors]
    xf = _flat_f64(x)
    fs = [np.ascontiguousarray(np.ravel(f, order="F"), dtype=np.float64) for f in factors]
    fp = (C.c_void_p * len(fs))(*[f.ctypes.data for f in fs])
    out = np.zeros(int(np.prod(ranks)))
    dims_a, ranks_a = _i64(dims), _i64(ranks)
    _check(_L().srtt_multi_ttm_core(h._h, xf.ctypes.data, 0, len(dims), dims_a.ctypes.data,
                                    ranks_a.ctypes.data, fp, 0, out.ctypes.data, 0))
    return out.reshape(tuple(ranks), order="F")


core_from_factors = multi_ttm_core


def pick_slice_mode(dims, workers):
    """parallel.hpp:331-348."""
    out = C.c_int64()
    dims_a = _i64(dims)
    _check(_L().srtt_pick_slice_mode(len(dims_a), dims_a.ctypes.data, int(workers), C.byref(out)))
    return int(out.value)


def sliced_core(x, factors, policy=None, *, handle=None):
    """parallel.hpp:355-445: the policy is validated as the reference does
    (slice mode, workers vs slices); the numbers are the same for every
    policy (one streaming pass on the GPU)."""
    if len(factors) != x.ndim:
        raise InvalidArgument("sliced_core: need one factor per mode")
    for k, f in enumerate(factors):
        if np.shape(f)[0] != x.shape[k]:
            raise InvalidArgument(f"sliced_core: factor rows mismatch in mode {k}")
    policy = policy or ExecPolicy()
    sm = policy.slice_mode if policy.slice_mode is not None else pick_slice_mode(x.shape, policy.workers)
    if not 0 <= sm < x.ndim:
        raise InvalidArgument("sliced_core: slice mode out of range")
    if policy.workers > x.shape[sm]:
        raise InvalidArgument("sliced_core: more workers than slices along the slicing mode")
    return multi_ttm_core(x, factors, handle=handle)


def transfer_tensor(u_node, u_left, u_right, *, handle=None):
    """htucker.hpp:44-63."""
    h = handle or default_handle()
    nl, rl = u_left.shape
    nr, rr = u_right.shape
    if u_node.shape[0] != nl * nr:
        raise InvalidArgument("transfer_tensor: node rows must equal product of child rows")
    rs = u_node.shape[1]
    a, b, c = (np.ascontiguousarray(np.ravel(m, order="F"), dtype=np.float64) for m in (u_node, u_left, u_right))
    out = np.zeros(rs * rl * rr)
    _check(_L().srtt_transfer_tensor(h._h, a.ctypes.data, b.ctypes.data, c.ctypes.data, nl, nr, rs, rl, rr, 0,
                                     out.ctypes.data))
    return out.reshape((rs, rl, rr), order="F")


def root_transfer(x, u_left, u_right, *, handle=None):
    """htucker.hpp:67-85."""
    h = handle or default_handle()
    nl, rl = u_left.shape
    nr, rr = u_right.shape
    if nl * nr != x.size:
        raise InvalidArgument("root_transfer: child rows do not factor the tensor size")
    xf = _flat_f64(x)
    a, b = (np.ascontiguousarray(np.ravel(m, order="F"), dtype=np.float64) for m in (u_left, u_right))
    out = np.zeros(rl * rr)
    _check(_L().srtt_root_transfer(h._h, xf.ctypes.data, 0, nl, nr, a.ctypes.data, rl, b.ctypes.data, rr, 0,
                                   out.ctypes.data, 0))
    return out.reshape((1, rl, rr), order="F")


# ---------------------------------------------------------------------------
# reconstruction and error (the step after the path, experiment.cpp:248/266)
# ---------------------------------------------------------------------------
def _is_dev(a):
    return hasattr(a, "is_cuda") and a.is_cuda


def _mat_f64(a):
    """Flat column-major float64 buffer of a factor / core / transfer."""
    if _is_dev(a):
        return _flat_f64(a.reshape(-1) if a.is_contiguous() else a.contiguous().reshape(-1))
    return np.ascontiguousarray(np.ravel(np.asarray(a, dtype=np.float64), order="F"))


def _numel(a):
    return int(a.numel()) if _is_dev(a) else int(np.size(a))


def _tucker_args(t, dims):
    factors = [_mat_f64(u) for u in t.factors]
    core = _mat_f64(t.core)
    if dims is None:
        dims = [int(np.shape(u)[0]) for u in t.factors]
        if any(np.ndim(u) != 2 for u in t.factors):
            raise InvalidArgument("reconstruct: pass dims= for flat factors")
    ranks = [_numel(f) // n for f, n in zip(factors, dims)]
    if int(np.prod(ranks)) != _numel(core):
        raise InvalidArgument("reconstruct: factor/core mismatch")
    ondev = {_is_dev(a) for a in factors + [core]}
    if len(ondev) != 1:
        raise InvalidArgument("reconstruct: core and factors must all be host or all be device buffers")
    fp = (C.c_void_p * len(factors))(*[_ptr(f)[0] for f in factors])
    return factors, core, list(dims), ranks, fp, int(ondev.pop())


def reconstruct(t, *, dims=None, handle=None, device_out=False):
    """tucker.hpp:18-28: G x_0 U_0 ... x_{d-1} U_{d-1} on the GPU."""
    h = handle or default_handle()
    factors, core, dims, ranks, fp, dev = _tucker_args(t, dims)
    out = _alloc_out([(int(np.prod(dims)),)], device_out, core if dev else np.zeros(1))[0]
    dims_a, ranks_a = _i64(dims), _i64(ranks)
    _check(_L().srtt_tucker_reconstruct(h._h, len(dims), dims_a.ctypes.data, ranks_a.ctypes.data, _ptr(core)[0], fp,
                                        dev, _ptr(out)[0], int(device_out)))
    return out if device_out else out.reshape(tuple(dims), order="F")


def tucker_rel_error(x, t, *, dims=None, handle=None):
    """rel_error(x, reconstruct(t)) (experiment.cpp:248) streamed on the GPU:
    X-hat is recomputed tile by tile and never materialised."""
    h = handle or default_handle()
    factors, core, dims, ranks, fp, dev = _tucker_args(t, dims)
    xf = _flat_f64(x)
    xp, xdev = _ptr(xf)
    if _numel(xf) != int(np.prod(dims)):
        raise InvalidArgument("rel_error: shape mismatch")
    out = C.c_double()
    dims_a, ranks_a = _i64(dims), _i64(ranks)
    _check(_L().srtt_tucker_rel_error(h._h, xp, xdev, len(dims), dims_a.ctypes.data, ranks_a.ctypes.data,
                                      _ptr(core)[0], fp, dev, C.byref(out)))
    return float(out.value)


def _ht_args(hd, dims):
    tree = hd.tree
    d = tree.order
    leaf = [_mat_f64(u) for u in hd.leaf_factors]
    if dims is None:
        dims = [int(np.shape(u)[0]) for u in hd.leaf_factors]
    ranks = [0] * tree.num_nodes
    for i in tree.leaves():
        m = tree.node(i).modes[0]
        ranks[i] = _numel(leaf[m]) // dims[m]
    trs = [None if b is None else _mat_f64(b) for b in hd.transfers]
    for i in tree.internal_nodes_bottom_up() + [0]:
        n = tree.node(i)
        ranks[i] = _numel(trs[i]) // (ranks[n.left] * ranks[n.right])
    if ranks[0] != 1:
        raise InvalidArgument("ht_reconstruct: root rank must be 1")
    bufs = leaf + [b for b in trs if b is not None]
    ondev = {_is_dev(a) for a in bufs}
    if len(ondev) != 1:
        raise InvalidArgument("ht_reconstruct: leaf factors and transfers must all be host or all be device")
    lp = (C.c_void_p * d)(*[_ptr(u)[0] for u in leaf])
    tp = (C.c_void_p * tree.num_nodes)(*[None if b is None else _ptr(b)[0] for b in trs])
    return leaf, trs, list(dims), ranks, lp, tp, int(ondev.pop()), bufs


def ht_reconstruct(hd, *, dims=None, handle=None, device_out=False):
    """htucker.hpp:346-378 on the GPU."""
    h = handle or default_handle()
    leaf, trs, dims, ranks, lp, tp, dev, keep = _ht_args(hd, dims)
    out = _alloc_out([(int(np.prod(dims)),)], device_out, keep[0] if dev else np.zeros(1))[0]
    dims_a, ranks_a = _i64(dims), _i64(ranks)
    ct = hd.tree._c()
    _check(_L().srtt_ht_reconstruct(h._h, len(dims), dims_a.ctypes.data, C.byref(ct), ranks_a.ctypes.data, lp, tp,
                                    dev, _ptr(out)[0], int(device_out)))
    return out if device_out else out.reshape(tuple(dims), order="F")


def ht_rel_error(x, hd, *, dims=None, handle=None):
    """rel_error(x, ht_reconstruct(h)) (experiment.cpp:266), streamed."""
    h = handle or default_handle()
    leaf, trs, dims, ranks, lp, tp, dev, keep = _ht_args(hd, dims)
    xf = _flat_f64(x)
    xp, xdev = _ptr(xf)
    if _numel(xf) != int(np.prod(dims)):
        raise InvalidArgument("rel_error: shape mismatch")
    out = C.c_double()
    dims_a, ranks_a = _i64(dims), _i64(ranks)
    ct = hd.tree._c()
    _check(_L().srtt_ht_rel_error(h._h, xp, xdev, len(dims), dims_a.ctypes.data, C.byref(ct), ranks_a.ctypes.data,
                                  lp, tp, dev, C.byref(out)))
    return float(out.value)


def rel_error(reference, approx, *, handle=None):
    """tensor.hpp:241-249."""
    h = handle or default_handle()
    a, b = _flat_f64(reference), _flat_f64(approx)
    if np.shape(reference) != np.shape(approx) and not (_is_dev(a) and a.numel() == b.numel()):
        raise InvalidArgument("rel_error: shape mismatch")
    pa, da = _ptr(a)
    pb, db = _ptr(b)
    if da != db:
        raise InvalidArgument("rel_error: both tensors must be host or both device buffers")
    out = C.c_double()
    _check(_L().srtt_rel_error(h._h, pa, pb, da, _numel(a), C.byref(out)))
    return float(out.value)


# ---------------------------------------------------------------------------
# containers (io.hpp:15-33)
# ---------------------------------------------------------------------------
def _path(p):
    import os

    return os.fsencode(p)


def tensor_file_info(path):
    """Dimensions and payload offset of an SRTT file."""
    order = C.c_int32()
    dims = np.zeros(64, np.int64)
    off = C.c_int64()
    _check(_L().srtt_tensor_file_info(_path(path), C.byref(order), dims.ctypes.data, 64, C.byref(off)))
    return [int(v) for v in dims[:order.value]], int(off.value)


def read_tensor(path, *, slab=None, device=False, handle=None):
    """read_tensor (io.cpp:106-117).  ``slab=(lo, hi)`` reads X[..., lo:hi)
    only (one contiguous byte range).  ``device=True`` returns a flat CUDA
    float64 tensor streamed through pinned staging; otherwise a numpy array
    of the (slab) shape."""
    dims, _ = tensor_file_info(path)
    lo, hi = (-1, -1) if slab is None else (int(slab[0]), int(slab[1]))
    shape = list(dims) if slab is None else dims[:-1] + [hi - lo]
    if slab is not None and not (0 <= lo < hi <= dims[-1]):
        raise InvalidArgument("read_tensor: slab out of range")
    n = int(np.prod(shape))
    if device:
        import torch

        h = handle or default_handle()
        out = torch.empty(n, dtype=torch.float64, device=f"cuda:{h.device}")
        _check(_L().srtt_read_tensor(h._h, _path(path), lo, hi, out.data_ptr(), 1, n))
        return out
    out = np.empty(n, dtype=np.float64)
    _check(_L().srtt_read_tensor(handle._h if handle else None, _path(path), lo, hi, out.ctypes.data, 0, n))
    return out.reshape(tuple(shape), order="F")


def write_tensor(path, x, *, dims=None, handle=None):
    """write_tensor (io.cpp:92-104); x: numpy array or flat CUDA tensor (dims=)."""
    if dims is None:
        dims = list(np.shape(x))
    xf = _flat_f64(x)
    p, dev = _ptr(xf)
    h = (handle or default_handle()) if dev else handle
    dims_a = _i64(dims)
    _check(_L().srtt_write_tensor(h._h if h else None, _path(path), len(dims), dims_a.ctypes.data, p, dev))


def write_htucker(path, hd):
    """write_htucker (io.cpp:123-150), host arrays."""
    tree = hd.tree
    d = tree.order
    dims = [int(np.shape(hd.leaf_factors[m])[0]) for m in range(d)]
    ranks = [0] * tree.num_nodes
    for i in tree.leaves():
        ranks[i] = int(np.shape(hd.leaf_factors[tree.node(i).modes[0]])[1])
    for i in range(tree.num_nodes):
        if not tree.node(i).is_leaf():
            ranks[i] = int(np.shape(hd.transfers[i])[0])
    leaf = [np.ascontiguousarray(np.ravel(u, order="F"), dtype=np.float64) for u in hd.leaf_factors]
    trs = [None if b is None else np.ascontiguousarray(np.ravel(b, order="F"), dtype=np.float64)
           for b in hd.transfers]
    lp = (C.c_void_p * d)(*[u.ctypes.data for u in leaf])
    tp = (C.c_void_p * tree.num_nodes)(*[None if b is None else b.ctypes.data for b in trs])
    ct = tree._c()
    dims_a, ranks_a = _i64(dims), _i64(ranks)
    _check(_L().srtt_write_htucker(_path(path), d, dims_a.ctypes.data, C.byref(ct), ranks_a.ctypes.data, lp, tp))


def read_htucker(path):
    """read_htucker (io.cpp:152-212) -> HTuckerDecomposition (host arrays)."""
    lib = _L()
    order, nn, nm = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib.srtt_read_htucker(_path(path), C.byref(order), C.byref(nn), C.byref(nm), *([None] * 8)))
    d, n = order.value, nn.value
    mb = np.zeros(n + 1, np.int32)
    modes = np.zeros(max(nm.value, 1), np.int32)
    left, right = np.zeros(n, np.int32), np.zeros(n, np.int32)
    ranks, dims = np.zeros(n, np.int64), np.zeros(d, np.int64)
    _check(lib.srtt_read_htucker(_path(path), None, None, None, mb.ctypes.data, modes.ctypes.data,
                                 left.ctypes.data, right.ctypes.data, ranks.ctypes.data, dims.ctypes.data,
                                 None, None))
    parent, level = [-1] * n, [0] * n
    for i in range(n):
        if left[i] >= 0:
            parent[left[i]] = parent[right[i]] = i
    for i in range(1, n):
        level[i] = level[parent[i]] + 1
    nodes = [TreeNode(modes[mb[i]:mb[i + 1]], int(left[i]), int(right[i]), parent[i], level[i]) for i in range(n)]
    tree = DimensionTree(nodes)
    leaf = [None] * d
    trs = [None] * n
    for i in range(n):
        if left[i] < 0:
            m = int(modes[mb[i]])
            leaf[m] = np.zeros((int(dims[m]), int(ranks[i])), order="F")
        else:
            trs[i] = np.zeros((int(ranks[i]), int(ranks[left[i]]), int(ranks[right[i]])), order="F")
    lp = (C.c_void_p * d)(*[u.ctypes.data for u in leaf])
    tp = (C.c_void_p * n)(*[None if b is None else b.ctypes.data for b in trs])
    _check(lib.srtt_read_htucker(_path(path), None, None, None, None, None, None, None, None, None, lp, tp))
    return HTuckerDecomposition(tree, leaf, trs)
