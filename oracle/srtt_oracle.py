"""ORACLE — test infrastructure only.  Never imported by the product path.

CPU restatement (numpy + the C restatement of the RNG in rng_oracle.c) of the
reference's Sub-R-HOSVD and Sub-R-RtL-HT path, used by tests/ as the parity
checker, by ``__graft_entry__.smoke()`` as the checker, and by bench.py's
``cpu_baseline`` / ``--impl reference`` leg as the CPU baseline ("port").

Every function cites the reference file:line it restates.  Storage
conventions follow the reference: tensors are flat with the FIRST index
fastest (tensor.hpp:17-20) -- here numpy arrays whose Fortran-order ravel is
that flat vector; matrices are column-major (common.hpp:21-24).

Pinning: the RNG/sampler is pinned bit-for-bit against the reference's own
rng.hpp/sampling.hpp (compiled in oracle/_ref) and the Appendix-A known
answers (tests/test_oracle_rng.py).  The linear algebra crosses the Eigen
boundary (BDCSVD, GEMM; Eigen is absent here), so it is pinned to the
reference's property tests (recovery medians, orthonormality, Kronecker
oracles, sliced-core equivalence) -- restated in tests/test_oracle_props.py.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_LIB_LOCK = threading.Lock()


def _lib():
    global _LIB
    with _LIB_LOCK:
        if _LIB is None:
            path = os.path.join(_HERE, "_build", "liboracle_rng.so")
            if not os.path.exists(path):
                import subprocess

                subprocess.run(["make", "-s", "-C", _HERE, os.path.join(_HERE, "_build", "liboracle_rng.so")],
                               check=True)
            lib = C.CDLL(path)
            lib.orc_stream_new.restype = C.c_void_p
            lib.orc_stream_new.argtypes = [C.c_uint64, C.c_uint64]
            lib.orc_stream_delete.argtypes = [C.c_void_p]
            lib.orc_stream_sample.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
            lib.orc_stream_normals.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
            lib.orc_stream_u64.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
            lib.orc_stream_uniform.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
            lib.orc_stream_draws.restype = C.c_uint64
            lib.orc_stream_draws.argtypes = [C.c_void_p]
            lib.orc_stream_state0.restype = C.c_uint64
            lib.orc_stream_state0.argtypes = [C.c_uint64, C.c_uint64]
            _LIB = lib
    return _LIB


# --------------------------------------------------------------------------
# RNG (rng.hpp:30-86) and sampling (sampling.hpp:14-77)
# --------------------------------------------------------------------------
class RngStream:
    """RngStream(seed, stream_id) -- rng.hpp:30-86 (C restatement underneath)."""

    def __init__(self, seed: int, stream_id: int):
        self.seed = int(seed) & (2**64 - 1)
        self.stream_id = int(stream_id) & (2**64 - 1)
        self._h = _lib().orc_stream_new(self.seed, self.stream_id)

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.orc_stream_delete(self._h)
            self._h = None

    def next_u64(self, n=1):
        out = np.zeros(n, np.uint64)
        _lib().orc_stream_u64(self._h, n, out.ctypes.data)
        return out

    def uniform01(self, n=1):
        out = np.zeros(n)
        _lib().orc_stream_uniform(self._h, n, out.ctypes.data)
        return out

    def normals(self, n):
        out = np.zeros(n)
        if n:
            _lib().orc_stream_normals(self._h, n, out.ctypes.data)
        return out

    @property
    def draws(self) -> int:
        return int(_lib().orc_stream_draws(self._h))


def sample_indices(m: int, s: int, rng: RngStream, partitions: int = 1) -> np.ndarray:
    """Floyd sampling in sampled order (sampling.hpp:14-32); partitioned
    variant with child streams when partitions > 1 (sampling.hpp:41-66)."""
    out = np.zeros(max(int(s), 0), np.int64)
    rc = _lib().orc_stream_sample(rng._h, int(m), int(s), int(partitions), out.ctypes.data)
    if rc:
        raise ValueError(f"sample_indices: invalid arguments m={m} s={s} partitions={partitions}")
    return out


def gaussian_matrix(rows: int, cols: int, rng: RngStream) -> np.ndarray:
    """Column-major fill of i.i.d. normals (sampling.hpp:69-77)."""
    if rows < 1 or cols < 1:
        raise ValueError("gaussian_matrix: rows and cols must be >= 1")
    return rng.normals(rows * cols).reshape((rows, cols), order="F")


# --------------------------------------------------------------------------
# tensors (tensor.hpp), gathers (unfolding.hpp)
# --------------------------------------------------------------------------
def strides_of(dims):
    """g_k = prod_{j<k} n_j (tensor.hpp:32-38)."""
    g, out = 1, []
    for n in dims:
        out.append(g)
        g *= int(n)
    return out


def flat(x: np.ndarray) -> np.ndarray:
    """First-index-fastest flat data (tensor.hpp:17-20)."""
    return np.ravel(x, order="F")


def as_tensor(data: np.ndarray, dims) -> np.ndarray:
    return np.reshape(np.asarray(data), tuple(int(n) for n in dims), order="F")


def fiber_offsets(dims, mode: int, cols) -> np.ndarray:
    """unfolding.hpp:32-52: flat offsets (n_k x s) of the sampled mode-k
    fibres -- column j has base (c % g) + (c / g)*g*n_k and stride g."""
    nk = int(dims[mode])
    g = strides_of(dims)[mode]
    total = int(np.prod(dims)) // nk
    cols = np.asarray(cols, np.int64)
    if np.any(cols < 0) or np.any(cols >= total):
        raise IndexError("extract_fibers: column index out of range")
    base = (cols % g) + (cols // g) * g * nk
    return base[None, :] + np.arange(nk, dtype=np.int64)[:, None] * g


def extract_fibers(x: np.ndarray, mode: int, cols) -> np.ndarray:
    """unfolding.hpp:32-52.  Pure copy (bitwise equal to the unfolding)."""
    return flat(x)[fiber_offsets(x.shape, mode, cols)]


def group_fiber_offsets(dims, modes, cols) -> np.ndarray:
    """unfolding.hpp:57-111: flat offsets (n_S x w) of the sampled node
    fibres; rows follow the linear map over S ascending (first fastest),
    columns are decoded over the complement modes ascending."""
    d = len(dims)
    modes = sorted(int(m) for m in modes)
    if len(modes) >= d:
        raise ValueError("extract_group_fibers: mode set must be a proper subset")
    comp = [k for k in range(d) if k not in modes]
    st = strides_of(dims)
    cols = np.asarray(cols, np.int64)
    ncols_total = int(np.prod([dims[k] for k in comp]))
    if np.any(cols < 0) or np.any(cols >= ncols_total):
        raise IndexError("extract_group_fibers: column index out of range")
    base = np.zeros(len(cols), np.int64)
    c = cols.copy()
    for k in comp:
        base += (c % dims[k]) * st[k]
        c //= dims[k]
    nrows = int(np.prod([dims[k] for k in modes]))
    r = np.arange(nrows, dtype=np.int64)
    roff = np.zeros(nrows, np.int64)
    for k in modes:
        roff += (r % dims[k]) * st[k]
        r //= dims[k]
    return roff[:, None] + base[None, :]


def extract_group_fibers(x: np.ndarray, modes, cols) -> np.ndarray:
    """unfolding.hpp:57-111 (gather through group_fiber_offsets)."""
    return flat(x)[group_fiber_offsets(x.shape, modes, cols)]


def unfold(x: np.ndarray, mode: int) -> np.ndarray:
    return extract_fibers(x, mode, np.arange(x.size // x.shape[mode]))


def ttm(x: np.ndarray, u: np.ndarray, mode: int) -> np.ndarray:
    """tensor.hpp:255-289: contracts U (m x n_mode) with the mode fibers, as
    the reference does it on the flat first-index-fastest data: X viewed as
    g x n x post (g = prod n_<k); mode 0 is ONE GEMM (m x n)(n x post), the
    last mode one GEMM (g x n)(n x m), middle modes one GEMM per trailing
    block (post of them).  No copy of X when it is Fortran-contiguous."""
    dims = x.shape
    if u.shape[1] != dims[mode]:
        raise ValueError("ttm: matrix/mode extent mismatch")
    n = int(dims[mode])
    g = int(np.prod(dims[:mode], dtype=np.int64))
    post = int(np.prod(dims[mode + 1:], dtype=np.int64))
    m = u.shape[0]
    xf = np.ravel(x, order="F")
    if g == 1:
        out = xf.reshape(post, n) @ u.T           # C (post, m) == F (m, post)
    elif post == 1:
        out = u @ xf.reshape(n, g)                # C (m, g) == F (g, m)
    else:
        out = np.matmul(u, xf.reshape(post, n, g))  # C (post, m, g) == F (g, m, post)
    nd = list(dims)
    nd[mode] = m
    return np.reshape(np.ravel(out), nd, order="F")


def multi_ttm(x, factors):
    """tensor.hpp:293-306: sequential TTMs in list order."""
    seen = set()
    for mode, _ in factors:
        if mode in seen:
            raise ValueError(f"multi_ttm: duplicate mode {mode}")
        seen.add(mode)
    cur = x
    for mode, mat in factors:
        cur = ttm(cur, mat, mode)
    return cur


def frobenius_norm(x):
    return float(np.linalg.norm(flat(x)))


def rel_error(ref, approx):
    """tensor.hpp:241-249."""
    nrm = frobenius_norm(ref)
    if nrm == 0.0:
        raise ValueError("rel_error: reference tensor has zero norm")
    return float(np.linalg.norm(flat(ref) - flat(approx)) / nrm)


# --------------------------------------------------------------------------
# basis of a sketch (sketch.hpp:44-93)
# --------------------------------------------------------------------------
@dataclass
class RangeBasis:
    q: np.ndarray
    numerical_rank: int
    singular_values: np.ndarray = None


def pad_basis(q: np.ndarray, filled: int, rng: RngStream):
    """sketch.hpp:48-65: orthonormalize fresh Gaussian columns from the SAME
    stream against the accepted ones (two Gram-Schmidt rounds, accept when
    the norm exceeds 1e-8)."""
    n = q.shape[0]
    for j in range(filled, q.shape[1]):
        while True:
            v = rng.normals(n)
            for _ in range(2):
                if j > 0:
                    v = v - q[:, :j] @ (q[:, :j].T @ v)
            nrm = float(np.linalg.norm(v))
            if nrm > 1e-8:
                q[:, j] = v / nrm
                break


def range_basis_of_sketch(sketch: np.ndarray, rank: int, rng: RngStream) -> RangeBasis:
    """sketch.hpp:74-93: thin SVD of the sketch (LAPACK gesdd stands in for
    Eigen's BDCSVD), tol = max(rows, cols) * eps * sigma_1, numerical rank
    = #sigma > tol, keep min(nrank, rank) leading left singular vectors and
    pad the rest."""
    if rank < 1 or rank > sketch.shape[1]:
        raise ValueError("range_basis_of_sketch: rank out of range")
    u, sv, _ = np.linalg.svd(sketch, full_matrices=False)
    tol = max(sketch.shape) * np.finfo(float).eps * sv[0]
    nrank = int(np.sum(sv > tol))
    q_cols = min(nrank, rank)
    q = np.zeros((sketch.shape[0], rank))
    q[:, :q_cols] = u[:, :q_cols]
    if q_cols < rank:
        pad_basis(q, q_cols, rng)
    return RangeBasis(q=q, numerical_rank=q_cols, singular_values=sv)


def orthonormality_defect(q):
    """sketch.hpp:162-167."""
    return float(np.max(np.abs(q.T @ q - np.eye(q.shape[1]))))


# --------------------------------------------------------------------------
# Tucker (tucker.hpp)
# --------------------------------------------------------------------------
@dataclass
class ExecPolicy:
    """parallel.hpp:23-28."""
    workers: int = 1
    slice_mode: int | None = None
    index_partitions: int = 1
    emulate_serial_root: bool = False


@dataclass
class SubsampleReport:
    """tucker.hpp:129-134."""
    sample_counts: list = field(default_factory=list)
    achieved_ranks: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    sampled_columns: list = field(default_factory=list)  # oracle extra: for parity
    sketches: list = field(default_factory=list)  # oracle extra: Z per target


@dataclass
class TuckerDecomposition:
    core: np.ndarray
    factors: list


def reconstruct(t: TuckerDecomposition):
    """tucker.hpp:18-28."""
    out = t.core
    for k, u in enumerate(t.factors):
        out = ttm(out, u, k)
    return out


def core_from_factors(x, factors):
    """tucker.hpp:43-50: X x_0 U_0^T x_1 ... in mode order."""
    core = x
    for k, u in enumerate(factors):
        core = ttm(core, u.T, k)
    return core


def subsampled_mode_basis(x, mode, rank, p, samples, partitions, seed, report=None):
    """tucker.hpp:141-168: stream (seed, mode) -> sample -> gather -> Omega ->
    sketch -> basis."""
    rng = RngStream(seed, mode)
    available = x.size // x.shape[mode]
    cols = sample_indices(available, samples, rng, partitions)
    y = extract_fibers(x, mode, cols)
    omega = gaussian_matrix(y.shape[1], rank + p, rng)
    z = y @ omega
    basis = range_basis_of_sketch(z, rank, rng)
    return basis, cols, z


def _validate_ranks(dims, r, what):
    """tucker.hpp:31-40 (detail::validate_ranks)."""
    if len(r) != len(dims):
        raise ValueError(f"{what}: rank vector order mismatch")
    for k, (rk, nk) in enumerate(zip(r, dims)):
        if rk < 1 or rk > nk:
            raise ValueError(f"{what}: rank out of range in mode {k}")


def sub_r_hosvd(x, target, oversampling, samples, seed, exec_policy=None, report=None,
                threads=None):
    """tucker.hpp:177-242.  Mode jobs run concurrently when exec_policy is
    given (workers threads); the core goes through sliced_core then."""
    dims = x.shape
    d = len(dims)
    _validate_ranks(dims, target, "sub_r_hosvd")
    if len(samples) != len(target):
        raise ValueError("sub_r_hosvd: samples vector order mismatch")
    for k in range(d):
        if samples[k] < target[k] + oversampling:
            raise ValueError(f"sub_r_hosvd: samples below rank + oversampling in mode {k}")
        if samples[k] > x.size // dims[k]:
            raise ValueError(f"sub_r_hosvd: more samples than fibers in mode {k}")
    rep = report if report is not None else SubsampleReport()
    rep.sample_counts = list(samples)
    rep.achieved_ranks = [0] * d
    if oversampling < 4:
        rep.warnings.append("oversampling below the recommended minimum of 4")
    policy = exec_policy or ExecPolicy()

    def job(k):
        return subsampled_mode_basis(x, k, target[k], oversampling, samples[k],
                                     policy.index_partitions, seed)

    workers = max(1, policy.workers if exec_policy else 1)
    if workers > 1:
        with ThreadPoolExecutor(workers) as ex:
            results = list(ex.map(job, range(d)))
    else:
        results = [job(k) for k in range(d)]
    factors = []
    for k, (basis, cols, z) in enumerate(results):
        rep.achieved_ranks[k] = basis.numerical_rank
        rep.sampled_columns.append(cols)
        rep.sketches.append(z)
        if basis.numerical_rank < target[k]:
            rep.warnings.append(f"mode {k}: sketch revealed rank {basis.numerical_rank} < target "
                                f"{target[k]}; basis padded")
        factors.append(basis.q)
    if exec_policy is not None:
        core = sliced_core(x, factors, policy)
    else:
        core = core_from_factors(x, factors)
    return TuckerDecomposition(core=core, factors=factors)


def sampling_fractions(dims, samples):
    """tucker.hpp:245-251."""
    n = int(np.prod(dims))
    return [samples[k] / (n // dims[k]) for k in range(len(dims))]


def pick_slice_mode(dims, workers):
    """parallel.hpp:331-348."""
    best, best_score = -1, None
    for k, nk in enumerate(dims):
        if nk < workers:
            continue
        rem = nk % workers
        score = 0 if rem == 0 else workers - rem
        if best_score is None or score < best_score:
            best, best_score = k, score
    if best < 0:
        raise ValueError(f"pick_slice_mode: no mode can host {workers} slices")
    return best


def sliced_core(x, factors, policy: ExecPolicy):
    """parallel.hpp:355-445: `workers` jobs reduce contiguous slabs of slices
    along the slice mode (bounds of :400-404), ONE SLICE AT A TIME over every
    other mode in mode order (reduce_slice, :386-395) -- so the bits do not
    depend on the worker count --, run concurrently on a thread pool
    (run_independent_jobs, :87-129); the coordinator gathers the reduced
    slabs and applies the final TTM along the slice mode (:424-441)."""
    dims = x.shape
    d = len(dims)
    if len(factors) != d:
        raise ValueError("sliced_core: need one factor per mode")
    sm = policy.slice_mode if policy.slice_mode is not None else pick_slice_mode(dims, policy.workers)
    if not 0 <= sm < d:
        raise ValueError("sliced_core: slice mode out of range")
    if policy.workers > dims[sm]:
        raise ValueError("sliced_core: more workers than slices along the slicing mode")
    nworkers = min(policy.workers, dims[sm])
    n = dims[sm]
    rdims = [n if k == sm else factors[k].shape[1] for k in range(d)]
    reduced = np.zeros(rdims, order="F")
    idx = [slice(None)] * d

    def reduce_slab(w):
        lo = w * (n // nworkers) + min(w, n % nworkers)
        hi = lo + n // nworkers + (1 if w < n % nworkers else 0)
        for i in range(lo, hi):
            j = list(idx)
            j[sm] = slice(i, i + 1)
            sl = np.asfortranarray(x[tuple(j)])  # copy of slice i (parallel.hpp:387-389)
            for k in range(d):
                if k != sm:
                    sl = ttm(sl, factors[k].T, k)
            reduced[tuple(j)] = sl

    if nworkers > 1:
        with ThreadPoolExecutor(nworkers) as ex:
            list(ex.map(reduce_slab, range(nworkers)))
    else:
        reduce_slab(0)
    return ttm(reduced, factors[sm].T, sm)


def sliced_core_streamed(read_slab, dims, factors, slab=128):
    """sliced_core's slab algebra (parallel.hpp:355-445) with the LAST mode as
    the slice mode, for tensors that do not fit the host: ``read_slab(lo, hi)``
    returns X[..., lo:hi) (an nd-array of dims[:-1] + [hi - lo]); each slab is
    reduced over modes 0..d-2 in mode order, the reduced slabs are gathered
    and the final TTM along mode d-1 is applied."""
    d = len(dims)
    n = int(dims[-1])
    reduced = np.zeros([f.shape[1] for f in factors[:-1]] + [n], order="F")
    for lo in range(0, n, slab):
        hi = min(n, lo + slab)
        sl = read_slab(lo, hi)
        for k in range(d - 1):
            sl = ttm(sl, factors[k].T, k)
        reduced[..., lo:hi] = sl
    return ttm(reduced, factors[-1].T, d - 1)


def rel_error_streamed(read_slab, dims, core, factors, slab=128):
    """rel_error(x, reconstruct(t)) (tensor.hpp:241-249, tucker.hpp:18-28)
    slab by slab along the last mode: X-hat[..., lo:hi) =
    (G x_0 U_0 ... x_{d-2} U_{d-2}) x_{d-1} U_{d-1}[lo:hi, :]."""
    d = len(dims)
    part = core
    for k in range(d - 1):
        part = ttm(part, factors[k], k)
    num = den = 0.0
    n = int(dims[-1])
    for lo in range(0, n, slab):
        hi = min(n, lo + slab)
        xs = flat(read_slab(lo, hi))
        xh = flat(ttm(part, factors[-1][lo:hi, :], d - 1))
        num += float(np.dot(xs - xh, xs - xh))
        den += float(np.dot(xs, xs))
    if den == 0.0:
        raise ValueError("rel_error: reference tensor has zero norm")
    return math.sqrt(num) / math.sqrt(den)


# --------------------------------------------------------------------------
# dimension tree (dimension_tree.hpp) and H-Tucker (htucker.hpp)
# --------------------------------------------------------------------------
@dataclass
class TreeNode:
    modes: list
    left: int = -1
    right: int = -1
    parent: int = -1
    level: int = 0

    def is_leaf(self):
        return self.left < 0


class DimensionTree:
    """dimension_tree.hpp:27-152."""

    def __init__(self, nodes):
        self.nodes = nodes
        self._validate()

    @staticmethod
    def balanced(order):
        """dimension_tree.hpp:36-64: recursive halving, BFS/heap ids."""
        if order < 2:
            raise ValueError("DimensionTree: order must be >= 2")
        nodes = [TreeNode(list(range(order)))]
        queue = [0]
        while queue:
            i = queue.pop(0)
            modes = nodes[i].modes
            if len(modes) == 1:
                continue
            half = (len(modes) + 1) // 2
            lvl = nodes[i].level + 1
            li = len(nodes)
            nodes.append(TreeNode(modes[:half], parent=i, level=lvl))
            ri = len(nodes)
            nodes.append(TreeNode(modes[half:], parent=i, level=lvl))
            nodes[i].left, nodes[i].right = li, ri
            queue += [li, ri]
        return DimensionTree(nodes)

    def _validate(self):
        d = len(self.nodes[0].modes)
        if d < 2:
            raise ValueError("DimensionTree: order must be >= 2")
        if self.nodes[0].modes != list(range(d)):
            raise ValueError("DimensionTree: root must hold modes 0..d-1")
        leaves = 0
        for i, n in enumerate(self.nodes):
            if (n.left < 0) != (n.right < 0):
                raise ValueError("DimensionTree: node must have zero or two children")
            if n.is_leaf():
                if len(n.modes) != 1:
                    raise ValueError("DimensionTree: leaves must hold a single mode")
                leaves += 1
                continue
            lm, rm = self.nodes[n.left].modes, self.nodes[n.right].modes
            if self.nodes[n.left].parent != i or self.nodes[n.right].parent != i:
                raise ValueError("DimensionTree: child parent link mismatch")
            if lm[-1] >= rm[0] or lm + rm != n.modes:
                raise ValueError("DimensionTree: children do not partition the node")
        if leaves != d:
            raise ValueError("DimensionTree: expected one leaf per mode")

    @property
    def num_nodes(self):
        return len(self.nodes)

    @property
    def order(self):
        return len(self.nodes[0].modes)

    def node(self, i):
        return self.nodes[i]

    def depth(self):
        return max(n.level for n in self.nodes)

    def leaves(self):
        return [i for i, n in enumerate(self.nodes) if n.is_leaf()]

    def internal_nodes_bottom_up(self):
        """dimension_tree.hpp:86-92."""
        out = []
        for lvl in range(self.depth(), 0, -1):
            out += [i for i in range(1, self.num_nodes)
                    if not self.nodes[i].is_leaf() and self.nodes[i].level == lvl]
        return out

    def node_rows(self, i, dims):
        return int(np.prod([dims[m] for m in self.nodes[i].modes]))

    def node_cols(self, i, dims):
        return int(np.prod(dims)) // self.node_rows(i, dims)


def uniform_node_ranks(tree, rank):
    """dimension_tree.hpp:159-163."""
    out = [rank] * tree.num_nodes
    out[0] = 1
    return out


def node_sample_counts(tree, dims, alpha):
    """dimension_tree.hpp:174-183."""
    out = [1] * tree.num_nodes
    for i in range(1, tree.num_nodes):
        out[i] = min(int(math.ceil(alpha * tree.node_rows(i, dims))), tree.node_cols(i, dims))
    return out


@dataclass
class HTuckerDecomposition:
    tree: DimensionTree
    leaf_factors: list
    transfers: list


@dataclass
class HtSubsampleReport:
    sample_counts: list = field(default_factory=list)
    achieved_ranks: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    sampled_columns: dict = field(default_factory=dict)
    sketches: dict = field(default_factory=dict)
    bases: dict = field(default_factory=dict)


def transfer_tensor(u_node, u_left, u_right):
    """htucker.hpp:44-63: B(i,j,k) = sum_{a,b} U_l(a,j) U_S(a+b*n_l, i) U_r(b,k)."""
    nl, nr = u_left.shape[0], u_right.shape[0]
    if u_node.shape[0] != nl * nr:
        raise ValueError("transfer_tensor: node rows must equal product of child rows")
    rs = u_node.shape[1]
    us = u_node.reshape((nl, nr, rs), order="F")
    return np.einsum("aj,abi,bk->ijk", u_left, us, u_right, optimize=True)


def root_transfer(x, u_left, u_right):
    """htucker.hpp:67-85: B(0,j,k) = (U_l^T M U_r)(j,k), M = X as n_l x n_r."""
    nl, nr = u_left.shape[0], u_right.shape[0]
    if nl * nr != x.size:
        raise ValueError("root_transfer: child rows do not factor the tensor size")
    m = flat(x).reshape((nl, nr), order="F")
    b0 = (u_left.T @ m) @ u_right
    return b0[None, :, :]


def expand_node_basis(u_left, u_right, b):
    """htucker.hpp:88-105."""
    rs = b.shape[0]
    nl, nr = u_left.shape[0], u_right.shape[0]
    u = np.zeros((nl * nr, rs))
    for i in range(rs):
        ui = u_left @ b[i] @ u_right.T
        u[:, i] = ui.reshape(-1, order="F")
    return u


def _validate_node_ranks(tree, dims, ranks, what):
    """htucker.hpp:109-121."""
    if len(ranks) != tree.num_nodes:
        raise ValueError(f"{what}: rank vector must have one entry per node")
    if ranks[0] != 1:
        raise ValueError(f"{what}: root rank must be 1")
    for i in range(1, tree.num_nodes):
        mx = min(tree.node_rows(i, dims), tree.node_cols(i, dims))
        if ranks[i] < 1 or ranks[i] > mx:
            raise ValueError(f"{what}: rank out of range at node {i}")


def node_basis(x, tree, node_id, rank, p, w, partitions, seed):
    """htucker.hpp:263-287: one basis job, stream bound to the node id."""
    n = tree.node(node_id)
    rng = RngStream(seed, node_id)
    cols_total = tree.node_cols(node_id, x.shape)
    picked = sample_indices(cols_total, w, rng, partitions)
    y = extract_fibers(x, n.modes[0], picked) if n.is_leaf() else \
        extract_group_fibers(x, n.modes, picked)
    omega = gaussian_matrix(y.shape[1], rank + p, rng)
    z = y @ omega
    return range_basis_of_sketch(z, rank, rng), picked, z


def sub_r_rtl_ht(x, tree, ranks, samples, oversampling, seed, exec_policy=None, report=None):
    """htucker.hpp:210-341."""
    dims = x.shape
    if tree.order != len(dims):
        raise ValueError("sub_r_rtl_ht: tree and tensor order mismatch")
    _validate_node_ranks(tree, dims, ranks, "sub_r_rtl_ht")
    if len(samples) != tree.num_nodes:
        raise ValueError("sub_r_rtl_ht: samples vector must have one entry per node")
    for i in range(1, tree.num_nodes):
        if samples[i] < ranks[i] + oversampling:
            raise ValueError(f"sub_r_rtl_ht: samples below rank + oversampling at node {i}")
        if samples[i] > tree.node_cols(i, dims):
            raise ValueError(f"sub_r_rtl_ht: more samples than fibers at node {i}")
    rep = report if report is not None else HtSubsampleReport()
    rep.sample_counts = list(samples)
    rep.achieved_ranks = [0] * tree.num_nodes
    rep.achieved_ranks[0] = 1
    if oversampling < 4:
        rep.warnings.append("oversampling below the recommended minimum of 4")
    policy = exec_policy or ExecPolicy()

    def job(i):
        return node_basis(x, tree, i, ranks[i], oversampling, samples[i],
                          policy.index_partitions, seed)

    workers = max(1, policy.workers if exec_policy else 1)
    ids = list(range(1, tree.num_nodes))
    if workers > 1:
        with ThreadPoolExecutor(workers) as ex:
            res = dict(zip(ids, ex.map(job, ids)))
    else:
        res = {i: job(i) for i in ids}
    bases = {i: res[i][0] for i in ids}
    for i in ids:
        rep.sampled_columns[i] = res[i][1]
        rep.sketches[i] = res[i][2]
        rep.bases[i] = bases[i].q
    transfers = [None] * tree.num_nodes
    for i in tree.internal_nodes_bottom_up():
        n = tree.node(i)
        transfers[i] = transfer_tensor(bases[i].q, bases[n.left].q, bases[n.right].q)
    root = tree.node(0)
    transfers[0] = root_transfer(x, bases[root.left].q, bases[root.right].q)
    for i in ids:
        rep.achieved_ranks[i] = bases[i].numerical_rank
        if bases[i].numerical_rank < ranks[i]:
            rep.warnings.append(f"node {i}: sketch revealed rank {bases[i].numerical_rank} "
                                f"< target; basis padded")
    leaf = [None] * tree.order
    for i in tree.leaves():
        leaf[tree.node(i).modes[0]] = bases[i].q
    return HTuckerDecomposition(tree=tree, leaf_factors=leaf, transfers=transfers)


def ht_reconstruct(h: HTuckerDecomposition):
    """htucker.hpp:346-378."""
    tree = h.tree
    bases = {}
    for i in tree.leaves():
        bases[i] = h.leaf_factors[tree.node(i).modes[0]]
    for i in tree.internal_nodes_bottom_up():
        n = tree.node(i)
        bases[i] = expand_node_basis(bases[n.left], bases[n.right], h.transfers[i])
    root = tree.node(0)
    ul, ur = bases[root.left], bases[root.right]
    fl = ul @ (h.transfers[0][0] @ ur.T)
    dims = [h.leaf_factors[m].shape[0] for m in range(tree.order)]
    return as_tensor(fl.reshape(-1, order="F"), dims)


def ht_storage_count(h):
    """htucker.hpp:382-388."""
    return sum(u.size for u in h.leaf_factors) + sum(b.size for b in h.transfers if b is not None)
