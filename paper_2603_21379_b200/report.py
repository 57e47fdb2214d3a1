"""Experiment / report layer around the B200 path.

Mirrors the reference's experiment driver for the two hot-path methods
(experiment.hpp:12-131, experiment.cpp:155-497): seeded repetitions of one
decomposition, CSV rows with the reference's fixed header, JSON five-number
summaries, sampling-fraction lines and the worker scaling table -- so tools
that consume the reference's CSV/JSON read these unchanged.

Differences, by design:
  * only ``sub-r-hosvd`` and ``sub-r-rtl-ht`` run (the other methods are the
    reference's deterministic baselines, outside the hot path);
  * the decomposition and ``rel_error(x, reconstruct(t))`` run on the GPU
    (the error is streamed, X-hat is never materialised);
  * ``stage_json`` holds the engine's device-measured stage times, one record
    per non-zero stage with worker 0 (the GPU), same stage names;
  * the planted generators build the same model family on the GPU (Gaussian
    core / transfers, Gaussian-QR factors, seeded by ``base_seed``) but not
    the reference generator's exact bits; the ``file`` generator reads the
    SRTT container and is exact.
"""
from __future__ import annotations

import io
import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import srtt as _s

CSV_HEADER = "seed,method,d,shape,rank,samples,p,workers,rel_error,total_s,stage_json"
METHODS = ("t-hosvd", "st-hosvd", "r-hosvd", "sub-r-hosvd", "rtl-ht", "sub-r-rtl-ht")
HOT_PATH_METHODS = ("sub-r-hosvd", "sub-r-rtl-ht")
GENERATORS = ("tucker-planted", "htucker-planted", "file")


class CheckFailure(RuntimeError):
    """experiment.hpp:74-77."""


def method_is_randomized(m):
    return m in ("r-hosvd", "sub-r-hosvd", "sub-r-rtl-ht")


def method_is_hierarchical(m):
    return m in ("rtl-ht", "sub-r-rtl-ht")


def method_needs_samples(m):
    return m in ("sub-r-hosvd", "sub-r-rtl-ht")


@dataclass
class ExperimentSpec:
    """experiment.hpp:29-48 (hot-path subset)."""
    generator: str = "tucker-planted"
    shape: list = field(default_factory=list)
    input_path: str = ""
    rank: int = 5
    method: str = "sub-r-hosvd"
    samples: int | None = None
    alpha: float | None = None
    oversampling: int = 4
    base_seed: int = 1
    runs: int = 1
    workers: int = 1
    use_exec: bool = False
    strict: bool = False
    timings: bool = True


@dataclass
class SeedResult:
    seed: int = 0
    rel_error: float = 0.0
    total_seconds: float = 0.0
    timings: list = field(default_factory=list)     # [{"stage", "worker", "seconds"}]
    achieved_ranks: list = field(default_factory=list)
    warnings: list = field(default_factory=list)


@dataclass
class SamplingFractionLine:
    target: str
    samples: int
    columns: int
    fraction: float
    percent_text: str


@dataclass
class RunReport:
    spec: ExperimentSpec
    shape: list
    ranks: list
    sample_counts: list
    rows: list = field(default_factory=list)
    fractions: list = field(default_factory=list)
    environment: str = ""


# ---------------------------------------------------------------------------
# formatting helpers (experiment.cpp:60-120, 236-264)
# ---------------------------------------------------------------------------
def join_x(values):
    return "x".join(str(int(v)) for v in values)


def csv_quote(s):
    return '"' + s.replace('"', '""') + '"'


def parse_csv_line(line):
    """experiment.cpp:385-411: fields with double-quoted, doubled quotes."""
    fields, cur, quoted, i = [], [], False, 0
    while i < len(line):
        c = line[i]
        if quoted:
            if c == '"':
                if i + 1 < len(line) and line[i + 1] == '"':
                    cur.append('"')
                    i += 1
                else:
                    quoted = False
            else:
                cur.append(c)
        elif c == '"':
            quoted = True
        elif c == ",":
            fields.append("".join(cur))
            cur = []
        else:
            cur.append(c)
        i += 1
    fields.append("".join(cur))
    return fields


def median(values):
    if not values:
        raise _s.InvalidArgument("median: empty sample")
    v = sorted(values)
    n = len(v)
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def _quantile(values, q):
    v = sorted(values)
    if len(v) == 1:
        return v[0]
    pos = q * (len(v) - 1)
    lo, hi = math.floor(pos), math.ceil(pos)
    frac = pos - math.floor(pos)
    return v[lo] * (1.0 - frac) + v[hi] * frac


def five_number_summary(values):
    return {"max": _quantile(values, 1.0), "median": _quantile(values, 0.5), "min": _quantile(values, 0.0),
            "q1": _quantile(values, 0.25), "q3": _quantile(values, 0.75)}


def format_percent_ceil(fraction):
    """experiment.cpp:255-277: percentage, mantissa rounded UP to one digit."""
    pct = fraction * 100.0
    if not pct > 0.0:
        return "0%"
    if pct >= 100.0:
        return "100%"
    e = int(math.floor(math.log10(pct)))
    digit = int(math.ceil(pct / 10.0 ** e - 1e-9))
    if digit == 10:
        digit, e = 1, e + 1
    if e >= 0:
        return str(digit * 10 ** e) + "%"
    return "0." + "0" * (-e - 1) + str(digit) + "%"


def environment_fingerprint():
    import platform

    dev = ""
    try:
        import torch

        if torch.cuda.is_available():
            dev = torch.cuda.get_device_name(0)
    except Exception:  # pragma: no cover
        pass
    return f"cores={os.cpu_count()} device={dev or 'none'} engine=libsrtt_b200 python={platform.python_version()}"


def _dumps(obj, indent=None):
    # nlohmann::json orders object keys; separators match its dump()
    if indent is None:
        return json.dumps(obj, sort_keys=True, separators=(",", ":"))
    return json.dumps(obj, sort_keys=True, indent=indent)


def factor_stage_seconds(row):
    """experiment.cpp:122-127."""
    tot = {}
    for r in row.timings:
        tot[r["stage"]] = tot.get(r["stage"], 0.0) + r["seconds"]
    if tot.get("factor_wall", 0.0) > 0.0:
        return tot["factor_wall"]
    return sum(tot.get(s, 0.0) for s in ("sampling", "extract", "sketch", "svd"))


# ---------------------------------------------------------------------------
# problems and runs (experiment.cpp:155-250, 279-365)
# ---------------------------------------------------------------------------
@dataclass
class _Problem:
    x: object          # flat CUDA float64 tensor
    dims: list
    tree: object
    ranks: list
    samples: list


def _planted_tucker(dims, rank, seed):
    import torch

    g = torch.Generator(device="cuda").manual_seed(int(seed))
    core = torch.randn([rank] * len(dims), dtype=torch.float64, device="cuda", generator=g)
    factors = [torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device="cuda", generator=g))[0]
               for n in dims]
    t = _s.TuckerDecomposition(core.permute(*reversed(range(len(dims)))).contiguous().reshape(-1),
                               [u.t().contiguous().reshape(-1) for u in factors])
    return _s.reconstruct(t, dims=list(dims), device_out=True)


def _planted_htucker(dims, tree, ranks, seed):
    import torch

    g = torch.Generator(device="cuda").manual_seed(int(seed))
    d = len(dims)
    leaf = [None] * d
    trs = [None] * tree.num_nodes
    for i in tree.leaves():
        m = tree.node(i).modes[0]
        u = torch.linalg.qr(torch.randn(dims[m], ranks[i], dtype=torch.float64, device="cuda", generator=g))[0]
        leaf[m] = u.t().contiguous().reshape(-1)           # column-major n x r
    for i in range(tree.num_nodes):
        nd = tree.node(i)
        if not nd.is_leaf():
            rs = 1 if i == 0 else ranks[i]
            trs[i] = torch.randn(rs * ranks[nd.left] * ranks[nd.right], dtype=torch.float64, device="cuda",
                                 generator=g)
    return _s.ht_reconstruct(_s.HTuckerDecomposition(tree, leaf, trs), dims=list(dims), device_out=True)


def resolve_problem(spec: ExperimentSpec, handle=None) -> _Problem:
    if spec.method not in METHODS:
        raise _s.InvalidArgument("unknown method: " + spec.method)
    if spec.method not in HOT_PATH_METHODS:
        raise _s.InvalidArgument(f"method {spec.method} is a reference baseline outside the B200 hot path")
    if spec.generator not in GENERATORS:
        raise _s.InvalidArgument("unknown generator: " + spec.generator)
    hier = method_is_hierarchical(spec.method)
    if spec.generator == "file":
        x = _s.read_tensor(spec.input_path, device=True, handle=handle)
        dims, _ = _s.tensor_file_info(spec.input_path)
    else:
        dims = [int(n) for n in spec.shape]
        if spec.generator == "tucker-planted":
            x = _planted_tucker(dims, spec.rank, spec.base_seed)
        else:
            t = _s.DimensionTree.balanced(len(dims))
            x = _planted_htucker(dims, t, _s.uniform_node_ranks(t, spec.rank), spec.base_seed)
    d = len(dims)
    N = int(np.prod(dims))
    if hier:
        tree = _s.DimensionTree.balanced(d)
        ranks = _s.uniform_node_ranks(tree, spec.rank)
        if spec.alpha is not None:
            samples = _s.node_sample_counts(tree, dims, spec.alpha)
        elif spec.samples is not None:
            samples = [1] + [min(spec.samples, tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
        else:
            raise _s.InvalidArgument("sub-r-rtl-ht requires --samples or --alpha")
    else:
        tree = None
        ranks = [spec.rank] * d
        samples = []
        for k in range(d):
            if spec.samples is not None:
                s = spec.samples
            elif spec.alpha is not None:
                s = int(math.ceil(spec.alpha * dims[k]))
            else:
                raise _s.InvalidArgument("SketchConfig: neither samples nor alpha is set")
            samples.append(min(s, N // dims[k]))
    return _Problem(x, dims, tree, ranks, samples)


_STAGE_KEYS = _s.STAGES


def run_one(spec: ExperimentSpec, problem: _Problem, seed: int, handle=None) -> SeedResult:
    import torch

    h = handle or _s.default_handle()
    row = SeedResult(seed=int(seed))
    rep = _s.SubsampleReport()
    ex = _s.ExecPolicy(workers=spec.workers) if spec.use_exec else None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if spec.method == "sub-r-hosvd":
        t = _s.sub_r_hosvd(problem.x, problem.ranks, spec.oversampling, problem.samples, seed, ex, rep,
                           dims=problem.dims, handle=h, device_out=True)
        torch.cuda.synchronize()
        row.total_seconds = time.perf_counter() - t0
        row.rel_error = _s.tucker_rel_error(problem.x, t, dims=problem.dims, handle=h)
    else:
        t = _s.sub_r_rtl_ht(problem.x, problem.tree, problem.ranks, problem.samples, spec.oversampling, seed, ex,
                            rep, dims=problem.dims, handle=h, device_out=True)
        torch.cuda.synchronize()
        row.total_seconds = time.perf_counter() - t0
        row.rel_error = _s.ht_rel_error(problem.x, t, dims=problem.dims, handle=h)
    row.timings = [{"seconds": float(v), "stage": k, "worker": 0} for k, v in rep.timings.items() if v > 0.0]
    row.achieved_ranks = list(rep.achieved_ranks)
    row.warnings = list(rep.warnings)
    return row


def run_experiment(spec: ExperimentSpec, handle=None) -> RunReport:
    """experiment.cpp:279-365."""
    if spec.runs < 1:
        raise _s.InvalidArgument("run_experiment: runs must be >= 1")
    if method_needs_samples(spec.method) and spec.samples is None and spec.alpha is None:
        raise _s.InvalidArgument("run_experiment: subsampled methods need --samples or --alpha")
    pb = resolve_problem(spec, handle)
    rep = RunReport(spec=spec, shape=list(pb.dims), ranks=list(pb.ranks), sample_counts=list(pb.samples),
                    environment=environment_fingerprint())
    if method_is_hierarchical(spec.method):
        for i in range(1, pb.tree.num_nodes):
            cols = pb.tree.node_cols(i, pb.dims)
            s = pb.samples[i]
            modes = "{" + ",".join(str(m) for m in pb.tree.node(i).modes) + "}"
            rep.fractions.append(SamplingFractionLine(f"node {i} {modes}", s, cols, s / cols,
                                                      format_percent_ceil(s / cols)))
    else:
        N = int(np.prod(pb.dims))
        for k, n in enumerate(pb.dims):
            cols = N // n
            s = pb.samples[k]
            rep.fractions.append(SamplingFractionLine(f"mode {k}", s, cols, s / cols, format_percent_ceil(s / cols)))
    for i in range(spec.runs):
        row = run_one(spec, pb, spec.base_seed + i, handle)
        if spec.strict:
            for k, a in enumerate(row.achieved_ranks):
                if 0 < a < pb.ranks[k]:
                    raise CheckFailure(f"numerical rank shortfall at target {k} (achieved {a} of {pb.ranks[k]})")
        if not spec.timings:
            row.total_seconds = 0.0
            row.timings = []
        rep.rows.append(row)
    return rep


def write_csv(report: RunReport, f):
    """experiment.cpp:367-383 (CSV_HEADER schema)."""
    workers = report.spec.workers if report.spec.use_exec else 1
    f.write(CSV_HEADER + "\n")
    for row in report.rows:
        p = str(report.spec.oversampling) if method_is_randomized(report.spec.method) else ""
        f.write(f"{row.seed},{report.spec.method},{len(report.shape)},{join_x(report.shape)},"
                f"{join_x(report.ranks)},{join_x(report.sample_counts)},{p},{workers},"
                f"{row.rel_error:.17g},{row.total_seconds:.6f},{csv_quote(_dumps(row.timings))}\n")


def report_to_json(report: RunReport):
    """experiment.cpp:415-463."""
    errors = [r.rel_error for r in report.rows]
    times = [r.total_seconds for r in report.rows]
    factor = [factor_stage_seconds(r) for r in report.rows]
    return {
        "method": report.spec.method, "generator": report.spec.generator, "shape": join_x(report.shape),
        "order": len(report.shape), "rank": join_x(report.ranks), "samples": join_x(report.sample_counts),
        "oversampling": report.spec.oversampling,
        "workers": report.spec.workers if report.spec.use_exec else 1, "runs": report.spec.runs,
        "base_seed": report.spec.base_seed, "errors": five_number_summary(errors),
        "total_seconds": five_number_summary(times), "factor_stage_seconds": five_number_summary(factor),
        "environment": report.environment,
        "sampling_fractions": [{"columns": ln.columns, "fraction": ln.fraction, "percent": ln.percent_text,
                                "samples": ln.samples, "target": ln.target} for ln in report.fractions],
        "warnings": [w for r in report.rows for w in r.warnings],
    }


def write_json_summary(report: RunReport, f):
    f.write(_dumps(report_to_json(report), indent=2) + "\n")


def write_scaling_json(runs, f):
    """experiment.cpp:470-497: runs = [(workers, RunReport), ...]."""
    table, base_total, base_factor = [], 0.0, 0.0
    for i, (w, rep) in enumerate(runs):
        mt = median([r.total_seconds for r in rep.rows])
        mf = median([factor_stage_seconds(r) for r in rep.rows])
        if i == 0:
            base_total, base_factor = mt, mf
        table.append({"median_factor_stage_s": mf, "median_total_s": mt,
                      "speedup_factor_stage": base_factor / mf if mf > 0 else 0.0,
                      "speedup_total": base_total / mt if mt > 0 else 0.0, "workers": w})
    f.write(_dumps({"environment": environment_fingerprint(), "scaling": table}, indent=2) + "\n")


def csv_string(report):
    buf = io.StringIO()
    write_csv(report, buf)
    return buf.getvalue()
