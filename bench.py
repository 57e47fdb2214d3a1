#!/usr/bin/env python
"""Headline benchmark: fp64 tensor entries decomposed per second.

One "step" = one full Sub-R-HOSVD (or Sub-R-RtL-HT for c4) of the config's
synthetic tensor: host index sampling + K1 sketch + K2 basis + K3 core pass,
X resident in HBM (``value``); ``e2e`` times the same call through the C-ABI
with X in pinned HOST memory (H2D of X and D2H of the factors/core inside
the timed region).  Default workload: BASELINE.json configs[4] (C5, order-3
Tucker 2048^3, 8.6e9 entries, 68.7 GB: the largest configuration that fits
one 180 GB B200; inputs far larger than L2, so no flush is needed).
``--config`` selects c1-c5 (or the added sketch-heavy variants).

``--impl reference`` times the CPU restatement of the reference (oracle/,
numpy + OpenBLAS on the host cores under the reference's own policies; the
reference itself needs Eigen, absent in this image) on the same config and
the same X bits (a bounded leading slab for c5).

Multi-GPU (torchrun, ``--mode auto``): ONE global tensor per step over the
ranks (strong scaling) through the fused NCCL C-ABI: slab-sharded for c5
(each rank holds its last-mode slab), replicated with modes / nodes assigned
to ranks for the configs that fit per GPU. ``--mode replicas`` runs
independent decompositions per rank instead (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tensor entries decomposed/sec (fp64)"
UNIT = "entries/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while running."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no_samples"], "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        sm = [num(s[0]) for s in self.samples if num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
# one decomposition through the product API
# ---------------------------------------------------------------------------
_OUT = {}


def _run_product(P, cfg, x, dims, seed, handle, device_out=True, report=None):
    if cfg.kind == "tucker":
        out = None
        if device_out:  # reuse the caller-side output buffers across steps
            out = _OUT.get(cfg.name)
            if out is None:
                import torch

                dev = x.device
                out = _OUT.setdefault(cfg.name, (torch.empty(cfg.rank ** cfg.order, dtype=torch.float64, device=dev),
                                                 [torch.empty(n * cfg.rank, dtype=torch.float64, device=dev)
                                                  for n in dims]))
        return P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), seed, report=report, dims=dims,
                             handle=handle, device_out=device_out, out=out)
    tree = P.DimensionTree.balanced(cfg.order)
    ranks = P.uniform_node_ranks(tree, cfg.rank)
    samples = cfg.node_samples(tree, dims)
    return P.sub_r_rtl_ht(x, tree, ranks, samples, cfg.p, seed, report=report, dims=dims, handle=handle,
                          device_out=device_out)


def _run_oracle(O, cfg, X, seed, policy=None):
    if cfg.kind == "tucker":
        return O.sub_r_hosvd(X, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), seed, exec_policy=policy)
    tree = O.DimensionTree.balanced(cfg.order)
    ranks = O.uniform_node_ranks(tree, cfg.rank)
    samples = cfg.node_samples(tree, X.shape)
    return O.sub_r_rtl_ht(X, tree, ranks, samples, cfg.p, seed, exec_policy=policy)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# The two ways the reference runs on a multicore host (srtt_main.cpp:70,
# 102-104; experiment.cpp:217-218):
#   "exec":   ExecPolicy{workers = nproc}: mode / node jobs on a thread pool
#             and the slice-by-slice sliced_core (parallel.hpp:87-147,
#             205-277, 355-445), one BLAS thread per worker (the reference's
#             Eigen GEMMs are single-threaded);
#   "serial": no policy (--workers 0): jobs in order, core_from_factors,
#             here with the BLAS threaded over all host cores.
# The CPU baseline reports the FASTER of the two on the box.
def _time_cpu_policies(O, cfg, X, seed, budget_s):
    from threadpoolctl import threadpool_limits

    ncpu = os.cpu_count() or 1
    out = {}
    for name in ("exec", "serial"):
        pol = O.ExecPolicy(workers=ncpu) if name == "exec" else None
        lim = 1 if name == "exec" else None

        def once():
            t0 = time.perf_counter()
            if lim:
                with threadpool_limits(lim):
                    _run_oracle(O, cfg, X, seed, pol)
            else:
                _run_oracle(O, cfg, X, seed, pol)
            return time.perf_counter() - t0

        first = once()  # warm-up (page faults, thread pools)
        times = []
        t_start = time.perf_counter()
        while len(times) < 5 and (not times or time.perf_counter() - t_start + first < budget_s / 2):
            times.append(once())
        out[name] = statistics.median(times), len(times)
    return out


def _host_tensor(cfg, dims=None):
    """The config's tensor bits as the GPU arm sees them: generated by
    synth's torch generator on cuda:0 (seed 0) and copied to the host (only
    the leading `dims` slab when given); numpy generation (different bits)
    only when no GPU is visible."""
    from paper_2603_21379_b200 import synth

    try:
        import torch

        if torch.cuda.is_available():
            xd = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
            n = int(np.prod(dims)) if dims is not None else cfg.entries
            xh = xd[:n].cpu().numpy()
            del xd
            torch.cuda.empty_cache()
            return xh, "the GPU arm's X bits (synth torch generator, seed 0)"
    except Exception:  # pragma: no cover - no usable GPU
        pass
    return synth.make_tensor(cfg, seed=0, backend="numpy", dims=dims), "numpy-generated X (no GPU visible)"


# CPU samples of tensors larger than CPU_SAMPLE_BYTES are cut to a leading
# slab of about CPU_SLAB_BYTES along the last mode (a contiguous byte range of
# X; same ranks, oversampling and fibre counts) -- C5 only
CPU_SAMPLE_BYTES = 16e9
CPU_SLAB_BYTES = 2.2e9


def cpu_sample(cfg, x_host_flat):
    """(config, flat data, description) of the bounded CPU sample of `cfg`."""
    import dataclasses

    if cfg.entries * 8 <= CPU_SAMPLE_BYTES:
        return cfg, x_host_flat, f"full {cfg.name} decomposition (N={cfg.entries})"
    inner = cfg.entries // cfg.dims[-1]
    last = max(cfg.rank, int(CPU_SLAB_BYTES // (8 * inner)))
    dims = tuple(cfg.dims[:-1]) + (last,)
    sub = dataclasses.replace(cfg, dims=dims)
    return sub, None if x_host_flat is None else x_host_flat[: inner * last], (f"leading slab {'x'.join(map(str, dims))} of {cfg.name} "
                                              f"(N={sub.entries}, same r/p/s) decomposed as one tensor")


def cpu_baseline(cfg, x_host_flat, seed, budget_s=30.0):
    """Oracle port on the host cores, bounded to ~budget_s of CPU work, same
    X bits as the GPU arm (the leading slab for C5)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import srtt_oracle as O

    cfg, x_host_flat, what = cpu_sample(cfg, x_host_flat)
    X = O.as_tensor(x_host_flat, cfg.dims)
    res = _time_cpu_policies(O, cfg, X, seed, budget_s)
    best = min(res, key=lambda k: res[k][0])
    med, runs = res[best]
    ncpu = os.cpu_count()
    return {"value": cfg.entries / med, "unit": UNIT, "cores": ncpu, "kind": "port",
            "cpu_model": _cpu_model(),
            "sample": f"{what}, median of {runs} runs of the oracle port (numpy + OpenBLAS restatement of the "
                      f"reference in oracle/; the reference needs Eigen, absent). Faster of the reference's two "
                      f"host policies: {best} ("
                      + ", ".join(f"{k}: {v[0]:.4g} s" for k, v in res.items())
                      + f"; exec = ExecPolicy{{workers={ncpu}}} + sliced_core, 1 BLAS thread per worker; "
                        f"serial = no policy, BLAS on {ncpu} threads)",
            "seconds_per_step": med, "policy": best,
            "policies_s": {k: v[0] for k, v in res.items()}}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    """The reference's CPU path (oracle port) on the host cores, same metric /
    unit / config dict as the GPU arm and the same X bits (the GPU arm's
    synth generator, copied to the host; C5: its leading 2.2 GB slab)."""
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    from paper_2603_21379_b200 import synth

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import srtt_oracle as O

    full = synth.CONFIGS[args.config]
    cfg, _, what = cpu_sample(full, None)
    if cfg is full:
        what = f"full {full.name} decomposition per step"
    x, bits = _host_tensor(full, dims=None if cfg is full else cfg.dims)
    X = O.as_tensor(x, cfg.dims)
    # warm-up: one run of each host policy picks the faster one
    res = _time_cpu_policies(O, cfg, X, 0, budget_s=0.0)
    best = min(res, key=lambda k: res[k][0])
    pol = O.ExecPolicy(workers=os.cpu_count()) if best == "exec" else None
    from threadpoolctl import threadpool_limits

    def step():
        if best == "exec":
            with threadpool_limits(1):
                _run_oracle(O, cfg, X, 0, pol)
        else:
            _run_oracle(O, cfg, X, 0, pol)

    for _ in range(max(0, args.warmup - 2)):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = cfg.entries * args.steps / el
    ncpu = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_dict(full), "parallelism": f"host, {ncpu} cores",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncpu, "kind": "port", "cpu_model": _cpu_model(),
                             "policy": best, "policies_s": {k: v[0] for k, v in res.items()},
                             "sample": f"{what}, {bits}; oracle port (numpy + OpenBLAS restatement of the "
                                       f"reference in oracle/; the reference needs Eigen, absent in this image), "
                                       f"faster of its two host policies: {best} (exec = ExecPolicy{{workers="
                                       f"{ncpu}}} + sliced_core, 1 BLAS thread per worker; serial = no policy, "
                                       f"BLAS on {ncpu} threads)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# FP64 tensor-core (DMMA.8x8x4) peak measured on this pool's B200
# (profiles/r01_fp64_peak_microbench.txt); the bf16 figure in
# MEASURED_PEAKS.json does not apply to an fp64 kernel.
DMMA_PEAK_TFLOPS = 37.07


def core_flops(cfg):
    """Algorithmic flops of the core pass: the TTM chain in mode order
    2 N r0 + 2 (N/n0) r0 r1 + ..., no padding."""
    n = float(cfg.entries)
    f, cur = 0.0, n
    for k, nk in enumerate(cfg.dims):
        r = cfg.rank if cfg.kind == "tucker" else (cfg.rank if k == 0 else 0)
        if r == 0:
            break
        f += 2.0 * cur * r
        cur = cur / nk * r
    if cfg.kind == "htucker":  # root transfer: 2 N r_left (+ tiny second GEMM)
        f = 2.0 * n * cfg.rank
    return f


def core_roofline(cfg, core_s, peaks, peak_kind):
    """Roofline of the dominant kernel (core pass, X streamed once): HBM-bound
    when its arithmetic intensity on the DMMA pipe is under the ridge, else
    FP64-tensor-bound (C5: 2 r0 = 64 flop per 8-byte entry)."""
    alg_bytes = 8.0 * cfg.entries
    flops = core_flops(cfg)
    ridge = DMMA_PEAK_TFLOPS * 1e12 / (peaks["hbm_gbs"] * 1e9)
    gbs = alg_bytes / core_s / 1e9 if core_s > 0 else None
    tfs = flops / core_s / 1e12 if core_s > 0 else None
    common = {"kernel": "core_kernel (K3/K5 streaming multi-TTM)", "traffic": _traffic_from_profiles(cfg.name),
              "algorithmic_bytes_per_launch": alg_bytes, "algorithmic_flops_per_launch": flops,
              "kernel_ms": core_s * 1e3}
    if flops / alg_bytes > ridge:
        return dict(common, bound="tensor", achieved=tfs, peak=DMMA_PEAK_TFLOPS,
                    peak_kind="measured (fp64 DMMA microbench, profiles/r01_fp64_peak_microbench.txt)",
                    unit="TFLOP/s", frac=(tfs / DMMA_PEAK_TFLOPS) if tfs else None,
                    hbm={"achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": (gbs / peaks["hbm_gbs"]) if gbs else None})
    return dict(common, bound="hbm", achieved=gbs, peak=peaks["hbm_gbs"], peak_kind=peak_kind, unit="GB/s",
                frac=(gbs / peaks["hbm_gbs"]) if gbs else None)


def _config_dict(cfg):
    return {"workload": cfg.name, "description": cfg.description, "dims": list(cfg.dims), "rank": cfg.rank,
            "oversampling": cfg.p,
            "samples_per_target": (f"alpha={cfg.alpha} rule" if cfg.alpha else cfg.samples()[0]), "entries": cfg.entries,
            "bytes": cfg.entries * 8, "l2": "inputs larger than L2 (126 MB); no flush" if cfg.entries * 8 > 126e6
            else "input smaller than L2: 256 MB L2 flush between steps, inside the timed span"}


# ---------------------------------------------------------------------------
# product arm
# ---------------------------------------------------------------------------
def run_product(args):
    import torch

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import synth

    cfg = synth.CONFIGS[args.config]
    dims = list(cfg.dims)
    x = synth.make_tensor(cfg, seed=rank, backend="torch", device=f"cuda:{local}")
    torch.cuda.synchronize()
    h = P.Handle(local, use_graphs=True)
    stream = torch.cuda.current_stream()
    h.set_stream(stream.cuda_stream)
    small = cfg.entries * 8 < 256e6
    flush = torch.empty(int(256e6 // 8), dtype=torch.float64, device=dev) if small else None

    rep = P.SubsampleReport()
    for _ in range(args.warmup):
        _run_product(P, cfg, x, dims, 0, h, report=rep)
    torch.cuda.synchronize()
    launches_per_step = rep.launches

    last = {}

    def digest(res):
        """All outputs of one decomposition, flattened (device -> host copy on
        the current stream, i.e. ordered after the recorded work)."""
        if hasattr(res, "core"):
            ts = [res.core] + list(res.factors)
        else:
            ts = list(res.leaf_factors) + [t for t in res.transfers if t is not None and t.numel() > 0]
        return torch.cat([t.reshape(-1) for t in ts]).cpu()

    def timed_loop(n):
        # one event pair around all n stream-ordered calls (device outputs, no
        # report): host preparation of step i+1 overlaps the kernels of step i,
        # and any idle gap between steps is inside the span. The optional L2
        # flush (inputs smaller than L2 only) is inside the span as well
        # (conservative).
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            if flush is not None:
                flush.fill_(1.0)
            last["res"] = _run_product(P, cfg, x, dims, 0, h)
        e1.record(stream)
        e1.synchronize()
        last["digest"] = digest(last["res"])  # read right after the span: must already be complete
        return e0.elapsed_time(e1) / 1e3

    def kernel_samples(n):
        # the core kernel's own duration (CUDA events around that launch
        # inside the library), from report-carrying calls outside the timed loop
        # (a stream-ordered call is enqueued right before each one, so the
        # measured launch starts on a busy GPU at load clocks, as inside the
        # timed loop, not on one that idled during the previous read-back)
        core_t = []
        for _ in range(n):
            _run_product(P, cfg, x, dims, 0, h)
            r = P.SubsampleReport()
            _run_product(P, cfg, x, dims, 0, h, report=r)
            core_t.append(r.kernel_seconds.get("core", 0.0))
        return core_t

    # the core kernel's own duration, sampled on both sides of the timed loop
    # (after the warm-ups; again after the loop, when a DMMA-heavy config has
    # run into the board's power cap): the smaller median is reported -- the
    # launch inside the loop cannot take longer than a whole step
    core_t_pre = kernel_samples(5)
    if world > 1:
        torch.distributed.barrier()
    out_buf = _OUT.get(cfg.name)
    if out_buf is not None:  # outputs the timed calls must rewrite
        out_buf[0].zero_()
        for f in out_buf[1]:
            f.zero_()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    elapsed = timed_loop(args.steps)
    timed_digest = last["digest"]
    torch.cuda.synchronize()
    # keep the same workload running until the clock sampler has >= 3 samples
    t_extra = time.perf_counter()
    while len(sampler.samples) < 3 and time.perf_counter() - t_extra < 10:
        timed_loop(max(1, args.steps // 4))
    sampler.stop()
    clocks = sampler.summary()
    core_t = kernel_samples(8)
    # the last timed call's outputs equal a synchronous call's, bit for bit
    # (deterministic engine): guards the timed span against unordered work
    torch.cuda.synchronize()
    ref_digest = digest(_run_product(P, cfg, x, dims, 0, h, report=P.SubsampleReport()))
    verified = bool(torch.equal(timed_digest, ref_digest))
    el = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(el, op=torch.distributed.ReduceOp.MAX)
    elapsed = float(el.item())
    value = world * cfg.entries * args.steps / elapsed

    # e2e: through the C-ABI with X in pinned host memory, outputs to host
    x_host = x.cpu().pin_memory()
    xh = x_host.numpy()
    if 2 * cfg.entries * 8 > 0.6 * torch.cuda.get_device_properties(dev).total_memory:
        # the library stages X into its own device buffer: drop the resident
        # copy first (C5: 68.7 GB twice does not fit with the workspace)
        del x
        _OUT.clear()
        torch.cuda.empty_cache()
    for _ in range(max(1, min(args.warmup, 2))):
        _run_product(P, cfg, xh, dims, 0, h, device_out=False)
    e2e_steps = max(1, min(args.steps, 20))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(e2e_steps):
        _run_product(P, cfg, xh, dims, 0, h, device_out=False)
    ev1.record(stream)
    ev1.synchronize()
    e2e_el = torch.tensor([ev0.elapsed_time(ev1) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_el, op=torch.distributed.ReduceOp.MAX)
    e2e_value = world * cfg.entries * e2e_steps / float(e2e_el.item())
    samples_total = (sum(cfg.samples()) if cfg.kind == "tucker"
                     else sum(cfg.node_samples(P.DimensionTree.balanced(cfg.order), dims)[1:]))
    if cfg.kind == "tucker":
        d2h = 8 * (cfg.rank ** cfg.order + sum(n * cfg.rank for n in dims))
    else:
        d2h = 8 * (sum(n * cfg.rank for n in dims) + (cfg.order - 2) * cfg.rank ** 3 + cfg.rank ** 2)
    h2d = 8 * cfg.entries + 8 * samples_total

    peaks, peak_kind = _peaks()
    core_med = statistics.median(core_t) if core_t else 0.0
    if core_t_pre:
        core_med = min(core_med, statistics.median(core_t_pre)) if core_med > 0 else statistics.median(core_t_pre)
    roofline = core_roofline(cfg, core_med, peaks, peak_kind)
    roofline["kernel_share_of_step"] = core_med / (elapsed / args.steps)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(cfg),
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "clocks": clocks, "gpu_launches": launches_per_step * args.steps,
            "outputs_verified": verified,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps},
            "roofline": roofline}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, x_host.numpy(), 0)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _local_part(cfg, x_full, world, rank, P, sharded):
    """This rank's part of the ONE global tensor: Tucker -> last-mode slab
    X[..., lo:hi) (parallel.hpp:400-404 bounds); H-Tucker -> columns
    [c_lo, c_hi) of the root matricization. Both are contiguous byte ranges."""
    dims = list(cfg.dims)
    if cfg.kind == "tucker":
        lo, hi = sharded.slab_bounds(dims[-1], world, rank)
        inner = cfg.entries // dims[-1]
        return x_full[lo * inner:hi * inner].clone(), (lo, hi)
    tree = P.DimensionTree.balanced(cfg.order)
    lo, hi, nl, _ = sharded.column_bounds(tree, dims, world, rank)
    return x_full[lo * nl:hi * nl].clone(), (lo, hi)


def run_sharded(args, replicated=False):
    """ONE decomposition of the config's global tensor per step, split over
    the ranks (strong scaling), through the fused C-ABI entries whose handle
    owns an NCCL communicator (kernels and allreduces in one CUDA graph per
    rank). Two regimes (north star): sharded -- each rank holds only its
    contiguous part (Tucker: last-mode slab; H-Tucker: a column range of the
    root matricization; srtt_sub_r_hosvd_sharded / srtt_sub_r_rtl_ht_sharded);
    replicated -- every rank holds all of X, modes / nodes are assigned to
    ranks and the full pass is split (srtt_sub_r_*_replicated)."""
    import torch
    import torch.distributed as dist

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import sharded, synth

    cfg = synth.CONFIGS[args.config]
    dims = list(cfg.dims)
    # every rank generates the SAME global tensor (seed 0, deterministic
    # generator) and keeps only its part
    x_full = synth.make_tensor(cfg, seed=0, backend="torch", device=f"cuda:{local}")
    if replicated:
        x_loc = x_full
    else:
        x_loc, part = _local_part(cfg, x_full, world, rank, P, sharded)
    del x_full
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    h = P.Handle(local, use_graphs=True)
    stream = torch.cuda.current_stream()
    h.set_stream(stream.cuda_stream)
    sharded.comm_init(h)
    if cfg.kind == "tucker":
        ranks = [cfg.rank] * cfg.order
        samples = cfg.samples()
        out = (torch.empty(cfg.rank ** cfg.order, dtype=torch.float64, device=dev),
               [torch.empty(n * cfg.rank, dtype=torch.float64, device=dev) for n in dims])

        def step(report=None, x=x_loc, device_out=True):
            return sharded.sub_r_hosvd_nccl(x, dims, ranks, cfg.p, samples, 0, handle=h, report=report,
                                            out=out if device_out else None, device_out=device_out,
                                            replicated=replicated)

        def digest(res):
            return torch.cat([res.core.reshape(-1)] + [f.reshape(-1) for f in res.factors]).cpu()
    else:
        tree = P.DimensionTree.balanced(cfg.order)
        ranks = P.uniform_node_ranks(tree, cfg.rank)
        samples = cfg.node_samples(tree, dims)

        def step(report=None, x=x_loc, device_out=True):
            return sharded.sub_r_rtl_ht_nccl(x, dims, tree, ranks, samples, cfg.p, 0, handle=h, report=report,
                                             device_out=device_out, replicated=replicated)

        def digest(res):
            return torch.cat([u.reshape(-1) for u in res.leaf_factors] +
                             [t.reshape(-1) for t in res.transfers if t is not None]).cpu()

    rep = P.SubsampleReport()
    for _ in range(args.warmup):
        step(report=rep)
    launches_per_step = rep.launches
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        res = step()
    ev1.record(stream)
    ev1.synchronize()
    timed_digest = digest(res)
    t_extra = time.perf_counter()
    while len(sampler.samples) < 3 and time.perf_counter() - t_extra < 10:
        step()
        torch.cuda.synchronize()
    sampler.stop()
    el = torch.tensor([ev0.elapsed_time(ev1) / 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    elapsed = float(el.item())
    # outputs of the last timed call == a synchronous call's, bit for bit
    core_t = []
    for _ in range(5):
        r = P.SubsampleReport()
        ref = step(report=r)
        core_t.append(r.kernel_seconds.get("core", 0.0))
    verified = bool(torch.equal(timed_digest, digest(ref)))
    ok = torch.tensor([1.0 if verified else 0.0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    verified = bool(ok.item() == 1.0)

    # e2e: the same call with this rank's part in pinned HOST memory and the
    # outputs copied back to the host inside the timed region
    xh = x_loc.cpu().pin_memory().numpy()
    if 2 * x_loc.numel() * 8 > 0.6 * torch.cuda.get_device_properties(dev).total_memory:
        del x_loc
        torch.cuda.empty_cache()
    step(x=xh, device_out=False)
    e2e_steps = max(1, min(args.steps, 10))
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        step(x=xh, device_out=False)
    e1.record(stream)
    e1.synchronize()
    e2e_el = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_el, op=dist.ReduceOp.MAX)
    if cfg.kind == "tucker":
        d2h = 8 * (cfg.rank ** cfg.order + sum(n * cfg.rank for n in dims))
    else:
        d2h = 8 * (sum(n * cfg.rank for n in dims) + (cfg.order - 2) * cfg.rank ** 3 + cfg.rank ** 2)

    # roofline of this rank's core / root pass over its part
    peaks, peak_kind = _peaks()
    core_med = statistics.median(core_t)
    local_cfg = _local_cfg(cfg, world, rank, P, sharded)
    roofline = core_roofline(local_cfg, core_med, peaks, peak_kind)
    roofline["kernel_share_of_step"] = core_med / (elapsed / args.steps)
    roofline["per_rank_part"] = list(local_cfg.dims)
    if world > 1:
        roofline["traffic"] = None  # the committed ncu capture is of the single-GPU launch
    line = {"metric": METRIC, "value": cfg.entries * args.steps / elapsed, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_dict(cfg),
            "parallelism": (f"replicated x{world}: X on every rank, {'modes' if cfg.kind == 'tucker' else 'nodes'} "
                            f"assigned to ranks, factor pack + full-pass partials allreduced (fused C-ABI + NCCL, "
                            f"one CUDA graph per rank)" if replicated else
                            f"{'slab' if cfg.kind == 'tucker' else 'column-range'}-sharded x{world} "
                            f"(one global tensor; fused C-ABI + NCCL allreduce of sketches and core, one CUDA "
                            f"graph per rank)"),
            "clocks": sampler.summary(), "gpu_launches": launches_per_step * args.steps,
            "outputs_verified": verified,
            "e2e": {"value": cfg.entries * e2e_steps / float(e2e_el.item()), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * (cfg.entries if replicated else int(np.prod(local_cfg.dims))),
                    "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "per_rank": True},
            "roofline": roofline}
    if rank == 0:
        print(json.dumps(line), flush=True)
    sharded.comm_destroy(h)
    dist.destroy_process_group()


def _local_cfg(cfg, world, rank, P, sharded):
    """A Config describing this rank's part (for the per-rank roofline)."""
    import dataclasses

    dims = list(cfg.dims)
    if cfg.kind == "tucker":
        lo, hi = sharded.slab_bounds(dims[-1], world, rank)
        return dataclasses.replace(cfg, dims=tuple(dims[:-1] + [hi - lo]))
    tree = P.DimensionTree.balanced(cfg.order)
    lo, hi, nl, _ = sharded.column_bounds(tree, dims, world, rank)
    # the root pass streams n_left x (hi - lo) entries: model it as a 2-mode part
    return dataclasses.replace(cfg, dims=(nl, hi - lo))


def _traffic_from_profiles(cfg_name):
    """dram bytes per core-kernel launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", f"ncu_core_{cfg_name}.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=["c1", "c2", "c3", "c4", "c5", "c4a20", "c5s64k"], default="c5",
                    help="c1-c5: BASELINE.json configs; c4a20 / c5s64k: sketch-heavy variants ADDED for the K1 "
                         "bandwidth measurement (not BASELINE configs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", choices=["auto", "replicas", "sharded", "replicated"], default="auto",
                    help="auto: N=1 single-GPU decomposition; N>1 ONE global tensor over the ranks (strong "
                         "scaling): slab-sharded for c5 / c5s64k (the BASELINE's sharded config), replicated with "
                         "modes / nodes assigned to ranks for the configs that fit per GPU; replicas: independent "
                         "decompositions per rank (weak scaling); sharded / replicated: force that NCCL path (also "
                         "at N=1)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "sharded" or (args.mode == "auto" and _dist_env()[1] > 1 and args.config.startswith("c5")):
        run_sharded(args)
    elif args.mode == "replicated" or (args.mode == "auto" and _dist_env()[1] > 1):
        run_sharded(args, replicated=True)
    else:
        run_product(args)


if __name__ == "__main__":
    main()
