"""Per-phase wall time of the slab-sharded path at world size 1 (development)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2603_21379_b200 as P  # noqa: E402
from paper_2603_21379_b200 import sharded, synth  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dims = list(cfg.dims)
x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
h = P.Handle(0, use_graphs=False)
h.set_stream(torch.cuda.current_stream().cuda_stream)
ph = sharded.GpuShardPhases(h)
ranks = [cfg.rank] * cfg.order
samples = cfg.samples()
L = len(dims) - 1
for it in range(4):
    t = [time.perf_counter()]
    zs = ph.shard_sketches(x, dims, 0, dims[L], ranks, cfg.p, samples, 0)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    for k in range(L):
        dist.all_reduce(zs[k])
    zs[L] = sharded._gather_rows(zs[L], dims[L], cfg.rank + cfg.p, [dims[L]], None)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    us, ach = ph.bases_from_sketches(dims, ranks, cfg.p, samples, 0, zs)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    g = ph.shard_core(x, dims, 0, dims[L], ranks, us)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    dist.all_reduce(g)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    names = ["sketch", "collect", "bases", "core", "allreduce"]
    print(it, {n: round((b - a) * 1e6) for n, a, b in zip(names, t[:-1], t[1:])})
dist.destroy_process_group()
