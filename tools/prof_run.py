"""Small driver for ncu: a few decompositions of one config (default c2)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2603_21379_b200 as P
from paper_2603_21379_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.CONFIGS[name]
x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
torch.cuda.synchronize()
h = P.Handle(0)
for i in range(reps):
    rep = P.SubsampleReport()
    if cfg.kind == "tucker":
        P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, report=rep, dims=list(cfg.dims), handle=h, device_out=True)
    else:
        tree = P.DimensionTree.balanced(cfg.order)
        ranks = P.uniform_node_ranks(tree, cfg.rank)
        samples = cfg.node_samples(tree, cfg.dims)
        P.sub_r_rtl_ht(x, tree, ranks, samples, cfg.p, 0, report=rep, dims=list(cfg.dims), handle=h, device_out=True)
    print(i, {k: round(v * 1e6, 1) for k, v in rep.timings.items() if v}, {k: round(v * 1e6, 1) for k, v in rep.kernel_seconds.items()}, rep.launches, 'sweeps', getattr(rep, 'jacobi_sweeps', None))
