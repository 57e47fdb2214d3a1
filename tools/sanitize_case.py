"""Workload for compute-sanitizer (memcheck / racecheck / synccheck):
C1 and C2 at full size, an order-8 H-Tucker (8^8) and the flat-mode core
pass, all through the C-ABI, checked against the previous run's outputs."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import paper_2603_21379_b200 as P
from paper_2603_21379_b200 import synth

h = P.Handle(0, use_graphs=False)
for name in ("c1", "c2"):
    cfg = synth.CONFIGS[name]
    x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
    rep = P.SubsampleReport()
    t = P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, report=rep, dims=list(cfg.dims), handle=h)
    e = P.tucker_rel_error(x, t, dims=list(cfg.dims), handle=h)
    print(name, rep.achieved_ranks, f"relerr {e:.3e}", flush=True)
    del x
dims = (8,) * 8
tree = P.DimensionTree.balanced(8)
y = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda")
ranks = P.uniform_node_ranks(tree, 4)
samples = [1] + [min(24, tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
rep = P.HtSubsampleReport()
hd = P.sub_r_rtl_ht(y, tree, ranks, samples, 4, 0, report=rep, dims=list(dims), handle=h)
print("ht 8^8", rep.achieved_ranks, flush=True)
xs = np.random.default_rng(0).standard_normal((30, 40, 50))
fs = [np.linalg.qr(np.random.default_rng(k).standard_normal((n, 5)))[0] for k, n in enumerate(xs.shape)]
os.environ["SRTT_FORCE_FLAT"] = "1"
g = P.multi_ttm_core(xs, fs, handle=h)
print("flat core", float(np.linalg.norm(g)), flush=True)
print("SANITIZE_CASE_DONE")
