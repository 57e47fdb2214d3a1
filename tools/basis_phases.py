"""Phase clocks of basis_small_kernel block 0 (development build: make PROF=1,
run with SRTT_PROFILE_BUILD=1)."""
import ctypes as C
import os
import sys

os.environ["SRTT_PROFILE_BUILD"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_21379_b200 as P  # noqa: E402
from paper_2603_21379_b200 import srtt, synth  # noqa: E402

names = ["load", "qr", "to_B", "jacobi", "sigma", "apply", "pad", "store"]
for name in sys.argv[1:] or ["c2"]:
    cfg = synth.CONFIGS[name]
    x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
    h = P.Handle(0, use_graphs=False)
    for _ in range(3):
        if cfg.kind == "tucker":
            P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, dims=list(cfg.dims), handle=h,
                          device_out=True)
        else:
            tree = P.DimensionTree.balanced(cfg.order)
            ranks = P.uniform_node_ranks(tree, cfg.rank)
            samples = [1] + [min(4 * (cfg.rank + cfg.p), tree.node_cols(i, cfg.dims)) for i in range(1, tree.num_nodes)]
            P.sub_r_rtl_ht(x, tree, ranks, samples, cfg.p, 0, dims=list(cfg.dims), handle=h, device_out=True)
        torch.cuda.synchronize()
    clk = (C.c_longlong * 16)()
    srtt._L().srtt_debug_basis_clocks(clk)
    v = list(clk)[:8]
    d = np.diff(v)
    print(name, "small cycles:", " ".join(f"{n}={int(c)}" for n, c in zip(names, d)), "total", v[7] - v[0])
    t = list(clk)[8:14]
    if os.environ.get("HJ"):
        print(name, "hj cycles: load", t[1] - t[0], "jacobi", t[2] - t[1], "rank", t[3] - t[2], "out", t[4] - t[3],
              "sweeps", clk[15])
        continue
    if t[0]:
        tn = ["qr", "jacobi", "sigma", "apply", "store"]
        print(name, "top cycles:", " ".join(f"{n}={int(b - a)}" for n, a, b in zip(tn, t[:-1], t[1:])))
