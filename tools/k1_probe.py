"""K1 (fused gather + sketch) per target: one srtt_sketch launch per Tucker
mode / H-Tucker node of a config, X resident on the device. Run under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
-k regex:sketch_kernel` for per-target DRAM traffic and duration; prints the
algorithmic (useful) bytes of each target: rows x w x 8 gathered + Z written.
It also times the grouped launch of a full decomposition (report events)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import paper_2603_21379_b200 as P
from paper_2603_21379_b200 import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c4a20"
cfg = synth.CONFIGS[name]
dims = list(cfg.dims)
x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
torch.cuda.synchronize()
h = P.Handle(0)
N = cfg.entries
targets = []
if cfg.kind == "tucker":
    for k, s in enumerate(cfg.samples()):
        targets.append((f"mode {k}", [k], N // dims[k], s, cfg.rank + cfg.p, k, dims[k]))
else:
    tree = P.DimensionTree.balanced(cfg.order)
    ws = cfg.node_samples(tree, dims)
    for i in range(1, tree.num_nodes):
        targets.append((f"node {i} {tree.node(i).modes}", tree.node(i).modes, tree.node_cols(i, dims), ws[i],
                        cfg.rank + cfg.p, i, tree.node_rows(i, dims)))
out = []
for label, modes, m, w, c, sid, rows in targets:
    cols, draws = P.sample_indices(m, w, 0, sid)
    for rep in range(2):  # launch 0 warms up, launch 1 is the measured one
        P.sketch(x, modes, cols, c, 0, sid, draws, dims=dims, handle=h)
    out.append({"target": label, "rows": rows, "w": w, "c": c,
                "useful_bytes": 8 * rows * w + 8 * rows * c, "contiguous_fibres": modes[0] == 0})
print(json.dumps(out))
# the grouped K1 of a full decomposition (device events around the launch)
ks = []
for _ in range(3):
    r = P.SubsampleReport()
    if cfg.kind == "tucker":
        P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, report=r, dims=dims, handle=h,
                      device_out=True)
    else:
        P.sub_r_rtl_ht(x, tree, P.uniform_node_ranks(tree, cfg.rank), cfg.node_samples(tree, dims), cfg.p, 0,
                       report=r, dims=dims, handle=h, device_out=True)
    ks.append(r.kernel_seconds["sketch"])
print(json.dumps({"grouped_sketch_s": ks, "useful_bytes_total": sum(o["useful_bytes"] for o in out),
                  "stages": r.timings}))
