"""Wall time of the host-memory (e2e) call path, per call (development)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_21379_b200 as P  # noqa: E402
from paper_2603_21379_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
dims = list(cfg.dims)
x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
xh = x.cpu().pin_memory().numpy()
h = P.Handle(0, use_graphs=True)
h.set_stream(0)
for _ in range(3):
    P.sub_r_hosvd(xh, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, dims=dims, handle=h)
ts = []
for _ in range(10):
    t = time.perf_counter()
    rep = P.SubsampleReport()
    P.sub_r_hosvd(xh, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, dims=dims, handle=h, report=rep)
    ts.append(time.perf_counter() - t)
print(cfg.name, "wall/call ms", round(1e3 * sorted(ts)[5], 3), {k: round(v * 1e6, 1) for k, v in rep.timings.items() if v})
