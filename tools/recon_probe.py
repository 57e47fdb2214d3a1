"""Times the streamed reconstruction error (tucker_rel_error / ht_rel_error)
on the BASELINE configs with X resident in HBM; prints ms and the X-read
bandwidth (8 N bytes / time)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_21379_b200 as P  # noqa: E402
from paper_2603_21379_b200 import synth  # noqa: E402

for name in sys.argv[1:] or ["c2", "c3", "c4"]:
    cfg = synth.CONFIGS[name]
    dims = list(cfg.dims)
    x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
    if cfg.kind == "tucker":
        t = P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, dims=dims, device_out=True)
        fn = lambda: P.tucker_rel_error(x, t, dims=dims)  # noqa: E731
    else:
        tree = P.DimensionTree.balanced(cfg.order)
        ranks = P.uniform_node_ranks(tree, cfg.rank)
        samples = [1] + [min(4 * (cfg.rank + cfg.p), tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
        t = P.sub_r_rtl_ht(x, tree, ranks, samples, cfg.p, 0, dims=dims, device_out=True)
        fn = lambda: P.ht_rel_error(x, t, dims=dims)  # noqa: E731
    try:
        e = fn()
    except P.InvalidArgument:
        e = float("nan")
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        try:
            fn()
        except P.InvalidArgument:
            pass
        ts.append(time.perf_counter() - t0)
    tm = sorted(ts)[len(ts) // 2]
    print(f"{name}: rel_error={e:.6e}  {tm*1e3:.3f} ms  X-read {8*cfg.entries/tm/1e9:.0f} GB/s", flush=True)
    del x, t
    torch.cuda.empty_cache()
