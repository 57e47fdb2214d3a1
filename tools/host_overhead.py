"""Host vs device time per call (device outputs, no report): if the wall
clock per call exceeds the device time, the path is host-bound."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_21379_b200 as P  # noqa: E402
from paper_2603_21379_b200 import synth  # noqa: E402

for name in sys.argv[1:] or ["c2", "c4"]:
    cfg = synth.CONFIGS[name]
    dims = list(cfg.dims)
    x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
    h = P.Handle(0, use_graphs=True)
    s = torch.cuda.current_stream()
    h.set_stream(s.cuda_stream)
    if cfg.kind == "tucker":
        call = lambda: P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, dims=dims, handle=h,  # noqa
                                     device_out=True)
    else:
        tree = P.DimensionTree.balanced(cfg.order)
        ranks = P.uniform_node_ranks(tree, cfg.rank)
        samples = [1] + [min(4 * (cfg.rank + cfg.p), tree.node_cols(i, dims)) for i in range(1, tree.num_nodes)]
        call = lambda: P.sub_r_rtl_ht(x, tree, ranks, samples, cfg.p, 0, dims=dims, handle=h, device_out=True)  # noqa
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    n = 30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    host = []
    for _ in range(n):
        a = time.perf_counter()
        call()
        host.append(time.perf_counter() - a)
    e1.record(s)
    e1.synchronize()
    wall = (time.perf_counter() - t0) / n
    dev = e0.elapsed_time(e1) / 1e3 / n
    host.sort()
    enq = []
    for _ in range(10):
        torch.cuda.synchronize()
        a = time.perf_counter()
        call()
        enq.append(time.perf_counter() - a)
    enq.sort()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ga.record(s)
    for a_, b_ in evs:
        a_.record(s)
        call()
        b_.record(s)
    gb.record(s)
    gb.synchronize()
    per = [a_.elapsed_time(b_) for a_, b_ in evs]
    gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(n - 1)]
    print(f"   per-step sum {sum(per)/n:.3f} ms/call, span {ga.elapsed_time(gb)/n:.3f} ms/call, "
          f"mean gap {sum(gaps)/len(gaps)*1e3:.1f} us, per-step min/max {min(per):.3f}/{max(per):.3f}")
    print(f"{name}: wall/call {wall*1e3:.3f} ms  device/call {dev*1e3:.3f} ms  host call median {host[n//2]*1e3:.3f} ms"
          f"  enqueue (GPU idle) median {enq[5]*1e3:.3f} ms")
