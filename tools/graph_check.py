"""Graph-mode (stream-ordered, no report) vs report-mode calls: same outputs,
and per-call device time of each (development check)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_21379_b200 as P  # noqa: E402
from paper_2603_21379_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = synth.CONFIGS[name]
dims = list(cfg.dims)
x = synth.make_tensor(cfg, seed=0, backend="torch", device="cuda")
torch.cuda.synchronize()
h = P.Handle(0, use_graphs=True)
s = torch.cuda.current_stream()
h.set_stream(s.cuda_stream)
core = torch.empty(cfg.rank ** cfg.order, dtype=torch.float64, device="cuda")
facs = [torch.empty(n * cfg.rank, dtype=torch.float64, device="cuda") for n in dims]


def call(rep=None):
    return P.sub_r_hosvd(x, [cfg.rank] * cfg.order, cfg.p, cfg.samples(), 0, dims=dims, handle=h,
                         device_out=True, out=(core, facs), report=rep)


for _ in range(3):
    call()
torch.cuda.synchronize()
n = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(n):
    call()
e1.record(s)
e1.synchronize()
print(f"graph mode: {e0.elapsed_time(e1) / n:.3f} ms/call")
c_graph = core.cpu().numpy().copy()
f_graph = [f.cpu().numpy().copy() for f in facs]
rep = P.SubsampleReport()
call(rep)
torch.cuda.synchronize()
print("report mode timings (us):", {k: round(v * 1e6, 1) for k, v in rep.timings.items() if v},
      {k: round(v * 1e6, 1) for k, v in rep.kernel_seconds.items()})
c_rep = core.cpu().numpy()
print("core identical:", np.array_equal(c_graph, c_rep), "max diff", np.abs(c_graph - c_rep).max(),
      "norm", np.linalg.norm(c_rep))
print("factors identical:", all(np.array_equal(a, b.cpu().numpy()) for a, b in zip(f_graph, facs)))

# per-call events, output zeroed before each call: every call must rewrite it
ref = c_rep
times = []
for i in range(6):
    core.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    call()
    b.record(s)
    b.synchronize()
    times.append(a.elapsed_time(b))
    ok = np.array_equal(core.cpu().numpy(), ref)
    print(f"call {i}: {times[-1]:.3f} ms, output rewritten and identical: {ok}")
