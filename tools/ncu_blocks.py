"""Executed-instruction weight of straight-line SASS blocks (same exec count)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src))); hh = rows[1]; ci = {n: i for i, n in enumerate(hh)}
data = [r for r in rows[2:] if len(r) > 5]
ex = [int(r[ci["Instructions Executed"]] or 0) for r in data]
tot = sum(ex)
blocks, cur = [], None
for i, e in enumerate(ex):
    if cur and cur[2] == e: cur[1] = i
    else:
        cur = [i, i, e]; blocks.append(cur)
print("total executed", tot)
for w, b in sorted(((b[2] * (b[1] - b[0] + 1), b) for b in blocks), reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    i0, i1, e = b
    ops = {}
    for r in data[i0:i1 + 1]:
        op = r[ci["Source"]].strip().split()[0]
        if op.startswith("@"): op = r[ci["Source"]].strip().split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = ", ".join(f"{k}x{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    print(f"{100*w/tot:5.1f}% exec={e:8d} len={i1-i0+1:4d} @{data[i0][ci['Address']][-5:]}  {top}")
