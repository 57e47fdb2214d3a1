"""Per-CUDA-source-line stall samples of an ncu report (cuda,sass source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = [r for r in rows if r and r[0] == "Line No"][0]
ci = hdr.index("Warp Stall Sampling (All Samples)")
lines, cur = {}, None
for r in rows:
    if not r or r[0] in ("File Path", "Function Name", "Line No"):
        continue
    if r[0]:
        cur = (int(r[0]), r[1])
        lines.setdefault(cur, 0.0)
    elif cur is not None and len(r) > ci:
        try:
            lines[cur] += float(r[ci] or 0)
        except ValueError:
            pass
tot = sum(lines.values()) or 1
for (ln, src), v in sorted(lines.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  {ln:5d}  {src.strip()[:100]}")
