"""Summarise an ncu report: key throughput metrics, stall reasons, hot SASS."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw))); h = rows[0]; v = rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]
out = {}
for i, n in enumerate(h):
    if n in keys:
        out[n] = v[i]
        print(f"{n:75s} {v[i]}")
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
        try: st.append((float(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
tot = sum(s for s, _ in st) or 1
print("stalls:", ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]; ci = {n: i for i, n in enumerate(hh)}
data = [r for r in rows[2:] if len(r) > 5]
tot = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data) or 1
for r in sorted(data, key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{100*int(r[ci['Warp Stall Sampling (All Samples)']])/tot:5.1f}% {r[ci['Address']][-5:]} {r[ci['Source']].strip()[:80]}")
