"""Per-target K1 table from an ncu csv of tools/k1_probe.py (launch 2i+1 of
target i is the measured one; the rest are the grouped launches)."""
import csv
import json
import sys

csvf, logf = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(csvf)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
idx = {n: i for i, n in enumerate(h)}
per, names = {}, {}
for r in rows[hi + 1:]:
    per.setdefault(int(r[idx["ID"]]), {})[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    names[int(r[idx["ID"]])] = r[idx["Kernel Name"]]
targets = json.loads(open(logf).read().splitlines()[0])
ids = sorted(per)
k1 = [i for i in ids if "sketch_kernel" in names[i] or "sketch_contig_kernel" in names[i]]
hbm = 6552.0
print(f"{'target':24s} {'useful MB':>10s} {'us':>9s} {'useful GB/s':>11s} {'of HBM':>7s} {'DRAM MB':>9s} {'sect/req':>8s}")
for t_i, t in enumerate(targets):
    m = per[k1[2 * t_i + 1]]
    us = m["gpu__time_duration.sum"] / 1e3
    gbs = t["useful_bytes"] / (us * 1e-6) / 1e9
    kind = "K1c" if "contig" in names[k1[2 * t_i + 1]] else "K1"
    print(f"{t['target'] + ' ' + kind:24s} {t['useful_bytes'] / 1e6:10.1f} {us:9.1f} {gbs:11.0f} {gbs / hbm:7.2f} "
          f"{(m['dram__bytes_read.sum'] + m['dram__bytes_write.sum']) / 1e6:9.1f} "
          f"{m['l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum'] / max(1.0, m['l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum']):8.1f}")
