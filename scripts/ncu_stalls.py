"""Warp-stall reasons and the hottest source lines of one kernel in an ncu --set full report.

  python scripts/ncu_stalls.py REPORT.ncu-rep KERNEL_REGEX [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = [r for r in rows if r and r[0] == "Line No"][0]
names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {n: hdr.index(n) for n in names}
tot, per, cur = collections.Counter(), collections.Counter(), None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 7 or r[0] == "Line No" or r[0] == "" or r[2] != "-":
        continue
    c = collections.Counter({n: int(r[idx[n]] or 0) for n in names})
    tot += c
    per[(cur, r[0], r[1][:100])] += sum(c.values())
T = sum(tot.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tot.most_common() if v))
for k, v in per.most_common(top):
    print(f"{100 * v / T:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
