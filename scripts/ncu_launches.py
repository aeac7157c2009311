"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file F) per kernel.

  python scripts/ncu_launches.py launches.csv "command line" > profiles/<round>/launches_<cfg>.txt
"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, kv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    short = r[ki].split("(")[0].replace("void ", "")[:72]
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += float(r[kv].replace(",", "")) / 1e6
tot = sum(v[1] for v in agg.values())
print("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)")
print(f"# command: {sys.argv[2] if len(sys.argv) > 2 else '?'}")
print(f"{'kernel':72s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:72s} {c:8d} {ms:10.3f} {100 * ms / tot:6.1f}%")
