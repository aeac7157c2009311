"""DRAM traffic per launch from an ncu --set full report -> profiles/<round>/traffic.json.

  python scripts/ncu_traffic.py REPORT.ncu-rep OUT.json [--prefix stress:] [--augs A] [--calls N]

For each library kernel name (bench.py's kernel_times names; e.g. ssp_kernel covers the 32-bit
launch and its 64-bit redo launch of one solve_batch call): dram__bytes_read.sum +
dram__bytes_write.sum summed over the captured launches, divided by N library calls (default 1).  --augs A also records the bytes per
augmentation (A = augmentations the captured launch performed), which bench.py scales to the
augmentations of its own launch.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
prefix = sys.argv[sys.argv.index("--prefix") + 1] if "--prefix" in sys.argv else ""
augs = float(sys.argv[sys.argv.index("--augs") + 1]) if "--augs" in sys.argv else None
calls = float(sys.argv[sys.argv.index("--calls") + 1]) if "--calls" in sys.argv else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
ki, kr, kw, kt = (hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"),
                  hdr.index("gpu__time_duration.sum"))
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
units = rows[1]
acc = {}
for r in rows[2:]:
    m = re.search(r"(ssp_cluster_kernel|ssp_kernel|rounds_cluster_kernel|rounds_kernel|churn_state_kernel|"
                  r"edge_update_kernel|warm_kernel|mc_rounds_kernel)", r[ki])
    if not m:
        continue
    name = {"rounds_cluster_kernel": "rounds_kernel"}.get(m.group(1), m.group(1))  # the library's names
    b = float(r[kr].replace(",", "")) * unit[units[kr]] + float(r[kw].replace(",", "")) * unit[units[kw]]
    a = acc.setdefault(prefix + name, [0.0, 0, 0.0])
    a[0] += b
    a[1] += 1
    a[2] += float(r[kt].replace(",", ""))
res = json.load(open(out)) if os.path.exists(out) else {"kernels": {}}
for k, (b, c, t) in acc.items():
    e = {"dram_bytes_per_launch": b / calls, "kernel_launches_captured": c, "library_calls": calls,
         "duration_per_call_" + units[kt]: t / calls, "source": os.path.basename(rep)}
    if augs:
        e["dram_bytes_per_aug"] = b / calls / augs
    res["kernels"][k] = e
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
