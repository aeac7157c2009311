"""Key metrics of an ncu --set full report, one line per kernel launch and metric.

  python scripts/ncu_summary.py REPORT.ncu-rep "header line" > profiles/<round>/ncu_full_<cfg>_summary.txt
"""
import csv
import io
import subprocess
import sys

KEEP = {
    ("GPU Speed Of Light Throughput", "Memory Throughput"), ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Duration"), ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Compute Workload Analysis", "Executed Ipc Active"), ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Memory Workload Analysis", "Memory Throughput"), ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Memory Workload Analysis", "L2 Hit Rate"), ("Scheduler Statistics", "No Eligible"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"), ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Cluster Size"), ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Registers Per Thread"), ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Theoretical Occupancy"), ("Occupancy", "Achieved Occupancy"),
}
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
ki, ks, km, ku, kv = (hdr.index(c) for c in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
for r in rows[1:]:
    if (r[ks], r[km]) in KEEP:
        print(" | ".join([r[ki].replace("void ", "").split("(")[0], r[ks], r[km], r[ku], r[kv]]))
