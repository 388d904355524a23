"""Key metrics per kernel from an `ncu --set full` report (details page):
python scripts/ncu_summary.py rep.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {k: i for i, k in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Compute (SM) Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size", "Warp Cycles Per Issued Instruction", "Issued Warp Per Scheduler", "Executed Ipc Active"]
kern = {}
for r in rows[1:]:
    if len(r) < ix["Metric Value"] + 1:
        continue
    k = r[ix["Kernel Name"]].split("(")[0] + "#" + r[ix["ID"]]
    n = r[ix["Metric Name"]]
    if n in want:
        kern.setdefault(k, {})[n] = (r[ix["Metric Value"]] + " " + r[ix["Metric Unit"]]).strip()
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                      "sm__ops_path_tensor_src_fp64.sum,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed,"
                      "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h = rr[0]
    for r in rr[2:]:
        d = dict(zip(h, r))
        k = d.get("Kernel Name", "").split("(")[0] + "#" + d.get("ID", "")
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "sm__ops_path_tensor_src_fp64.sum", "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
                  "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"):
            if m in d:
                kern.setdefault(k, {})[m] = d[m] + " " + rr[1][h.index(m)]
for k, v in kern.items():
    print(k)
    for n, val in v.items():
        print(f"   {n:40s} {val}")
if "--json" in sys.argv:
    json.dump(kern, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
