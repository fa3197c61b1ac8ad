"""Summarise an ncu --set full report (details + raw counters + top stall reasons) as text:
python tools/ncu_summary.py REPORT.ncu-rep "header line" > profiles/....txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
if len(sys.argv) > 2:
    print("#", sys.argv[2])


def page(name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


want = ["Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy",
        "L2 Hit Rate"]
r = page("details")
h = r[0]
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(d["Kernel Name"].split("(")[0], "|", d["Metric Name"], "|", d["Metric Value"],
              d["Metric Unit"])
print("# raw counters")
r = page("raw")
h = r[0]
keys = ["l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]
for d in r[2:]:
    name = d[h.index("Kernel Name")].split("(")[0]
    for k in keys:
        if k in h:
            print(name, "|", k, "|", d[h.index(k)])
    st = []
    for k, v in zip(h, d):
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((k.replace("smsp__average_warps_issue_stalled_", "")
                           .replace("_per_issue_active.ratio", ""), float(v)))
            except ValueError:
                pass
    st.sort(key=lambda x: -x[1])
    print(name, "| stalls per issue |", ", ".join(f"{k} {v:.2f}" for k, v in st[:7]))
