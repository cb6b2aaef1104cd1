"""Pipe, shared-memory and stall-reason metrics of every kernel of an ncu --set full report as
JSON (profiles/<tag>_stalls.json): python tools/ncu_stalls.py report.ncu-rep out.json"""
import csv, json, subprocess, sys

KEEP = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_dmma.sum", "sm__icc_request_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, units = r[0], r[1]
res = []
for row in r[2:]:
    d = {"kernel": row[hdr.index("Kernel Name")]}
    for k, h in enumerate(hdr):
        if h in KEEP:
            d[h] = (row[k] + " " + units[k]).strip()
        elif h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            d["stall_" + h[len("smsp__average_warps_issue_stalled_"):]] = (row[k] + " " + units[k]).strip()
    res.append(d)
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
