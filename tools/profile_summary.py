"""Summarise ncu outputs (launch list CSV + --set full report) into profiles/<tag>_*.{json,md}."""
import csv
import collections
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
           "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(d["Metric Unit"], 1e-3)
        agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
             "share": sum(v) / tot} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))], tot


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                d[m] = row[hdr.index(m)] + (" " + units[hdr.index(m)] if units[hdr.index(m)] else "")
        res.append(d)
    return res


if __name__ == "__main__":
    tag, launch_csv, rep = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None
    L, tot = launches(launch_csv)
    F = full(rep) if rep else []
    json.dump({"launch_list": L, "total_us": tot, "full": F}, open(f"profiles/{tag}_ncu.json", "w"), indent=1)
    with open(f"profiles/{tag}_ncu.md", "w") as f:
        f.write(f"# ncu summary {tag}\n\nLaunch list (ncu --metrics gpu__time_duration.sum --clock-control none, "
                f"timed steps only via cudaProfilerStart/Stop; cold-cache serialised: compare shares)\n\n")
        f.write("| kernel | launches | mean us | share |\n|---|---|---|---|\n")
        for e in L:
            f.write(f"| {e['kernel'][:70]} | {e['launches']} | {e['mean_us']:.1f} | {e['share']:.3f} |\n")
        if F:
            f.write("\n--set full (one launch per kernel)\n\n")
            for d in F:
                f.write(f"## {d['kernel'][:100]}\n\n")
                for m in METRICS:
                    if m in d:
                        f.write(f"- {m}: {d[m]}\n")
                f.write("\n")
    print(open(f"profiles/{tag}_ncu.md").read())
