"""Summarise ncu outputs (launch list CSV + one --set full report) into profiles/ (dev tool).

    python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <out-prefix>
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic",
        "launch__grid_size", "launch__block_size", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            tot[name] += float(r[vi].replace(",", ""))
            cnt[name] += 1
    allt = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_ns": tot[k], "avg_ns": tot[k] / cnt[k],
             "share": tot[k] / allt} for k in sorted(tot, key=lambda k: -tot[k])]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
               float(v)) for h, v in zip(hdr, r)
              if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("ratio") and v]
        d["top_stalls"] = sorted(st, key=lambda x: -x[1])[:6]
        res.append(d)
    return res


if __name__ == "__main__":
    lcsv, rep, prefix = sys.argv[1:4]
    summary = {"launch_list": launches(lcsv), "full_capture": full(rep)}
    json.dump(summary, open(prefix + ".json", "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])
