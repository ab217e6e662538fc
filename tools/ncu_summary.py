"""Summarise an ncu report (one or more kernels) into JSON under profiles/."""
import csv, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(txt))
hdr, units = rows[0], rows[1]
res = []
for vals in rows[2:]:
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            d[k] = {"value": vals[i], "unit": units[i]}
    def num(k, scale):
        u = d[k]["unit"]; v = float(d[k]["value"].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) if scale else v
    try:
        d["dram_bytes_per_launch"] = num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1)
    except Exception:
        pass
    res.append(d)
json.dump({"report": rep, "kernels": res}, open(out, "w"), indent=1)
print(json.dumps([{k: r.get(k) for k in ("kernel", "dram_bytes_per_launch")} for r in res]))
