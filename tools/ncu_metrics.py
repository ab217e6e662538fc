"""Print selected raw metrics of every kernel in an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
pats = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "lts__t_sector_hit_rate.pct", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
                        "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                        "lts__t_sectors.sum", "lts__d_sectors.sum", "smsp__warps_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    print("kernel:", vals[hdr.index("Kernel Name")][:80])
    for p in pats:
        for i, h in enumerate(hdr):
            if h == p:
                print(f"   {h:70s} {units[i]:10s} {vals[i]}")
