"""Top source lines / SASS by warp-stall samples from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
# find header row
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
idx = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[hi + 1:]:
    if len(r) <= idx:
        continue
    try:
        s = int(r[idx])
    except ValueError:
        continue
    lines.append((s, r[0], r[1][:110]))
tot = sum(s for s, _, _ in lines)
for s, ln, src in sorted(lines, reverse=True)[:k]:
    print(f"{s:8d} {100*s/tot:5.1f}%  L{ln:5s} {src}")
