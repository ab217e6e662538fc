"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X`
launch list into per-kernel launches / total time / share (JSON).
Times are cold-cache and serialised: compare shares, not absolutes."""
import csv, io, json, sys

log, out, cmd = sys.argv[1], sys.argv[2], " ".join(sys.argv[3:])
lines = [l for l in open(log) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
agg = {}
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[r["Metric Unit"]]
    k = agg.setdefault(r["Kernel Name"][:100], [0, 0.0])
    k[0] += 1
    k[1] += us
tot = sum(v[1] for v in agg.values())
res = {"command": cmd, "note": "cold-cache, serialised per-launch times; compare shares, "
                               "not absolutes",
       "kernels": [{"kernel": k, "launches": n, "total_us": round(t, 1),
                    "share": round(t / tot, 4)}
                   for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]}
json.dump(res, open(out, "w"), indent=1)
for k in res["kernels"][:8]:
    print(f"{k['share']:.3f} {k['launches']:4d} {k['total_us']:10.1f} us  {k['kernel'][:70]}")
