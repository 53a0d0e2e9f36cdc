"""Per-launch device times from an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, by = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = by.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0][:40]})
        e[d["Metric Name"]] = d["Metric Value"]
for k, v in by.items():
    t = float(v.get("gpu__time_duration.sum", "nan").replace(",", ""))
    print(f"{k:>4} {v['name']:<40} {t / 1000:8.2f} us")
