"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import csv, io, re, sys
text = open(sys.argv[1]).read()
start = text.index('"ID"')
rows = [r for r in csv.DictReader(io.StringIO(text[start:])) if r["Metric Name"] == "gpu__time_duration.sum"]
for r in rows:
    name = re.sub(r"\(.*", "", r["Kernel Name"])[:48]
    print(f'{r["ID"]:>4} {name:<48} grid={r["Grid Size"]:<14} {float(r["Metric Value"])/1e3:10.1f} us')
