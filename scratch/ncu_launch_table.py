"""Summarise an ncu --csv launch list: per kernel name, median duration and DRAM bytes."""
import csv, sys, collections, statistics
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if "Metric Value" in r][0]
h = rows[i]
d = collections.defaultdict(dict)
for r in rows[i + 1:]:
    x = dict(zip(h, r))
    d[int(x["ID"])][x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
    d[int(x["ID"])]["name"] = x["Kernel Name"][:60]
for idd in sorted(d):
    e = d[idd]
    print(idd, e["name"], "%.2f us" % (e.get("gpu__time_duration.sum", 0) / 1000), "%.2f MB" % (e.get("dram__bytes_read.sum", 0) / 1e6))
