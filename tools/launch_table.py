"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ other metrics]) per kernel:
python tools/launch_table.py launches.csv [last_n_launches]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if "Kernel Name" in r][0]
launch = collections.OrderedDict()
for r in rows:
    if len(r) != len(hdr) or r == hdr:
        continue
    d = dict(zip(hdr, r))
    launch.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", "")[:48]})[d["Metric Name"]] = \
        (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
ids = list(launch)
if len(sys.argv) > 2:
    ids = ids[-int(sys.argv[2]):]
for i in ids:
    m = launch[i]
    t = m.get("gpu__time_duration.sum", (0, "ns"))
    us = t[0] / 1000 if t[1] == "ns" else t[0] * (1000 if t[1] == "ms" else 1)
    extra = " ".join(f"{k.split('__')[1][:18]}={v[0]:.3g}" for k, v in m.items() if k not in ("name", "gpu__time_duration.sum"))
    print(f"{i:>5} {m['name']:48s} {us:9.1f} us  {extra}")
