"""Summarise an ncu --csv launch list (gpu__time_duration.sum, optional dram
bytes) per kernel: count, mean time, total, DRAM GB per launch."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"])
    agg.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
per = collections.OrderedDict()
for (i, name), m in agg.items():
    k = name.split("(")[0][:70]
    per.setdefault(k, []).append(m)
print(f"{'kernel':70s} {'n':>4s} {'mean ms':>9s} {'total ms':>9s} {'DRAM GB/launch':>14s}")
for k, ms in per.items():
    t = [m.get("gpu__time_duration.sum", 0) / 1e6 for m in ms]
    b = [(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e9 for m in ms]
    print(f"{k:70s} {len(ms):4d} {sum(t)/len(t):9.3f} {sum(t):9.3f} {sum(b)/len(b):14.3f}")
