"""Summarize an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, tot, cnt = None, collections.defaultdict(float), collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[d["Metric Unit"]]
        tot[name] += float(d["Metric Value"].replace(",", "")) * scale
        cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{k:36s} {cnt[k]:4d} {v:10.1f} us {100 * v / T:5.1f}%")
print(f"total {T / 1e3:.2f} ms over {sum(cnt.values())} launches")
