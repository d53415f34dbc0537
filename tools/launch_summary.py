"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel: total ms, launches."""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in csv.DictReader(io.StringIO(txt)):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.3f} ms {100 * t / tot:5.1f}% {c:6d}  {n}")
print(f"{tot:9.3f} ms total")
