"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name (dev tool)."""
import csv, re, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    name = re.sub(r"\(.*", "", name)[:110]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
    tot[name] += ms
    cnt[name] += 1
T = sum(tot.values())
print(f"Total kernel time {T:.1f} ms over {sum(cnt.values())} launches.\n")
print("| share | launches | total ms | kernel |\n|---:|---:|---:|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print(f"| {100 * v / T:.2f}% | {cnt[k]} | {v:.2f} | `{k}` |")
