"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file):
   python tools/launch_summary.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows:
    if r[-3] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(CUtensorMap_st.*|\(.*", "", r[4]).strip()
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(r[-2], 1.0)
    tot[name] += float(r[-1].replace(",", "")) * scale
    cnt[name] += 1
all_us = sum(tot.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 "
      "--warmup 1 --no-e2e --no-cpu")
print("# (cold-cache, serialised launches: compare SHARES, not absolute times)")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:70s} n={cnt[k]:4d} total={tot[k] / 1e3:9.3f} ms share={tot[k] / all_us * 100:5.1f}% "
          f"avg={tot[k] / cnt[k]:9.3f} us")
