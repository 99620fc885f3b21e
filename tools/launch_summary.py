"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import csv, sys, collections, re
rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"k_items<hk::(\w+)>", name)
    key = m.group(1) if m else name.split("(")[0][-60:]
    rows.append((key, float(r["Metric Value"].replace(",", "")) / 1e3))
tot = collections.defaultdict(float); cnt = collections.Counter()
for k, us in rows:
    tot[k] += us; cnt[k] += 1
all_us = sum(tot.values())
print(f"{len(rows)} launches, {all_us/1e3:.2f} ms total (ncu, serialised, cold-cache)")
print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg us':>9s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} {cnt[k]:8d} {tot[k]/1e3:10.3f} {tot[k]/all_us:7.1%} {tot[k]/cnt[k]:9.2f}")
